# round-2 call 55: occupancy bound of the persistent occlusion pass; assembly CTA split
bash tools/variants.sh
