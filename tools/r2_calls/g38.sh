# round-2 call 38: k_primary CTA size (256 default vs 128 / 64 / 32; 64 with 20 CTAs per SM)
bash tools/variants.sh
