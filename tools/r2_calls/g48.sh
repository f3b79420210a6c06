# round-2 call 48: CTA sizes of the emitter filter and the survivor evaluation (256 default vs 128 / 64)
bash tools/variants.sh
