# round-2 call 34: k_asm_eval occupancy variants (VC_ASM_EVAL_MINB 6 / 10 / 12 / 16 vs the default 8)
bash tools/variants.sh
