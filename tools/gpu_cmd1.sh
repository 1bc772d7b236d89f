bash tools/exit_diag.sh
bash tools/variants.sh "base|GACE_NO_REFINE=1" "refine|GACE_X=1" "refine_pf2|GACE_JIT_DEFS=GACE_L2_PREFETCH=2" "base_pf2|GACE_NO_REFINE=1 GACE_JIT_DEFS=GACE_L2_PREFETCH=2" > gpurun_out/var_summary.txt 2>&1
cat gpurun_out/var_summary.txt
