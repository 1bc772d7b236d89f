bash tools/exit_diag.sh
bash tools/variants.sh "pf2|GACE_X=1" "pf1|GACE_JIT_DEFS=GACE_L2_PREFETCH=1" "pf2b|GACE_X=2" > gpurun_out/var_summary.txt 2>&1
for c in C3 C3B C2 C4 C5_i64; do CFG=$c bash tools/variants.sh "head|GACE_X=1" >> gpurun_out/var_summary.txt 2>&1; done
CFG=C3 bash tools/variants.sh "nofd|GACE_NO_FDIRECT=1" >> gpurun_out/var_summary.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/fd_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/var_summary.txt
timeout 600 python tools/cold_diag.py C5 C4 C2 C3 C3B C1 > gpurun_out/fd_cold.log 2>&1
cat gpurun_out/var_summary.txt
