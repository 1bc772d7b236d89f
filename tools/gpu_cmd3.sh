python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fd_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fd_smoke.log 2>&1; echo "smoke rc=$?" > gpurun_out/var_summary.txt
bash tools/variants.sh "head|GACE_X=1" "noest|GACE_NO_LUT_ESTIMATE=1" >> gpurun_out/var_summary.txt 2>&1
for c in C4 C5_i64 C3 C1; do CFG=$c bash tools/variants.sh "head|GACE_X=1" >> gpurun_out/var_summary.txt 2>&1; done
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/fd_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/var_summary.txt
timeout 600 python tools/cold_diag.py C5 C4 C2 C3 C3B C1 > gpurun_out/fd_cold.log 2>&1
cat gpurun_out/var_summary.txt
