python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fin_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc=$?" > gpurun_out/var_summary.txt
for c in C2 C5 C1; do CFG=$c bash tools/variants.sh "head|GACE_X=1" >> gpurun_out/var_summary.txt 2>&1; done
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/fin_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/var_summary.txt
cat gpurun_out/var_summary.txt
