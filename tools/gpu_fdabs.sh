python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fin_build.log 2>&1
for c in C3 C3B C5; do CFG=$c bash tools/variants.sh "abs|GACE_X=1" >> gpurun_out/var_summary.txt 2>&1; done
CFG=C3 bash tools/variants.sh "nofd|GACE_NO_FDIRECT=1" >> gpurun_out/var_summary.txt 2>&1
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/fin_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/var_summary.txt
cat gpurun_out/var_summary.txt
