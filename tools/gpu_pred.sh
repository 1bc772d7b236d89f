python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pr_build.log 2>&1
timeout 600 python tools/rate_sweep.py > gpurun_out/pr_rates.log 2>&1
CFG=C2 bash tools/variants.sh "pred|GACE_X=1" >> gpurun_out/pr_rates.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/fin_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/pr_rates.log
cat gpurun_out/pr_rates.log
