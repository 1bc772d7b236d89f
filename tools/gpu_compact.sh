python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cp_build.log 2>&1
timeout 600 python tools/rate_sweep.py > gpurun_out/cp_rates.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/fin_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/cp_rates.log
cat gpurun_out/cp_rates.log
