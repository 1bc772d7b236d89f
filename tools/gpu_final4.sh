python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fin_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc=$?" > gpurun_out/fin_rc.txt
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/fin_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fin_rc.txt
bash tools/evidence.sh > gpurun_out/fin_evidence.log 2>&1; echo "evidence rc=$?" >> gpurun_out/fin_rc.txt
cat gpurun_out/fin_rc.txt gpurun_out/ev_rc.txt
