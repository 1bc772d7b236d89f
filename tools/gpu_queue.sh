python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fin_build.log 2>&1
CFG=C2 bash tools/variants.sh "scanq|GACE_X=1" "scanq2|GACE_X=2" > gpurun_out/var_summary.txt 2>&1
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/fin_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/var_summary.txt
python tools/profile_probe.py --config C2 --probes 4 > gpurun_out/c2q_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gace_jit_probe -s 1 -c 1 -o gpurun_out/c2_q python tools/profile_probe.py --config C2 --probes 4 > gpurun_out/c2q_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/var_summary.txt
cat gpurun_out/var_summary.txt
