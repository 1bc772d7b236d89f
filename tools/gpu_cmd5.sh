python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c5_build.log 2>&1
timeout 900 python tools/calibrate_cost.py gpurun_out/cost_cold.json --cold > gpurun_out/cost_cold.log 2>&1; echo "cold rc=$?" > gpurun_out/c5_rc.txt
timeout 900 python tools/calibrate_cost.py gpurun_out/cost_warm.json > gpurun_out/cost_warm.log 2>&1; echo "warm rc=$?" >> gpurun_out/c5_rc.txt
python tools/profile_probe.py --config C2 --probes 4 > gpurun_out/c2_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gace_jit_probe -s 1 -c 1 -o gpurun_out/c2_head python tools/profile_probe.py --config C2 --probes 4 > gpurun_out/c2_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/c5_rc.txt
cat gpurun_out/c5_rc.txt
