python -c "import __graft_entry__ as g; g.build()" > gpurun_out/nm_build.log 2>&1
python tools/profile_probe.py --config C4 --probes 4 > gpurun_out/nm_c4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gace_jit_probe -s 1 -c 1 -o gpurun_out/nm_c4 python tools/profile_probe.py --config C4 --probes 4 > gpurun_out/nm_c4_ncu.log 2>&1; echo "c4 rc=$?" > gpurun_out/nm_rc.txt
python tools/profile_probe.py --config C5_i64 --probes 4 > gpurun_out/nm_i64_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gace_jit_probe -s 1 -c 1 -o gpurun_out/nm_i64 python tools/profile_probe.py --config C5_i64 --probes 4 > gpurun_out/nm_i64_ncu.log 2>&1; echo "i64 rc=$?" >> gpurun_out/nm_rc.txt
cat gpurun_out/nm_rc.txt
