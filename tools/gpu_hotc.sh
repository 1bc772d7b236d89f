python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fin_build.log 2>&1
CFG=C3 bash tools/variants.sh "hotc|GACE_X=1" "nohotc|GACE_NO_HOTC=1" > gpurun_out/var_summary.txt 2>&1
CFG=C3B bash tools/variants.sh "hotc|GACE_X=1" "nohotc|GACE_NO_HOTC=1" >> gpurun_out/var_summary.txt 2>&1
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/fin_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/var_summary.txt
python tools/profile_probe.py --config C3 --probes 4 > gpurun_out/c3h_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gace_jit_probe -s 1 -c 1 -o gpurun_out/c3_hotc python tools/profile_probe.py --config C3 --probes 4 > gpurun_out/c3h_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/var_summary.txt
cat gpurun_out/var_summary.txt
