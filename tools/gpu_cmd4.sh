python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c4_build.log 2>&1
CFG=C3 bash tools/variants.sh "head|GACE_X=1" "pref|GACE_JIT_DEFS=GACE_PREFETCH=1" "pref768|GACE_JIT_DEFS=GACE_PREFETCH=1 GACE_JIT_THREADS=768" "l2u|GACE_JIT_DEFS=GACE_L2_PREFETCH_U=1" "t768|GACE_JIT_THREADS=768" "t512|GACE_JIT_THREADS=512" > gpurun_out/var_summary.txt 2>&1
CFG=C2 bash tools/variants.sh "head|GACE_X=1" >> gpurun_out/var_summary.txt 2>&1
python tools/profile_probe.py --config C3 --probes 4 > gpurun_out/c3_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gace_jit_probe -s 1 -c 1 -o gpurun_out/c3_head python tools/profile_probe.py --config C3 --probes 4 > gpurun_out/c3_ncu.log 2>&1
cat gpurun_out/var_summary.txt
