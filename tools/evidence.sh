set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ev_build.log 2>&1
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ev_smi.txt
python bench.py > gpurun_out/ev_bench_default.json 2> gpurun_out/ev_bench_default.err; echo "default rc=$?" >> gpurun_out/ev_rc.txt
for c in C1 C2 C3 C3B C4 C5_i64 D D_m1_k16; do python bench.py --config $c --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/ev_bench_$c.json 2> gpurun_out/ev_bench_$c.err; echo "$c rc=$?" >> gpurun_out/ev_rc.txt; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err; echo "ref rc=$?" >> gpurun_out/ev_rc.txt
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ev_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'gace_jit_probe|probe_kernel|fin_|minmax|ceil_|sample_mask' -c 600 --csv --log-file gpurun_out/ev_launches_C5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ev_ncu_launch.log 2>&1; echo "launches rc=$?" >> gpurun_out/ev_rc.txt
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --cold-batches 0 > gpurun_out/ev_plain_dev.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'gace_jit_probe|probe_kernel|fin_|minmax|ceil_|sample_mask' -c 600 --csv --log-file gpurun_out/ev_launches_C5_device.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --cold-batches 0 > gpurun_out/ev_ncu_launch_dev.log 2>&1; echo "launches dev rc=$?" >> gpurun_out/ev_rc.txt
python tools/profile_probe.py --probes 4 > gpurun_out/ev_prof_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gace_jit_probe -s 1 -c 1 -o gpurun_out/ev_c5 python tools/profile_probe.py --probes 4 > gpurun_out/ev_ncu_full.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/ev_rc.txt
# the HLL-completion exit switched off (report the number without the data-dependent exit)
GACE_NO_CEIL=1 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --cold-batches 0 > gpurun_out/ev_bench_C5_noceil.json 2> gpurun_out/ev_bench_C5_noceil.err; echo "noceil rc=$?" >> gpurun_out/ev_rc.txt
timeout 600 python tools/cold_diag.py C5 C4 C5_i64 C3 C3B C2 C1 > gpurun_out/ev_cold.log 2>&1; echo "cold rc=$?" >> gpurun_out/ev_rc.txt
echo done
