python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fd_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fd_rc.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fd_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fd_rc.txt
for c in C3 C3B C2; do python bench.py --config $c --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/fd_bench_$c.json 2>gpurun_out/fd_bench_$c.err; echo "$c rc=$?" >> gpurun_out/fd_rc.txt; done
GACE_NO_FDIRECT=1 python bench.py --config C3 --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/fd_bench_C3_nofd.json 2>&1
python tools/cold_diag.py C5 C4 C2 C3 C3B C1 > gpurun_out/fd_cold.log 2>&1; echo "cold rc=$?" >> gpurun_out/fd_rc.txt
GACE_PLAN_PROFILE=1 python tools/cold_diag.py C5 C3B > gpurun_out/fd_cold_prof.log 2>&1
