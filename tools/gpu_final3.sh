python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fin_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc=$?" > gpurun_out/var_summary.txt
for c in C1 C3 C2 C5 C4; do python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --cold-batches 0 > gpurun_out/var_$c.json 2>gpurun_out/var_$c.err; python -c "
import json; d=json.loads(open('gpurun_out/var_$c.json').read().strip().splitlines()[-1]); print('$c', {k: round(v,4) for k,v in d['stages_ms'].items()}, 'step', round(d['ms_per_step'],4), 'p50', round(d['latency_ms']['p50'],4))" >> gpurun_out/var_summary.txt 2>&1; done
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/fin_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/var_summary.txt
cat gpurun_out/var_summary.txt
