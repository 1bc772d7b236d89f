mkdir -p gpurun_out
cat > /tmp/sd.py <<'PY'
import sys; sys.path.insert(0,'.')
import torch, synth
from paper_2512_19750_b200 import gace
w=synth.get('D'); cols=[w.column(c,device='cuda') for c in range(4)]; torch.cuda.synchronize()
t=gace.Table(cols); print(t.probe_sets(w.preds,w.sets,1.0,0)[0], t.last_timing()['scan_ms']); t.detach()
PY
python /tmp/sd.py > gpurun_out/sd_plain.log 2>&1 && ncu --set full --clock-control none -k regex:sets_kernel -c 1 -o gpurun_out/prof_D_1 python /tmp/sd.py > gpurun_out/ncu_D1.log 2>&1; echo rc=$?; tail -2 gpurun_out/ncu_D1.log
