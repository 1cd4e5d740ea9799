python -c "import __graft_entry__ as g; g.build()"
cat > /tmp/cmp3.py <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2404_19075_b200 import _lib as D, synth
dev = torch.device("cuda", 0)
name = sys.argv[1]; n = int(sys.argv[2])
over = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
g = synth.geometry(name, **over); th, t = synth.views(name, **over); f = synth.field(name)
ctx = D.create(0)
D.set_geometry(ctx, g, th, t)
D.set_field_weights(ctx, f, torch.tensor(synth.grff_matrix(f["C"], 0.1, 0.5), device=dev), torch.tensor(synth.init_params(f["C"], f["L"]), device=dev))
idx = torch.tensor(synth.pixel_batch(name, n, seed=3, **over), device=dev)
y = torch.tensor(synth.synthetic_y(n, 1.0), device=dev)
P = synth.param_count(f["C"], f["L"])
grad = torch.zeros(P + 1, device=dev)
D.project_and_grad(ctx, idx, y, grad)
torch.cuda.synchronize()
print("status", D.get_device_status(ctx))
np.save(sys.argv[4] if len(sys.argv) > 4 else "/tmp/g.npy", grad.cpu().numpy())
PY
DINR_BWD3=1 timeout 120 python /tmp/cmp3.py cone4d2048 128 "{}" /tmp/g3.npy > gpurun_out/r3e_cmp.log 2>&1
timeout 120 python /tmp/cmp3.py cone4d2048 128 "{}" /tmp/g2.npy >> gpurun_out/r3e_cmp.log 2>&1
python -c "
import numpy as np
a=np.load('/tmp/g3.npy'); b=np.load('/tmp/g2.npy')
print('bwd3 vs k3 maxrel', np.max(np.abs(a-b))/np.max(np.abs(b)))" >> gpurun_out/r3e_cmp.log 2>&1
for i in 1 2; do
DINR_BWD3=1 timeout 300 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r3e_bwd3_$i.json 2>>gpurun_out/r3e.err
timeout 300 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r3e_k3_$i.json 2>>gpurun_out/r3e.err
done
timeout 300 python bench.py --workload parallel64 --steps 20 --warmup 5 > gpurun_out/r3e_p64.json 2>>gpurun_out/r3e.err
