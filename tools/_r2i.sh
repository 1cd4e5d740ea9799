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
for case in "cone512 40 {\"n_s\":64}" "cone512 300 {}" "cone4d2048 128 {}"; do
  set -- $case
  DINR_BWD3=1 timeout 120 python /tmp/cmp3.py $1 $2 "$3" /tmp/g3.npy > gpurun_out/r2i_cmp_$1_$2.log 2>&1; echo "bwd3 rc $?" >> gpurun_out/r2i_cmp_$1_$2.log
  timeout 120 python /tmp/cmp3.py $1 $2 "$3" /tmp/g2.npy >> gpurun_out/r2i_cmp_$1_$2.log 2>&1
  python -c "
import numpy as np
a=np.load('/tmp/g3.npy'); b=np.load('/tmp/g2.npy')
print('maxabs', np.max(np.abs(a-b)), 'rel', np.max(np.abs(a-b))/np.max(np.abs(b)), 'equal', np.array_equal(a,b))" >> gpurun_out/r2i_cmp_$1_$2.log 2>&1
done
DINR_BWD3=1 timeout 300 python bench.py --workload cone4d2048 --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r2i_cone4d2048_bwd3.json 2>gpurun_out/r2i.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_fwd3 -c 1 -o gpurun_out/r2i_fwd3 python bench.py --workload cone4d2048 --steps 2 --warmup 3 --cpu-baseline-seconds 0 > gpurun_out/r2i_ncu.log 2>&1
DINR_BWD3=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_bwd3 -c 1 -o gpurun_out/r2i_bwd3 python bench.py --workload cone4d2048 --steps 2 --warmup 3 --cpu-baseline-seconds 0 > gpurun_out/r2i_ncu2.log 2>&1
