python -c "import __graft_entry__ as g; g.build()"
python -m paper_2404_19075_b200.build --variant p2 -DF3_PIECES=2 > /dev/null
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
sed -i 's#^from paper_2404_19075_b200 import _lib as D, synth#from paper_2404_19075_b200 import _lib as D, synth\nif os.environ.get("DINR_LIB"): D.load(os.path.join(os.getcwd(), "paper_2404_19075_b200", os.environ["DINR_LIB"]))#' /tmp/cmp3.py
timeout 120 python /tmp/cmp3.py cone4d2048 128 "{}" /tmp/g3.npy > gpurun_out/r3a_cmp.log 2>&1
DINR_LIB=libdinr_var_p2.so timeout 120 python /tmp/cmp3.py cone4d2048 128 "{}" /tmp/g2.npy >> gpurun_out/r3a_cmp.log 2>&1
python -c "
import numpy as np
a=np.load('/tmp/g3.npy'); b=np.load('/tmp/g2.npy')
print('p4 vs p2 maxabs', np.max(np.abs(a-b)), 'equal', np.array_equal(a,b))" >> gpurun_out/r3a_cmp.log 2>&1
for w in cone4d2048 cone512; do python tools/variant_time.py $w libdinr.so libdinr_var_p2.so libdinr.so libdinr_var_p2.so > gpurun_out/r3a_vt_$w.txt 2>&1; done
timeout 300 python bench.py --steps 20 --warmup 5 --cpu-baseline-seconds 0 > gpurun_out/r3a_c.json 2>gpurun_out/r3a.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "cone or full" > gpurun_out/r3a_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3a_pytest.log
