mkdir -p gpurun_out
out=gpurun_out/b26.txt; : > $out
SPDNN_NVCC_DEFINES="-DSPDNN_LTRACE" python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 300 python tools/trace_layers.py c2 --runs 1 >> $out 2>&1
SPDNN_CHAIN=0 timeout 300 python tools/trace_layers.py c2 --runs 1 >> $out 2>&1
python - >> $out 2>&1 <<'PY'
import time, torch, numpy as np, sys, os
sys.path.insert(0, '.')
import bench
from paper_2007_14152_b200 import engine
from paper_2007_14152_b200.model import InferenceConfig
cfg = bench.CONFIGS['c2']
model, inputs = bench.build_workload(cfg)
net = engine.device_network(engine.prepare_model(model, InferenceConfig(), "optimized"), model.bias)
m, L = inputs.active_count, model.num_layers
ws = engine.workspace(net.neurons, m, L)
x = torch.from_numpy(np.ascontiguousarray(np.asarray(inputs.data).T)).cuda()
c = torch.from_numpy(np.ascontiguousarray(inputs.categories)).cuda()
for _ in range(2):
    engine.stage_inputs(ws, x, c, net); engine.run_layers(net, ws, m)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter(); engine.stage_inputs(ws, x, c, net); t1 = time.perf_counter()
    engine.run_layers(net, ws, m); t2 = time.perf_counter(); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"host stage {1e3*(t1-t0):.2f} ms, run_layers call {1e3*(t2-t1):.2f} ms, to sync {1e3*(t3-t2):.2f} ms")
PY
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
cat $out
