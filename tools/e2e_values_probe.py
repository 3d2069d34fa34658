"""Where the values=True end-to-end time goes (diagnostics): python tools/e2e_values_probe.py"""
import sys, time; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2007_14152_b200 import engine
from paper_2007_14152_b200.model import InferenceConfig
cfg=bench.CONFIGS['c2']
pinned, batch = bench.pinned_inputs(cfg)
model, _ = bench.build_workload(cfg)
prep = engine.prepare_model(model, InferenceConfig(), "optimized")
net = engine.device_network(prep, model.bias)
for rep in range(2):
    torch.cuda.synchronize(); t0=time.perf_counter()
    r = engine.infer(model, batch, InferenceConfig(), prepared=prep, values=True)
    t1=time.perf_counter()
    print('infer values=True', round((t1-t0)*1e3,1), 'ms; elapsed(loop)', round(r.elapsed_seconds*1e3,1))
m, n = batch.active_count, batch.neurons
ws = engine.workspace(n, m, model.num_layers)
x = engine.host_tensor(np.asarray(batch.data).T); c = engine.host_tensor(np.ascontiguousarray(batch.categories))
torch.cuda.synchronize(); t0=time.perf_counter()
engine.stage_inputs(ws, x, c, net); torch.cuda.synchronize(); t1=time.perf_counter()
run = engine.run_layers(net, ws, m); torch.cuda.synchronize(); t2=time.perf_counter()
counts, cats, vals = engine.collect(run, want_values=True); torch.cuda.synchronize(); t3=time.perf_counter()
h = vals.cpu(); t4=time.perf_counter()
hp = torch.empty(vals.shape, dtype=vals.dtype, pin_memory=True); t5=time.perf_counter()
hp.copy_(vals); torch.cuda.synchronize(); t6=time.perf_counter()
fb = engine.FeatureBatch(neurons=n, data=h.numpy().T, categories=cats.cpu().numpy(), total_inputs=m); t7=time.perf_counter()
print(f"stage {1e3*(t1-t0):.1f} layers {1e3*(t2-t1):.1f} collect {1e3*(t3-t2):.1f} d2h pageable {1e3*(t4-t3):.1f} pin alloc {1e3*(t5-t4):.1f} d2h pinned {1e3*(t6-t5):.1f} FeatureBatch {1e3*(t7-t6):.1f} (MB {vals.numel()*4/1e6:.0f})")
