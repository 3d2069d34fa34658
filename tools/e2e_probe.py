import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2007_14152_b200 import engine
from paper_2007_14152_b200.model import InferenceConfig
cfg = bench.CONFIGS["c2"]
pinned, batch = bench.pinned_inputs(cfg)
model, _ = bench.build_workload(dict(cfg, inputs=1))
prepared = engine.prepare_model(model, InferenceConfig(), "optimized")
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = engine.infer(model, batch, InferenceConfig(), prepared=prepared, values=False)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"e2e {1e3*(t1-t0):.1f} ms; elapsed(in-call clock) {1e3*r.elapsed_seconds:.1f} ms; device {1e3*r.device_seconds:.1f} ms")
n, L = model.neurons, model.num_layers
print("head features:", engine.pipeline_head(batch.active_count, n, L,
                                              sum(l.nnz for l in model.layers)))
