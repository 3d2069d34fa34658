"""Per-layer latency of the layer kernel at tiny batches (diagnostics):
M = 0 (every launch exits at once: launch + teardown cost), M = 128 (one
feature tile: a single item's prologue -> fill -> compute -> publish chain),
and a few larger M. Prints microseconds per layer launch, CUDA-event timed
over the whole C2 layer loop."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2007_14152_b200 import engine  # noqa: E402
from paper_2007_14152_b200.model import InferenceConfig  # noqa: E402

cfg = dict(bench.CONFIGS["c2"], inputs=8192)
model, inputs = bench.build_workload(cfg)
prepared = engine.prepare_model(model, InferenceConfig(), "optimized")
net = engine.device_network(prepared, model.bias)
ws = engine.workspace(model.neurons, 8192, model.num_layers)
x = torch.from_numpy(np.ascontiguousarray(np.asarray(inputs.data).T)).cuda()
c = torch.from_numpy(np.ascontiguousarray(inputs.categories)).cuda()
L = model.num_layers
for m in (0, 128, 1024, 4096, 8192):
    ts = []
    for rep in range(4):
        engine.stage_inputs(ws, x, c, net)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        engine.run_layers(net, ws, m)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / L)
    print(f"M={m:5d}: {np.median(ts[1:]):7.1f} us per layer")
