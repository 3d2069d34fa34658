"""Cycle accounting of the layer kernel (library built with -DSPDNN_PROFILE).

    SPDNN_NVCC_DEFINES=-DSPDNN_PROFILE python tools/prof_cycles.py [c2] [--plan k=v,...]

Runs one warm inference, resets the counters, runs one more and prints where
the consumer and producer warps spend their cycles. Diagnostics only (the
clock64 marks perturb the kernel slightly); never a bench number.
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2007_14152_b200 import _native, engine  # noqa: E402
from paper_2007_14152_b200.model import InferenceConfig  # noqa: E402

_native.build(force=True)
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c2"]
plan = sys.argv[sys.argv.index("--plan") + 1] if "--plan" in sys.argv else ""
if "--inputs" in sys.argv:
    cfg = dict(cfg, inputs=int(sys.argv[sys.argv.index("--inputs") + 1]))
params = engine.PlanParams(**{k: int(v) for k, v in (kv.split("=") for kv in plan.split(",") if kv)})
model, inputs = bench.build_workload(cfg)
prepared = engine.prepare_model(model, InferenceConfig(), "optimized", params=params)
net = engine.device_network(prepared, model.bias)
m = inputs.active_count
ws = engine.workspace(model.neurons, m, model.num_layers)
x = torch.from_numpy(np.ascontiguousarray(np.asarray(inputs.data).T)).cuda()
c = torch.from_numpy(np.ascontiguousarray(inputs.categories)).cuda()
lib = _native.lib()
out = (ctypes.c_uint64 * 16)()
for rep in range(2):
    torch.cuda.synchronize()
    lib.spdnn_profile_read(out, 16, 1)
    engine.stage_inputs(ws, x, c, net)
    engine.run_layers(net, ws, m)
    torch.cuda.synchronize()
lib.spdnn_profile_read(out, 16, 0)
v = np.array(list(out), dtype=np.float64)
cons, prod = v[:8], v[8:]
names_c = ["wait for data", "record loop", "epilogue", "bookkeeping"]
names_p = ["empty-slot wait", "barrier A", "bulk copies", "metadata", "barrier B", "header+fetch",
           "gather4 issue", "cp.async path"]
print("consumer warps: total %.3g warp-cycles" % cons.sum())
for i, nm in enumerate(names_c):
    print(f"  {nm:16s} {cons[i] / cons.sum() * 100:6.1f} %")
print("producer warps: total %.3g warp-cycles" % prod.sum())
for i, nm in enumerate(names_p):
    print(f"  {nm:16s} {prod[i] / prod.sum() * 100:6.1f} %")
