"""Where a layer launch's fixed cost goes (library built with -DSPDNN_LTRACE;
diagnostics, never a bench number).

    SPDNN_NVCC_DEFINES=-DSPDNN_LTRACE python tools/trace_layers.py [c1|c2] [--runs R]

Runs R whole inferences, then reads the per-CTA %globaltimer marks of the last
64 layer launches and prints, per layer: its share of the chain (end of the
layer's last CTA minus the previous one's), how long CTAs sat in the grid
dependency wait, the ramp from the wait to the first entry's data, the busy
span, and the tail (last CTA's exit minus the mean exit).
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2007_14152_b200 import _native, engine  # noqa: E402
from paper_2007_14152_b200.model import InferenceConfig  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c1"]
runs = int(sys.argv[sys.argv.index("--runs") + 1]) if "--runs" in sys.argv else 3
model, inputs = bench.build_workload(cfg)
prepared = engine.prepare_model(model, InferenceConfig(), "optimized")
net = engine.device_network(prepared, model.bias)
m, L = inputs.active_count, model.num_layers
ws = engine.workspace(net.neurons, m, L)
x = torch.from_numpy(np.ascontiguousarray(np.asarray(inputs.data).T)).cuda()
c = torch.from_numpy(np.ascontiguousarray(inputs.categories)).cuda()
lib = _native.lib()
for _ in range(runs):
    engine.stage_inputs(ws, x, c, net)
    run = engine.run_layers(net, ws, m)
torch.cuda.synchronize()
counts = ws.counts[: L + 1].cpu().numpy()
buf = (ctypes.c_int64 * (64 * 160 * 6))()
_native.check(lib.spdnn_ltrace_read(buf, 64 * 160 * 6), "spdnn_ltrace_read")
tr = np.array(list(buf), dtype=np.float64).reshape(64, 160, 6)
if not tr.any():
    print("no trace (build with -DSPDNN_LTRACE)")
    sys.exit(0)
total = runs * L  # every spdnn_layer_forward call since the library loaded
grid = int((tr[:, :, 0] > 0).sum(axis=1).max())
layers = list(range(L - 64, L)) if L >= 64 else list(range(L))
print(f"{cfg['name'][:40]}: grid {grid} CTAs; per layer (us): chain share | dep wait | "
      "ramp to first data | busy | tail | entries/CTA")
prev_end = None
rows = []
for l in layers:
    s = (total - L + l) % 64
    t = tr[s, :grid] / 1e3  # ns -> us
    start, dep, first, end, grant, ent = (t[:, i] for i in range(6))
    ok = end > 0
    end_max = end[ok].max()
    share = end_max - prev_end if prev_end is not None else np.nan
    prev_end = end_max
    rows.append((l, counts[l], share, np.mean(dep[ok] - start[ok]), np.mean(first[ok] - dep[ok]),
                 np.mean(end[ok] - first[ok]), end_max - np.mean(end[ok]), np.mean(tr[s, :grid, 5][ok])))
for r in rows[1:12] + rows[-3:]:
    print(f"  layer {r[0]:4d} M={r[1]:6d}: {r[2]:7.1f} | {r[3]:6.1f} | {r[4]:6.1f} | {r[5]:7.1f} | "
          f"{r[6]:5.1f} | {r[7]:5.1f}")
a = np.array([r[2:] for r in rows[1:]], dtype=np.float64)
print("  mean: chain %.1f, dep wait %.1f, ramp %.1f, busy %.1f, tail %.1f, entries %.1f" %
      tuple(np.nanmean(a, axis=0)))
