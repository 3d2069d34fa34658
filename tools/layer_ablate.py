"""Time one steady-state layer launch in isolation (diagnostics).

    SPDNN_NVCC_DEFINES="-DSPDNN_ABLATE_STORE" python tools/layer_ablate.py [c2] [--layer 200]

Runs the network up to --layer, then launches that layer 20 times on the same
input state (the outputs are not chained) and prints the mean CUDA-event
time. With the SPDNN_ABLATE_* build flags (no stores / no record loop / no
row staging) the deltas show which part of the kernel the time is bound by.
Never a bench number.
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
layer = int(sys.argv[sys.argv.index("--layer") + 1]) if "--layer" in sys.argv else 200
model, inputs = bench.build_workload(cfg)
plan = sys.argv[sys.argv.index("--plan") + 1] if "--plan" in sys.argv else ""
params = engine.PlanParams(**{k: int(v) for k, v in (kv.split("=") for kv in plan.split(",") if kv)})
prepared = engine.prepare_model(model, InferenceConfig(), "optimized", params=params)
net = engine.device_network(prepared, model.bias)
m = inputs.active_count
ws = engine.workspace(model.neurons, m, model.num_layers)
x = torch.from_numpy(np.ascontiguousarray(np.asarray(inputs.data).T)).cuda()
c = torch.from_numpy(np.ascontiguousarray(inputs.categories)).cuda()
# replay `layer` on the staged network inputs (values do not matter for the
# timing) with a fixed active count: --m (default: C2's steady state)
engine.stage_inputs(ws, x, c, net)
mi = int(sys.argv[sys.argv.index("--m") + 1]) if "--m" in sys.argv else 30924
# replay `layer` from a fresh contiguous state of mi features: buffer 0 holds
# the inputs (any values), a = 0..mi-1
i, o = 0, 1
ws.a[0][:mi].copy_(ws.iota[:mi])
opts = engine.run_opts(net)
lib = _native.lib()
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
prof = (ctypes.c_uint64 * 24)()
torch.cuda.synchronize()
lib.spdnn_profile_read(prof, 24, 1)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
for r in range(21):
    ws.counts[layer] = mi
    ws.counts[layer + 1] = 0
    ws.work[layer] = 0
    ev[r].record()
    _native.check(lib.spdnn_layer_forward(
        ctypes.byref(net.layer_devs[layer]), engine._dptr(net.bias), engine._dptr(ws.y[i]),
        engine._dptr(ws.y[o]), ws.ld, engine._dptr(ws.a[i]), engine._dptr(ws.cat[i]),
        ctypes.c_void_p(ws.counts.data_ptr() + 4 * layer), engine._dptr(ws.a[o]),
        engine._dptr(ws.cat[o]), ctypes.c_void_p(ws.counts.data_ptr() + 4 * (layer + 1)),
        ctypes.byref(ws.scratch), ctypes.c_void_p(ws.work.data_ptr() + 4 * layer),
        ctypes.byref(opts), sp), "spdnn_layer_forward")
torch.cuda.synchronize()
ts = [ev[r].elapsed_time(ev[r + 1]) * 1e3 for r in range(20)]
plan = sys.argv[sys.argv.index("--plan") + 1] if "--plan" in sys.argv else ""
print(f"{os.environ.get('SPDNN_NVCC_DEFINES', '(default)')} [{plan}]: layer {layer} "
      f"{np.median(ts):.1f} us (M={mi})")
lib.spdnn_profile_read(prof, 24, 0)
v = np.array(list(prof), dtype=np.float64)
if v.sum() > 0:
    c, p = v[:4], v[8:16]
    print("  consumer %%: wait %.1f loop %.1f epilogue %.1f bookkeeping %.1f" %
          tuple(c / c.sum() * 100))
    print("  producer %%: empty %.1f barA %.1f bulk %.1f meta %.1f barB %.1f hdr %.1f "
          "gather4 %.1f cpasync %.1f" % tuple(p / p.sum() * 100))
    ch = v[16:22]
    if ch[4] > 0:
        print("  ring entry chain (us @1.965 GHz): issue %.2f fill %.2f consume %.2f release %.2f"
              % (ch[0] / ch[4] / 1965, ch[1] / ch[4] / 1965, ch[2] / ch[4] / 1965,
                 ch[3] / max(ch[5], 1) / 1965))
