"""Experiment: the batch split into independent chains (features never
interact), each chain's layer loop on its own stream, so one chain's layer
boundary (tail, grid completion, first fill) overlaps the other chain's
layer. Prints device ms per inference for 1, 2 and 3 chains. Diagnostics.

    python tools/dual_chain.py [c1|c2|c3] [--steps K]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2007_14152_b200 import engine  # noqa: E402
from paper_2007_14152_b200.model import InferenceConfig  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c1"]
steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 5
model, inputs = bench.build_workload(cfg)
prepared = engine.prepare_model(model, InferenceConfig(), "optimized")
net = engine.device_network(prepared, model.bias)
m, n, L = inputs.active_count, model.neurons, model.num_layers
x = torch.from_numpy(np.ascontiguousarray(np.asarray(inputs.data).T)).cuda()
c = torch.from_numpy(np.ascontiguousarray(inputs.categories)).cuda()
ref = None
for chains in (1, 2, 3, 4):
    bounds = np.linspace(0, m, chains + 1).astype(int)
    # bounds on 128-feature tile boundaries
    bounds[1:-1] = (bounds[1:-1] + 64) // 128 * 128
    wss = [engine.Workspace(n, int(bounds[i + 1] - bounds[i]), L, torch.device("cuda"))
           for i in range(chains)]
    streams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(chains - 1)]

    def step():
        main = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(main)
        runs = []
        for i in range(chains):
            s = streams[i]
            s.wait_event(ev)
            with torch.cuda.stream(s):
                lo, hi = int(bounds[i]), int(bounds[i + 1])
                engine.stage_inputs(wss[i], x[lo:hi], c[lo:hi], net)
                runs.append(engine.run_layers(net, wss[i], hi - lo))
        for s in streams[1:]:
            e = torch.cuda.Event()
            e.record(s)
            main.wait_event(e)
        return runs

    for _ in range(3):
        runs = step()
    torch.cuda.synchronize()
    cats = np.sort(np.concatenate([engine.collect(r, want_values=False)[1].cpu().numpy()
                                   for r in runs]))
    if ref is None:
        ref = cats
    assert np.array_equal(cats, ref), "chains changed the survivors"
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    te = m * float(sum(l.nnz for l in model.layers)) / (ms / 1e3) / 1e12
    print(f"{cfg['name'][:40]} chains={chains}: {ms:.2f} ms/inference, {te:.2f} TE/s "
          f"(survivors {len(cats)})", flush=True)
    del wss
    torch.cuda.empty_cache()
