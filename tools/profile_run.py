"""One inference of a bench workload, for ncu captures (never a bench number).

    python tools/profile_run.py [c1|c2|c3|c4] [--steps S]
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

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 1
if cfg.get("chunked"):  # C4: the network planned and uploaded 64 layers at a time
    from paper_2007_14152_b200 import ingest
    spec = ingest.GeneratorSpec(neurons=cfg["neurons"], layers=cfg["layers"],
                                connections_per_neuron=bench.K_CONN, bias_value=cfg["bias"],
                                seed=bench.MODEL_SEED)
    net = engine.DeviceNetwork.from_layers(ingest.iter_synthetic_layers(spec),
                                           ingest.synthetic_bias(spec), chunk=64)
    inputs = ingest.generate_synthetic_inputs(cfg["neurons"], cfg["inputs"], cfg["density"],
                                              seed=bench.INPUT_SEED)
else:
    model, inputs = bench.build_workload(cfg)
    prepared = engine.prepare_model(model, InferenceConfig(), "optimized")
    net = engine.device_network(prepared, model.bias)
m = inputs.active_count
ws = engine.workspace(net.neurons, m, net.num_layers)
x = torch.from_numpy(np.ascontiguousarray(np.asarray(inputs.data).T)).cuda()
c = torch.from_numpy(np.ascontiguousarray(inputs.categories)).cuda()
del inputs
for _ in range(steps):
    engine.stage_inputs(ws, x, c, net)
    run = engine.run_layers(net, ws, m)
torch.cuda.synchronize()
counts, cats, _ = engine.collect(run, want_values=False)
print("survivors", int(counts[-1]), "sum_active", int(counts[:-1].sum()))
