#!/usr/bin/env python
"""Benchmark: TeraEdges/s of the sparse-DNN inference hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Workload (BASELINE.json configs[2], the configuration the metric "TeraEdges/s
at 1/2/4/8 B200" is quoted on; it fits one GPU): Graph-Challenge-style
synthetic network, 16384 neurons x 1920 layers, 32 connections per neuron,
weights 1/16, bias -0.4; 60000 binary inputs with density 0.4 (= |bias|,
SURVEY.md section 0 finding 4; the generator is the reference's, bit for
bit). One step = one full inference (all 1920 layers with pruning) over the
60000-input batch. `--config c1|c2|c4|c5` selects the other configs.

metric  : credited TeraEdges/s = 60000 * sum(nnz) / step time (the
          reference's and the paper's convention, spdnn/engine.py:290,
          PAPER.md:715: dead inputs are still credited at every layer).
value   : device-timed (CUDA events), inputs resident in HBM; each step
          re-lays the inputs out (spdnn_transpose_in) and runs every layer.
e2e     : the same metric through the public API (engine.infer on a
          FeatureBatch in pinned host memory): H2D of the inputs, the layer
          loop, D2H of the sorted survivor categories, every step.
roofline: the layer kernel (csrc/layer.cu), bytes per launch
          = 8*N*M_l + 6*nnz_l + 4*N, over the kernel's
          CUDA-event time measured around every launch in the timed steps.
cpu_baseline: the oracle port (oracle/spdnn_oracle.c) on the host cores, on a
          bounded column sample of the same workload.
--impl reference: the unmodified reference (baseline/_ref: spdnn.parallel.
          run_batch_parallel with one worker per host core) on a bounded
          sample, next to the port (run_reference).

--gpus N > 1: relaunched under torch.distributed.run with N local ranks
(or launched that way by the driver): batch-parallel over ranks (paper
section "Multi-GPU"; spdnn/parallel.py): the 60000 inputs are partitioned,
weights replicated, counts allgathered over NCCL, categories gathered to
rank 0; time = max over ranks.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(neurons=1024, layers=120, bias=-0.30, density=0.30, inputs=60000,
               name="graph-challenge-synthetic 1024x120, bias -0.3 (BASELINE.json configs[0])"),
    "c2": dict(neurons=4096, layers=480, bias=-0.35, density=0.35, inputs=60000,
               name="graph-challenge-synthetic 4096x480, bias -0.35 (BASELINE.json configs[1])"),
    "c3": dict(neurons=16384, layers=1920, bias=-0.40, density=0.40, inputs=60000,
               name="graph-challenge-synthetic 16384x1920, bias -0.4 (BASELINE.json configs[2])"),
    "c4": dict(neurons=65536, layers=1920, bias=-0.45, density=0.45, inputs=60000, chunked=True,
               name="graph-challenge-synthetic 65536x1920, bias -0.45 (BASELINE.json configs[3])"),
    "c5": dict(neurons=16384, layers=1920, bias=-0.40, density=0.40, inputs=60000, stress=True,
               workers=8,
               name="load-imbalance stress: skewed shards on config 3's network, rebalancing "
                    "on vs off (BASELINE.json configs[4])"),
}
K_CONN = 32
MODEL_SEED, INPUT_SEED = 1, 2


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def init_nccl_log():
    """NCCL's communicator-init lines (`nRanks N`) on stderr, so the run shows
    how many ranks the communicator really had; stdout keeps the JSON line."""
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")


def build_workload(cfg, rank=0, world=1):
    from paper_2007_14152_b200 import ingest
    spec = ingest.GeneratorSpec(neurons=cfg["neurons"], layers=cfg["layers"],
                                connections_per_neuron=K_CONN, bias_value=cfg["bias"],
                                seed=MODEL_SEED)
    model = ingest.generate_synthetic_network(spec)
    inputs = ingest.generate_synthetic_inputs(cfg["neurons"], cfg["inputs"], cfg["density"],
                                              seed=INPUT_SEED)
    return model, inputs


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, flag in zip(names, parts[4:8]):
                if flag.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfg_key: str):
    """DRAM bytes of one steady-state launch of the layer kernel from the
    newest committed ncu capture (profiles/r<N>_ncu_layer<L>_<cfg>.json).
    Returns (bytes, file name, layer index) or (None, None, None)."""
    import glob
    import re
    scale = {"byte": 1.0, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}
    files = glob.glob(os.path.join(ROOT, "profiles", f"r*_ncu_layer*_{cfg_key}.json"))
    if not files:
        return None, None, None
    files.sort(key=lambda f: int(re.search(r"r(\d+)_", os.path.basename(f)).group(1)))
    with open(files[-1]) as f:
        d = json.load(f)
    try:
        tot = sum(float(d[k][0]) * scale[d[k][1].lower()]
                  for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    except (KeyError, TypeError, ValueError):
        return None, None, None
    layer = int(re.search(r"_ncu_layer(\d+)_", os.path.basename(files[-1])).group(1))
    return tot, os.path.basename(files[-1]), layer


def cpu_baseline(model, inputs, sample_cols: int, threads: int, target_s: float = 0.0):
    """The oracle port on the host cores, on the first `sample_cols` inputs.
    With target_s > 0 the sample is first calibrated on a small slice and
    grown to about target_s seconds of CPU work (bounded by the batch)."""
    from oracle import oracle
    from paper_2007_14152_b200.model import make_feature_batch
    m_all = inputs.active_count
    if target_s > 0:
        probe = min(m_all, max(threads * 4, 64))
        sub = make_feature_batch(model.neurons, np.asfortranarray(inputs.data[:, :probe]))
        t0 = time.perf_counter()
        oracle.infer(model, sub, threads=threads, want_final=False)
        per_col = (time.perf_counter() - t0) / probe
        sample_cols = int(min(m_all, max(probe, target_s / max(per_col, 1e-9))))
    sub = make_feature_batch(model.neurons, np.asfortranarray(inputs.data[:, :sample_cols]))
    t0 = time.perf_counter()
    r = oracle.infer(model, sub, threads=threads, want_final=False)
    dt = time.perf_counter() - t0
    edges = sample_cols * sum(l.nnz for l in model.layers)
    return dict(value=edges / dt / 1e12, seconds=dt, counts=r.counts, sample_cols=sample_cols,
                categories=r.categories)


def run_reference_streamed(args, cfg):
    """C4's reference arm: the 32 GB network is generated layer by layer and
    the oracle runs each layer on a fixed 32-column sample as it streams by
    (only the oracle's time is counted); one pass = one step."""
    from paper_2007_14152_b200 import ingest
    spec = ingest.GeneratorSpec(neurons=cfg["neurons"], layers=cfg["layers"],
                                connections_per_neuron=K_CONN, bias_value=cfg["bias"],
                                seed=MODEL_SEED)
    threads = os.cpu_count() or 1
    cols = np.sort(np.random.default_rng(123).choice(cfg["inputs"], 32, replace=False))
    full = _sample_columns(cfg, cols)
    orc = StreamedOracle(full, np.arange(len(cols)), ingest.synthetic_bias(spec), threads)
    nnz = 0
    chunk = []
    for lay in ingest.iter_synthetic_layers(spec):
        nnz += lay.nnz
        chunk.append(lay)
        if len(chunk) == 16:
            orc(0, chunk)
            chunk = []
    if chunk:
        orc(0, chunk)
    v = len(cols) * nnz / orc.seconds / 1e12
    return v, orc.seconds, len(cols), threads, (
        f"{len(cols)} fixed-seed columns of {cfg['inputs']} through all {cfg['layers']} "
        f"layers, generated and run layer by layer (oracle/spdnn_oracle.c, {threads} threads, "
        f"{orc.seconds:.1f} s of oracle time)"), orc.counts


def _sample_columns(cfg, cols):
    """Columns `cols` of the synthetic input stream without holding the batch."""
    n, m = cfg["neurons"], cfg["inputs"]
    rng = np.random.default_rng(INPUT_SEED)
    out = np.empty((n, len(cols)), np.float32, order="F")
    for r0 in range(0, n, 1024):
        r1 = min(n, r0 + 1024)
        out[r0:r1, :] = rng.random((r1 - r0, m))[:, cols] < cfg["density"]
    return out


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_spdnn(cfg, port_counts, port_cols: int, workers: int, target_s: float = 10.0):
    """The unmodified reference (baseline/_ref, `spdnn` + numba) through its own
    public API, spdnn.parallel.run_batch_parallel(..., InferenceConfig(workers=
    host cores)), on a bounded sample: the first `cols` inputs through the
    network's first `lp` layers (its per-layer ELL preparation, ~0.26 s/layer
    at 16384 neurons, keeps the whole network out of reach of one bench run).
    Its active-edge rate (sum over layers of active_before * nnz / the
    reference's own elapsed_seconds) is extrapolated to the full network with
    the port's per-layer count sequence of the same inputs:
      t_full = sum_l count_l * nnz_l / rate,  TE/s = port_cols * sum nnz / t_full.
    Returns None when the reference is not installed."""
    if not os.path.isdir(os.path.join(REF_DIR, "spdnn")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        from spdnn import ingest as ring, parallel as rpar
        from spdnn.engine import prepare_model as rprep
        from spdnn.model import InferenceConfig as RConf, make_feature_batch as rbatch
    except ImportError as e:  # numba missing on this host
        log(f"reference not importable: {e}")
        return None
    n = cfg["neurons"]
    nnz_layer = n * K_CONN
    cols = int(min(cfg["inputs"], max(48 * workers, 512)))
    # layers: ELL preparation time ~ n * 16 us per layer; keep it near 10 s
    lp = int(max(4, min(cfg["layers"], 10.0 / (n * 16e-6))))
    t0 = time.perf_counter()
    model = ring.generate_synthetic_network(ring.GeneratorSpec(
        neurons=n, layers=lp, connections_per_neuron=K_CONN, bias_value=cfg["bias"],
        seed=MODEL_SEED))
    conf = RConf(workers=workers)
    prepared = rprep(model, conf, "optimized")
    t_prep = time.perf_counter() - t0
    data = _sample_columns(cfg, np.arange(cols))
    batch = rbatch(n, data)
    # numba JIT / cache load outside the clock
    rpar.run_batch_parallel(model, rbatch(n, data[:, :min(cols, 2 * workers)]), conf,
                            prepared=prepared)
    rates, secs = [], 0.0
    while secs < target_s or not rates:
        res, _, _ = rpar.run_batch_parallel(model, batch, conf, prepared=prepared)
        active_edges = sum(o.active_before for o in res.per_layer) * nnz_layer
        rates.append(active_edges / res.elapsed_seconds)
        secs += res.elapsed_seconds
    rate = float(np.median(rates))
    L = cfg["layers"]
    t_full = float(np.sum(np.asarray(port_counts[:L], np.float64))) * nnz_layer / rate
    value = port_cols * L * nnz_layer / t_full / 1e12
    return {"value": value, "unit": "TE/s", "cores": workers, "kind": "reference",
            "active_edge_rate_G": rate / 1e9,
            "sample": f"spdnn.parallel.run_batch_parallel (baseline/_ref, numba) with "
                      f"{workers} workers on the first {cols} inputs x first {lp} of {L} "
                      f"layers ({len(rates)} runs, {secs:.1f} s; ELL prep {t_prep:.1f} s "
                      f"untimed); active-edge rate {rate / 1e9:.2f} G/s extrapolated over "
                      f"the port's per-layer counts of the first {port_cols} inputs",
            "cpu_model": cpu_model()}


def run_reference(args, cfg):
    """--impl reference: rank 0 times the reference's CPU path on the host
    cores. The line's value is the unmodified reference (reference_spdnn,
    kind "reference") when baseline/_ref imports, else the C port
    (oracle/spdnn_oracle.c, kind "port"); the port's own figure is always
    reported under "port" (it also supplies the per-layer counts the
    reference's rate is extrapolated over)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    if cfg.get("chunked"):
        v, secs, sample, _, what, counts = run_reference_streamed(args, cfg)
        steps, warmup = 1, 0
    else:
        if cfg.get("stress"):
            model, _ = build_workload(dict(cfg, inputs=0))
            inputs = stress_inputs(cfg)
        else:
            model, inputs = build_workload(cfg)
        sample = args.cpu_sample
        vals, secs_l = [], []
        for _ in range(args.steps):
            r = cpu_baseline(model, inputs, sample, threads, target_s=args.cpu_seconds)
            sample = r["sample_cols"]
            vals.append(r["value"])
            secs_l.append(r["seconds"])
        v, secs, counts = float(np.median(vals)), float(np.median(secs_l)), r["counts"]
        steps, warmup = args.steps, args.warmup
        edges_full = cfg["inputs"] * sum(l.nnz for l in model.layers)
        what = (f"first {sample} of {cfg['inputs']} inputs through all {cfg['layers']} layers "
                f"(oracle/spdnn_oracle.c, {threads} threads); full-batch time extrapolates to "
                f"{edges_full / (v * 1e12):.1f} s")
        del model, inputs
    port = {"value": v, "unit": "TE/s", "cores": threads, "kind": "port", "sample": what,
            "cpu_model": cpu_model()}
    ref = None if args.port_only else reference_spdnn(cfg, counts, sample, threads)
    base = ref if ref is not None else port
    line = {
        "metric": "TeraEdges/s", "impl": "reference", "value": base["value"], "unit": "TE/s",
        "n_gpus": world, "steps": steps, "warmup": warmup, "ms_per_step": secs * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["name"], "inputs": cfg["inputs"],
                   "input_density": cfg["density"], "sample_inputs": sample},
        "cpu_baseline": base, "port": port,
        "e2e": {"value": base["value"], "unit": "TE/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours_multi(args, cfg):
    """N > 1: the batch-parallel runner (parallel.py) over NCCL, one rank per
    GPU: per layer the survivor counts are allgathered, transfers planned and
    executed when max/min exceeds the threshold; categories gathered at the
    end. Time = max over ranks of the CUDA-event span of K full inferences.
    Each rank generates only its own shard of the inputs, and C4's network is
    built chunk by chunk (DeviceNetwork.from_layers) on every rank."""
    import torch
    import torch.distributed as dist
    from paper_2007_14152_b200 import engine, ingest, parallel
    from paper_2007_14152_b200.model import InferenceConfig

    rank, world, local = dist_env()
    # one rank per GPU over NCCL; SPDNN_DIST_BACKEND=gloo lets several ranks
    # share one GPU (test boxes with a single device)
    backend = os.environ.get("SPDNN_DIST_BACKEND", "nccl")
    init_nccl_log()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist.init_process_group(backend, init_method="env://")
    dev = torch.device("cuda", local)
    n, total = cfg["neurons"], cfg["inputs"]
    spec = ingest.GeneratorSpec(neurons=n, layers=cfg["layers"], connections_per_neuron=K_CONN,
                                bias_value=cfg["bias"], seed=MODEL_SEED)
    bounds = parallel.shard_bounds(total, world)
    lo, hi = bounds[rank]
    m_cap = max(b - a for a, b in bounds)
    pinned = torch.empty((hi - lo, n), dtype=torch.float32).pin_memory()
    shard_batch = ingest.generate_synthetic_inputs(n, total, cfg["density"], seed=INPUT_SEED,
                                                   out=pinned.numpy().T, columns=(lo, hi))
    if cfg.get("chunked"):
        net = engine.DeviceNetwork.from_layers(ingest.iter_synthetic_layers(spec),
                                               ingest.synthetic_bias(spec), chunk=64)
        unpadded = None
    else:
        model = ingest.generate_synthetic_network(spec)
        prepared = engine.prepare_model(model, InferenceConfig(), "optimized")
        net = engine.device_network(prepared, model.bias)
        unpadded = lambda: engine.DeviceNetwork(engine._unpadded(prepared, model), model.bias)
    L = net.num_layers
    edges_per_input = int(sum(net.nnz))
    shard = parallel.DeviceShard(net, n, m_cap, L, unpadded=unpadded)
    x_dev = pinned.to(dev)
    c_dev = engine.host_tensor(np.ascontiguousarray(shard_batch.categories)).to(dev)
    transport = parallel.DistTransport(None, dev)
    thr = InferenceConfig().rebalance_threshold

    def step():
        shard.load(x_dev, c_dev)
        return parallel.run_layers_parallel(L, {rank: shard}, transport, thr, world,
                                            values=False)

    for _ in range(args.warmup):
        out = step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            out = step()
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    totals, comm, bal, parts = out
    edges = total * edges_per_input
    value = edges / (ms / 1e3) / 1e12
    sum_active = sum(b for b, _ in totals)
    bytes_total = sum(8.0 * n * b + 6.0 * nz + 4.0 * n
                      for (b, _), nz in zip(totals, net.nnz) if b) / world
    peak, peak_src = measured_peaks()
    ratios = [e.imbalance_before for e in bal.entries]
    del x_dev
    # e2e: the public API with host inputs (each rank uploads its own shard)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    res, _, _ = parallel.run_batch_parallel_device(
        net, shard_batch, InferenceConfig(workers=world), values=False,
        edges_per_input=edges_per_input, unpadded=unpadded, shard_only=True)
    torch.cuda.synchronize()
    e2e = torch.tensor([time.perf_counter() - t0], device=dev)
    dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({
            "metric": "TeraEdges/s", "value": value, "unit": "TE/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["name"], "inputs": total,
                       "input_density": cfg["density"], "survivors": int(len(res.categories)),
                       "sum_active": int(sum_active), "parallelism": f"batch-parallel x{world}",
                       "process_group": {"backend": dist.get_backend(),
                                         "world_size": dist.get_world_size()},
                       "l2": "inputs larger than L2",
                       "imbalance_max_before": max(ratios) if ratios else 1.0,
                       "rebalances": sum(e.rebalanced for e in bal.entries),
                       "rows_moved": comm.total_moved},
            "e2e": {"value": edges / float(e2e.item()) / 1e12, "unit": "TE/s",
                    "h2d_bytes_per_step": (hi - lo) * n * 4 + (hi - lo) * 8,
                    "d2h_bytes_per_step": int(len(res.categories)) * 8,
                    "path": "parallel.run_batch_parallel_device(values=False, shard_only=True)"},
            "roofline": {"bound": "hbm", "achieved": bytes_total / (ms / 1e3) / 1e9,
                         "peak": peak, "unit": "GB/s",
                         "frac": bytes_total / (ms / 1e3) / 1e9 / peak, "traffic": None,
                         "traffic_single_gpu": ncu_traffic(args.config)[0],
                         "traffic_single_gpu_source": (
                             "profiles/%s: DRAM read+write of one steady launch of the same "
                             "kernel on the whole batch (one GPU); a rank's launch moves its "
                             "shard's share" % ncu_traffic(args.config)[1]),
                         "peak_source": peak_src,
                         "note": "per-GPU algorithmic bytes over the whole step (count "
                                 "exchange, one allgather per layer window, included)"},
            "cpu_baseline": None, "clocks": clocks.summary(),
            "gpu_launches": args.steps * L}), flush=True)
    dist.destroy_process_group()


class Workload:
    """What the single-GPU timing loop needs, however the network was built."""

    def __init__(self, **kw):
        self.__dict__.update(kw)


def pinned_inputs(cfg):
    """The synthetic batch generated straight into pinned host memory: the
    e2e leg uploads from it and the device-resident copy is made once."""
    import torch
    from paper_2007_14152_b200 import ingest
    n, m = cfg["neurons"], cfg["inputs"]
    pinned = torch.empty((m, n), dtype=torch.float32).pin_memory()
    batch = ingest.generate_synthetic_inputs(n, m, cfg["density"], seed=INPUT_SEED,
                                             out=pinned.numpy().T)
    return pinned, batch


def resident_workload(args, cfg, params):
    """C1-C3: the whole model on the host, prepared once (engine.prepare_model)."""
    from paper_2007_14152_b200 import engine, ingest
    from paper_2007_14152_b200.model import InferenceConfig
    spec = ingest.GeneratorSpec(neurons=cfg["neurons"], layers=cfg["layers"],
                                connections_per_neuron=K_CONN, bias_value=cfg["bias"],
                                seed=MODEL_SEED)
    model = ingest.generate_synthetic_network(spec)
    t0 = time.time()
    prepared = engine.prepare_model(model, InferenceConfig(), "optimized", params=params)
    net = engine.device_network(prepared, model.bias)
    log(f"prepared+uploaded {model.num_layers} layers in {time.time() - t0:.1f}s "
        f"({net.hbm_bytes / 1e6:.0f} MB of layout)")

    def e2e(batch):
        return engine.infer(model, batch, InferenceConfig(), prepared=prepared, values=False)

    sample = {}

    def cpu(inputs):
        threads = os.cpu_count() or 1
        r = cpu_baseline(model, inputs, args.cpu_sample, threads, target_s=args.cpu_seconds)
        sample.update(r)
        return {"value": r["value"], "unit": "TE/s", "cores": threads, "kind": "port",
                "sample": f"first {r['sample_cols']} of {cfg['inputs']} inputs, all "
                          f"{model.num_layers} layers, oracle/spdnn_oracle.c on {threads} "
                          f"host threads ({r['seconds']:.1f} s)"}

    def parity(full_cats):
        """The timed CPU sample doubles as a full-size parity sample: the GPU
        run's survivors among the first sample_cols inputs must be exactly the
        oracle's (features never interact, so a prefix is a valid sample)."""
        if not sample:
            return None
        n_s = sample["sample_cols"]
        got = np.asarray(full_cats)[np.asarray(full_cats) < n_s]
        return {"sample_columns": int(n_s), "survivors_in_sample": int(len(sample["categories"])),
                "bit_exact": bool(np.array_equal(got, sample["categories"]))}

    def e2e_variant(batch, values):
        return engine.infer(model, batch, InferenceConfig(), prepared=prepared, values=values)

    return Workload(net=net, nnz=np.array([l.nnz for l in model.layers], np.float64),
                    e2e=e2e, e2e_path="engine.infer(values=False) on a pinned-host FeatureBatch",
                    e2e_variant=e2e_variant,
                    cpu=cpu, parity=parity, parity_after_cpu=True)


class StreamedOracle:
    """The CPU oracle run layer by layer on a fixed column sample while the
    network is generated chunk by chunk (no whole-model host copy): the C4
    CPU baseline and its full-size parity sample. Columns are split over host
    threads (the oracle's C call releases the GIL)."""

    def __init__(self, data, cols, bias, threads):
        self.y = np.asfortranarray(data[:, cols])
        self.cats = np.asarray(cols, np.int64)
        self.bias = bias
        self.threads = threads
        self.seconds = 0.0
        self.counts = [len(cols)]

    def __call__(self, l0, layers):
        from concurrent.futures import ThreadPoolExecutor
        from oracle import oracle
        t0 = time.perf_counter()
        with ThreadPoolExecutor(self.threads) as ex:
            for lay in layers:
                m = self.y.shape[1]
                if m == 0:
                    self.counts.append(0)
                    continue
                parts = np.array_split(np.arange(m), min(self.threads, m))
                outs = list(ex.map(lambda p: oracle.layer(lay, self.bias, self.y[:, p]), parts))
                out = np.concatenate([o for o, _ in outs], axis=1)
                alive = np.concatenate([a for _, a in outs])
                self.y = np.asfortranarray(out[:, alive])
                self.cats = self.cats[alive]
                self.counts.append(int(alive.sum()))
        self.seconds += time.perf_counter() - t0


def chunked_workload(args, cfg, params, batch):
    """C4 (65536 x 1920): the network is generated, planned (C++) and uploaded
    64 layers at a time; its 32 GB host CSR never exists at once. The CPU
    oracle follows the same stream on a fixed 32-column sample."""
    from paper_2007_14152_b200 import engine, ingest
    spec = ingest.GeneratorSpec(neurons=cfg["neurons"], layers=cfg["layers"],
                                connections_per_neuron=K_CONN, bias_value=cfg["bias"],
                                seed=MODEL_SEED)
    bias = ingest.synthetic_bias(spec)
    threads = os.cpu_count() or 1
    cols = np.sort(np.random.default_rng(123).choice(cfg["inputs"], 32, replace=False))
    orc = StreamedOracle(np.asarray(batch.data), cols, bias, threads) \
        if args.cpu_sample > 0 else None
    t0 = time.time()
    net = engine.DeviceNetwork.from_layers(ingest.iter_synthetic_layers(spec), bias,
                                           params=params, chunk=64, on_chunk=orc)
    log(f"generated+prepared+uploaded {net.num_layers} layers in {time.time() - t0:.1f}s "
        f"({net.hbm_bytes / 1e9:.1f} GB of layout)"
        + (f"; oracle sample {orc.seconds:.1f}s" if orc else ""))

    def e2e(b):
        return engine.infer_device(net, b, values=False)

    def cpu(inputs):
        if orc is None:
            return None
        edges = len(cols) * float(np.sum(net.nnz))
        return {"value": edges / orc.seconds / 1e12, "unit": "TE/s", "cores": threads,
                "kind": "port",
                "sample": f"{len(cols)} fixed-seed columns of {cfg['inputs']} through all "
                          f"{net.num_layers} layers, layer-streamed oracle/spdnn_oracle.c on "
                          f"{threads} host threads ({orc.seconds:.1f} s)"}

    def parity(full_cats):
        """Full-size sampled parity: the GPU on the sample columns alone vs the
        oracle, bit for bit; and the full run's survivors within the sample."""
        if orc is None:
            return None
        from paper_2007_14152_b200.model import make_feature_batch
        sub = make_feature_batch(cfg["neurons"], np.asfortranarray(np.asarray(batch.data)[:, cols]),
                                 categories=cols, total_inputs=cfg["inputs"])
        got = engine.infer_device(net, sub, values=True)
        ok = (got.categories.tolist() == orc.cats.tolist()
              and np.array_equal(np.asarray(got.final.data).view(np.uint32),
                                 orc.y.view(np.uint32))
              and np.intersect1d(full_cats, cols).tolist() == orc.cats.tolist()
              and [o.active_before for o in got.per_layer] + [len(got.categories)]
              == orc.counts)
        return {"sample_columns": len(cols), "survivors_in_sample": len(orc.cats),
                "bit_exact": bool(ok)}

    return Workload(net=net, nnz=np.asarray(net.nnz, np.float64), e2e=e2e, parity_after_cpu=False,
                    e2e_path="engine.infer_device(values=False) on a pinned-host FeatureBatch "
                             "(network resident, built by DeviceNetwork.from_layers)",
                    cpu=cpu, parity=parity)


def run_ours(args, cfg):
    import torch
    from paper_2007_14152_b200 import _native, engine

    rank, world, local = dist_env()
    if cfg.get("stress"):
        return run_stress(args, cfg)
    # SPDNN_BENCH_PARALLEL=1 times the batch-parallel runner even at N=1
    # (its per-window overhead against the single-worker engine)
    if world > 1 or os.environ.get("SPDNN_BENCH_PARALLEL") == "1":
        return run_ours_multi(args, cfg)
    dev = torch.device("cuda", torch.cuda.current_device())
    t0 = time.time()
    pinned, batch = pinned_inputs(cfg)
    n, m = cfg["neurons"], cfg["inputs"]
    log(f"inputs generated in {time.time() - t0:.1f}s")
    params = engine.PlanParams(**{k: int(v) for k, v in
                                  (kv.split("=") for kv in args.plan.split(",") if kv)})
    W = chunked_workload(args, cfg, params, batch) if cfg.get("chunked") else \
        resident_workload(args, cfg, params)
    net = W.net
    L = net.num_layers
    ws = engine.workspace(n, m, L)
    x_dev = pinned.to(dev)
    cats_dev = engine.host_tensor(np.ascontiguousarray(batch.categories)).to(dev)
    stream = torch.cuda.current_stream()
    opts = engine.run_opts(net)

    import ctypes
    lib = _native.lib()
    sp = ctypes.c_void_p(stream.cuda_stream)

    def step(evs=None):
        engine.stage_inputs(ws, x_dev, cats_dev, net)
        if evs is None:
            return engine.run_layers(net, ws, m)
        engine.reset_run(ws, m)
        # the whole layer loop in one C call (spdnn_infer_layers_timed), an
        # event recorded before every layer: launches are not paced by Python
        handles = evs
        _native.check(lib.spdnn_infer_layers_timed(
            L, net.layer_devs, engine._dptr(net.bias), engine._dptr(ws.y[0]),
            engine._dptr(ws.y[1]), ws.ld, engine._dptr(ws.a[0]), engine._dptr(ws.a[1]),
            engine._dptr(ws.cat[0]), engine._dptr(ws.cat[1]), engine._dptr(ws.counts),
            ctypes.byref(ws.scratch), ctypes.byref(opts), sp, handles),
            "spdnn_infer_layers_timed")
        return engine.DeviceRun(ws, L, m)

    # correctness of the timed configuration: categories after one step
    run0 = step()
    counts_chk, cats_chk, _ = engine.collect(run0, want_values=False)
    assert run0.guard == 0, "FMA-form guard tripped on the bench workload"
    log(f"arithmetic form: {'fma' if run0.fma else 'exact'}; survivors {int(counts_chk[-1])}")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region (device): K steps, the layer loop as the engine runs it
    # (one C call; consecutive layers overlap through programmatic dependent
    # launch, which an event between two layers would defeat)
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clocks:
        torch.cuda.synchronize()
        e_start.record()
        for k in range(args.steps):
            step()
        e_end.record()
        torch.cuda.synchronize()
    ms_total = e_start.elapsed_time(e_end)
    counts = ws.counts[: L + 1].cpu().numpy().astype(np.int64)

    # ---- per-launch kernel times (roofline), from separate steps with an
    # event before every layer (spdnn_infer_layers_timed)
    prof_steps = max(1, min(args.steps, 3))
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(L + 1)] for _ in range(prof_steps)]
    for row in evs:  # create the CUDA events before use
        for e in row:
            e.record()
    torch.cuda.synchronize()
    ev_handles = [(ctypes.c_void_p * (L + 1))(*[e.cuda_event for e in row]) for row in evs]
    for k in range(prof_steps):
        step(ev_handles[k])
    torch.cuda.synchronize()
    layer_ms = np.array([[evs[k][l].elapsed_time(evs[k][l + 1]) for l in range(L)]
                         for k in range(prof_steps)])
    if args.dump_layers:
        with open(args.dump_layers, "w") as f:
            json.dump({"counts": counts.tolist(), "layer_ms": layer_ms.mean(axis=0).tolist()}, f)
    ms_step = ms_total / args.steps
    edges_step = cfg["inputs"] * float(W.nnz.sum())  # credited: every input, every layer
    value = edges_step / (ms_step / 1e3) / 1e12

    # ---- roofline of the layer kernel: algorithmic bytes / CUDA-event time
    bytes_l = 8.0 * n * counts[:L] + 6.0 * W.nnz + 4.0 * n
    active = counts[:L] > 0
    achieved = float(bytes_l[active].sum() / (layer_ms.mean(axis=0)[active].sum() / 1e3) / 1e9)
    peak, peak_src = measured_peaks()
    kernel_share = float(layer_ms.mean(axis=0).sum() / (ms_total / args.steps))
    traffic, traffic_src, traffic_layer = ncu_traffic(args.config)
    del x_dev
    torch.cuda.empty_cache()

    # ---- end to end through the public API: pinned host inputs -> categories
    e2e_steps = max(1, min(args.steps, 5))
    res = W.e2e(batch)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        res = W.e2e(batch)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    assert np.array_equal(res.categories, cats_chk.cpu().numpy()), "e2e categories differ"
    h2d = m * n * 4 + m * 8
    d2h = len(res.categories) * 8 + (L + 1) * 4
    # the same call as a reference caller makes it: a pageable numpy batch,
    # and with the final values copied back (engine.infer's default)
    variants = None
    if getattr(W, "e2e_variant", None) is not None:
        from paper_2007_14152_b200.model import make_feature_batch
        pageable = make_feature_batch(n, np.array(batch.data, order="F"), batch.categories)
        variants = {}
        for key, b_, vals in (("pageable_values_false", pageable, False),
                              ("pinned_values_true", batch, True)):
            r_ = W.e2e_variant(b_, vals)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r_ = W.e2e_variant(b_, vals)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            assert np.array_equal(r_.categories, res.categories), key
            variants[key] = {"value": edges_step / dt / 1e12, "unit": "TE/s",
                             "ms_per_step": dt * 1e3,
                             "d2h_bytes_per_step": d2h + (len(r_.categories) * n * 4
                                                          if vals else 0)}
        del pageable
    parity = W.parity(res.categories) if W.parity and not W.parity_after_cpu else None
    cpu = W.cpu(batch) if args.cpu_sample > 0 else None
    if W.parity and W.parity_after_cpu:
        parity = W.parity(res.categories)
    if parity is not None:
        log(f"full-size sampled parity: {parity}")
        assert parity["bit_exact"], "GPU differs from the oracle on the sampled columns"
    line = {
        "metric": "TeraEdges/s", "value": value, "unit": "TE/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["name"], "inputs": cfg["inputs"],
                   "input_density": cfg["density"], "connections": K_CONN,
                   "survivors": int(counts[L]), "sum_active": int(counts[:L].sum()),
                   "l2": "inputs larger than L2 (Y = %.0f MB per buffer vs 126 MB)"
                         % (n * ws.ld * 4 / 1e6),
                   "parallelism": "single",
                   "arithmetic": "fma form (weights 2^-4, guard clean)" if opts.fma_form
                                 else "exact form",
                   "plan": dataclasses.asdict(params),
                   "layout_hbm_gb": round(net.hbm_bytes / 1e9, 2)},
        "e2e": {"value": edges_step / e2e_s / 1e12, "unit": "TE/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_s * 1e3, "path": W.e2e_path,
                "variants": variants},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": (f"profiles/{traffic_src}: dram read+write of one "
                                        f"steady-state launch (layer {traffic_layer}, ncu "
                                        "--set full); that launch's algorithmic bytes: "
                                        f"{float(bytes_l[traffic_layer]):.4g}")
                                       if traffic and traffic_layer is not None
                                       and traffic_layer < L else None,
                     "peak_source": peak_src,
                     "kernel": "layer_kernel (csrc/layer.cu)",
                     "bytes_per_launch": "8*N*M_l + 6*nnz_l + 4*N",
                     "kernel_share_of_step": kernel_share,
                     "active_edge_rate_T": float(counts[:L].sum() * K_CONN * n /
                                                 (ms_step / 1e3) / 1e12)},
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        "gpu_launches": args.steps * (L + 1),
    }
    if parity is not None:
        line["parity"] = parity
    print(json.dumps(line), flush=True)
    return line


def stress_inputs(cfg):
    """C5: 8 contiguous shards of 7500 inputs, shard s drawn
    at density |b| + 0.04 - 0.01 s with seed 100 + s -- the same recipe as
    tests/golden/make_stress.py, here on config 3's network."""
    from paper_2007_14152_b200 import ingest
    from paper_2007_14152_b200.model import make_feature_batch
    n, w, per = cfg["neurons"], cfg["workers"], cfg["inputs"] // cfg["workers"]
    parts = [np.asarray(ingest.generate_synthetic_inputs(
        n, per, abs(cfg["bias"]) + 0.04 - 0.01 * s, seed=100 + s).data) for s in range(w)]
    return make_feature_batch(n, np.concatenate(parts, axis=1))


def balance_summary(bal, shard_sizes):
    """Per-layer work model of the 8-GPU run: layer l+1's time on worker w is
    proportional to the features it holds after layer l's (re)balancing, and
    every layer ends at the slowest worker (the count exchange is a barrier).
    time-weighted max/mean = sum_l max_w / sum_l mean_w (1.0 = perfect)."""
    inputs = [list(shard_sizes)] + [list(e.after_counts) for e in bal.entries[:-1]]
    mx = sum(max(c) for c in inputs)
    mean = sum(sum(c) / len(c) for c in inputs)
    ratios = [e.imbalance_before for e in bal.entries if np.isfinite(e.imbalance_before)]
    return {"time_weighted_max_over_mean": mx / mean if mean else 1.0,
            "max_imbalance_before": max(ratios) if ratios else 1.0,
            "max_imbalance_after": max((e.imbalance_after for e in bal.entries
                                        if np.isfinite(e.imbalance_after)), default=1.0),
            "rebalances": int(sum(e.rebalanced for e in bal.entries)),
            "rows_moved": int(bal.total_moved)}


def run_stress(args, cfg):
    """C5: skewed shards, rebalancing on (threshold 1.25) vs off (inf).
    N = 1: the 8 workers share this GPU (parallel.run_batch_parallel's
    in-process transport), so the device time is the SUM over workers and the
    8-GPU effect is reported through the count-based work model
    (balance_summary). N = 8 under torchrun: one worker per GPU over NCCL,
    timed as the max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2007_14152_b200 import engine, ingest, parallel
    from paper_2007_14152_b200.model import InferenceConfig, count_edges

    rank, world, local = dist_env()
    if world > 1:
        init_nccl_log()
        torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
        dist.init_process_group(os.environ.get("SPDNN_DIST_BACKEND", "nccl"),
                                init_method="env://")
        if world != cfg["workers"]:
            log(f"C5 is defined for {cfg['workers']} workers; running with {world}")
    workers = world if world > 1 else cfg["workers"]
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=cfg["neurons"], layers=cfg["layers"], connections_per_neuron=K_CONN,
        bias_value=cfg["bias"], seed=MODEL_SEED))
    inputs = stress_inputs(dict(cfg, workers=workers))
    prepared = engine.prepare_model(model, InferenceConfig(), "optimized")
    edges = inputs.total_inputs * count_edges(model)
    bounds = parallel.shard_bounds(inputs.active_count, workers)
    sizes = [hi - lo for lo, hi in bounds]
    out = {}
    for tag, thr in (("on", 1.25), ("off", float("inf"))):
        conf = InferenceConfig(workers=workers, rebalance_threshold=thr)
        for _ in range(max(1, args.warmup)):
            res, comm, bal = parallel.run_batch_parallel(model, inputs, conf,
                                                         prepared=prepared, values=False)
        times = []
        with ClockSampler(torch.cuda.current_device()) as clocks:
            for _ in range(args.steps):
                if world > 1:
                    dist.barrier()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                res, comm, bal = parallel.run_batch_parallel(model, inputs, conf,
                                                             prepared=prepared, values=False)
                e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1)
                if world > 1:
                    tt = torch.tensor([t], device="cuda")
                    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                    t = float(tt.item())
                times.append(t)
        ms = float(np.median(times))
        out[tag] = dict(balance_summary(bal, sizes), ms_per_step=ms,
                        value=edges / (ms / 1e3) / 1e12, survivors=len(res.categories),
                        clocks=clocks.summary(), categories=res.categories)
    same = np.array_equal(out["on"].pop("categories"), out["off"].pop("categories"))
    if rank == 0:
        on, off = out["on"], out["off"]
        line = {
            "metric": "TeraEdges/s", "value": on["value"], "unit": "TE/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": on["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["name"], "inputs": inputs.total_inputs,
                       "workers": workers,
                       "shards": f"{workers} x {sizes[0]}, density |b|+0.04-0.01*s, seed 100+s",
                       "transport": "NCCL, one worker per GPU" if world > 1 else
                                    "in-process: all workers on this GPU (time = sum)",
                       "categories_identical_on_off": bool(same)},
            "rebalancing_on": on, "rebalancing_off": off,
            "modelled_8gpu_speedup_from_rebalancing":
                off["time_weighted_max_over_mean"] / on["time_weighted_max_over_mean"],
            "clocks": on["clocks"], "gpu_launches": None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def relaunch_command(argv, gpus: int, port: int | None = None):
    """`--gpus N` without a torchrun environment: the same command under
    torch.distributed.run with N local ranks (one per GPU), rendezvous on
    127.0.0.1. Returns None when no relaunch is needed."""
    if gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if port is None:
        import socket
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
            os.path.abspath(__file__)] + list(argv)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dump-layers", default="", help="write per-layer counts/times (JSON)")
    ap.add_argument("--plan", default="", help="layout knobs, e.g. max_groups=8,footprint_cap=96")
    ap.add_argument("--cpu-sample", type=int, default=1024,
                    help="inputs in the CPU-baseline sample (0 = skip the CPU leg)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="grow the CPU sample to about this much CPU time (0 = fixed sample)")
    ap.add_argument("--port-only", action="store_true",
                    help="reference arm: time only the C port, not baseline/_ref's spdnn")
    ap.add_argument("--inputs", type=int, default=0,
                    help="override the batch size (diagnostics: e.g. one rank's share at N=8)")
    args = ap.parse_args()
    cmd = relaunch_command(sys.argv[1:], args.gpus)
    if cmd is not None:
        # one process per GPU; rank 0 prints the single JSON line
        log("relaunching: " + " ".join(cmd))
        sys.exit(subprocess.call(cmd))
    rank, world, _ = dist_env()
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE")
    if args.warmup < 3 and args.impl == "ours":
        log("warning: fewer than 3 warm-up steps")
    cfg = CONFIGS[args.config]
    if args.inputs > 0:
        cfg = dict(cfg, inputs=args.inputs,
                   name=cfg["name"] + f" [diagnostic: {args.inputs} inputs]")
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
