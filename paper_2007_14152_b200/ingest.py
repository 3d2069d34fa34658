"""Synthetic Graph-Challenge-style networks and inputs (host data preparation).

This is the boundary data source, not the accelerated path: the bench and the
parity tests need the *same* networks and inputs the reference builds, bit for
bit, on a box where the reference itself is absent. The draw sequence follows
``spdnn/ingest.py:140-180``:

* per layer: ``offset = rng.integers(1, N)``, then a stride redrawn with
  ``rng.integers(1, N)`` until ``gcd(stride, N) == 1``; row ``r`` connects to
  ``{(r*offset + i*stride) mod N : i < K}`` (sorted), every weight 1/16, one
  constant bias;
* inputs: ``rng.random((N, M)) < density`` in row-major draw order.

Inputs are produced in row chunks so the 65536 x 60000 case never builds the
31 GB float64 temporary; the chunked stream equals the one-shot stream
(PCG64 ``random`` fills row-major).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .model import FeatureBatch, LayerCSR, ModelError, NetworkModel

WEIGHT_VALUE = np.float32(0.0625)


@dataclass(frozen=True)
class GeneratorSpec:
    """Synthetic fixed-fan-in network parameters (``spdnn/ingest.py:37-53``)."""

    neurons: int
    layers: int
    connections_per_neuron: int = 32
    bias_value: float = -0.3
    seed: int = 0
    input_count: int = 0
    input_density: float = 0.3

    def __post_init__(self):
        if self.connections_per_neuron > self.neurons:
            raise ModelError("connections_per_neuron cannot exceed neurons")
        if not 0.0 < self.input_density <= 1.0:
            raise ModelError("input_density must be in (0, 1]")


def layer_parameters(neurons: int, layers: int, seed: int) -> list[tuple[int, int]]:
    """(offset, stride) per layer, drawn exactly as the reference draws them."""
    rng = np.random.default_rng(seed)
    params = []
    for _ in range(layers):
        offset = int(rng.integers(1, neurons)) if neurons > 1 else 0
        stride = 1
        if neurons > 1:
            while True:
                stride = int(rng.integers(1, neurons))
                if math.gcd(stride, neurons) == 1:
                    break
        params.append((offset, stride))
    return params


def synthetic_layer(neurons: int, k: int, offset: int, stride: int) -> LayerCSR:
    """Row r -> sorted {(r*offset + i*stride) mod N}, all weights 1/16."""
    base = (np.arange(neurons, dtype=np.int64) * offset) % neurons
    cols = (base[:, None] + (np.arange(k, dtype=np.int64) * stride)[None, :]) % neurons
    cols.sort(axis=1)
    return LayerCSR(row_ptr=np.arange(0, neurons * k + 1, k, dtype=np.int64),
                    col_idx=cols.reshape(-1).astype(np.int32),
                    values=np.full(neurons * k, WEIGHT_VALUE, dtype=np.float32))


def generate_synthetic_network(spec: GeneratorSpec) -> NetworkModel:
    n, k = spec.neurons, spec.connections_per_neuron
    layers = tuple(synthetic_layer(n, k, off, st)
                   for off, st in layer_parameters(n, spec.layers, spec.seed))
    return NetworkModel(neurons=n, layers=layers,
                        bias=np.full(n, np.float32(spec.bias_value), dtype=np.float32))


def generate_synthetic_inputs(neurons: int, count: int, density: float, seed: int,
                              chunk_rows: int = 1024) -> FeatureBatch:
    """Bernoulli(density) binary features, (N, M) Fortran fp32, categories 0..M-1."""
    rng = np.random.default_rng(seed)
    data = np.empty((neurons, count), dtype=np.float32, order="F")
    thr = float(density)
    for r0 in range(0, neurons, chunk_rows):
        r1 = min(neurons, r0 + chunk_rows)
        data[r0:r1, :] = rng.random((r1 - r0, count)) < thr
    return FeatureBatch(neurons=neurons, data=data,
                        categories=np.arange(count, dtype=np.int64), total_inputs=count)
