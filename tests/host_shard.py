"""CPU shard for exercising the batch-parallel orchestration without a GPU
(test infrastructure: the layer step is the oracle). Implements the
interface parallel.run_layers_parallel drives: .m, .n, take_top, append, final."""

import numpy as np
import torch

from oracle import oracle


class HostShard:
    def __init__(self, model, x_cols, cats):
        self.model = model
        self.n = model.neurons
        self.x = np.asfortranarray(x_cols, dtype=np.float32)  # (N, m)
        self.cats = np.asarray(cats, dtype=np.int64)
        self.m = self.x.shape[1]

    def step(self, l):
        if self.m:
            out, alive = oracle.layer(self.model.layers[l], self.model.bias, self.x)
            self.x = np.asfortranarray(out[:, alive])
            self.cats = self.cats[alive]
        self.m = self.x.shape[1]
        return self.m

    def take_top(self, k):
        order = np.argsort(self.cats, kind="stable")
        top = order[self.m - k:]
        keep = np.sort(order[: self.m - k])
        vals = torch.from_numpy(np.ascontiguousarray(self.x[:, top].T))
        cats = torch.from_numpy(self.cats[top].copy())
        self.x = np.asfortranarray(self.x[:, keep])
        self.cats = self.cats[keep]
        self.m -= k
        return vals, cats

    def append(self, vals, cats):
        self.x = np.asfortranarray(np.concatenate([self.x, vals.numpy().T], axis=1))
        self.cats = np.concatenate([self.cats, cats.numpy()])
        self.m = self.x.shape[1]

    def final(self, values=True):
        return (torch.from_numpy(self.cats.copy()),
                torch.from_numpy(np.ascontiguousarray(self.x.T)) if values else None)
