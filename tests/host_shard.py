"""CPU shard for exercising the batch-parallel orchestration without a GPU
(test infrastructure: the layer step is the oracle). Implements the
interface parallel.run_layers_parallel drives: .m, .n, begin_window,
window_counts, rewind, replay, commit, set_exact, take_top, append, final."""

import numpy as np
import torch

from oracle import oracle


class HostShard:
    uses_fma = False
    unpadded_active = True

    def __init__(self, model, x_cols, cats):
        self.model = model
        self.n = model.neurons
        self.x = np.asfortranarray(x_cols, dtype=np.float32)  # (N, m)
        self.cats = np.asarray(cats, dtype=np.int64)
        self.m = self.x.shape[1]
        self.windows = []  # (l0, k) of every window run, for the tests

    def _step(self, l):
        if self.m:
            out, alive = oracle.layer(self.model.layers[l], self.model.bias, self.x)
            self.x = np.asfortranarray(out[:, alive])
            self.cats = self.cats[alive]
        self.m = self.x.shape[1]
        return self.m

    def begin_window(self, l0, k):
        self._ck = (self.x, self.cats, self.m)
        self._l0 = l0
        self.windows.append((l0, k))
        self._counts = [self._step(l0 + j) for j in range(k)]

    def window_counts(self):
        return torch.tensor(self._counts + [0], dtype=torch.int64)

    def rewind(self):
        self.x, self.cats, self.m = self._ck

    def replay(self, k):
        self.rewind()
        self._counts = [self._step(self._l0 + j) for j in range(k)]

    def commit(self, m_last_in, m):
        assert m == self.m

    def set_exact(self, unpadded):
        pass

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
