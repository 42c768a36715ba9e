"""CPU stand-in for the per-phase kernels of the partitioned solve (TEST
INFRASTRUCTURE): same contract as paper_1912_01478_b200.distributed.DeviceOps
on the same state-word encoding, so the distributed driver's partition /
exchange / termination logic is exercised under gloo without a GPU."""

import numpy as np
import torch

FBIT = 0x80000000
CMASK = 0x7FFFFFFF


class CpuOps:
    def __init__(self, ro, ci, n):
        self.ro = np.asarray(ro, dtype=np.int64)
        self.ci = np.asarray(ci, dtype=np.int64)
        self.n = n

    def new_state(self):
        return torch.zeros(max(self.n, 1), dtype=torch.int32)

    def buffers(self, lo, hi):
        self.nxt = [None, None]

    def boundary(self, lo, hi):
        f = np.zeros(max(hi - lo, 1), dtype=np.uint8)
        for u in range(lo, hi):
            nb = self.ci[self.ro[u]:self.ro[u + 1]]
            f[u - lo] = bool(((nb < lo) | (nb >= hi)).any())
        return torch.from_numpy(f)

    def _nodes(self, X, items, count, lo):
        x = X.numpy().view(np.uint32)
        if items is None:
            return [u for u in range(lo, lo + count) if not (x[u] & FBIT)]
        return items[:count].tolist()

    def assign(self, X, items, count, lo, boundary):
        x = X.numpy().view(np.uint32)
        ids, vals = [], []
        for u in self._nodes(X, items, count, lo):
            taken = {int(x[v]) & CMASK for v in self.ci[self.ro[u]:self.ro[u + 1]] if x[v] & FBIT}
            t = 1
            while t in taken:
                t += 1
            x[u] = t
            if boundary[u - lo]:
                ids.append(u)
                vals.append(t)
        return (torch.tensor(ids, dtype=torch.int32), torch.tensor(vals, dtype=torch.int64).to(torch.int32),
                len(ids))

    def resolve(self, X, items, count, lo, boundary, out_slot):
        x = X.numpy().view(np.uint32)
        nxt, ids, vals, conf = [], [], [], 0
        for u in self._nodes(X, items, count, lo):
            tu = int(x[u])
            k = sum(1 for v in self.ci[self.ro[u]:self.ro[u + 1]] if v < u and (int(x[v]) & CMASK) == tu)
            conf += k
            if k:
                nxt.append(u)
            else:
                x[u] = tu | FBIT
                if boundary[u - lo]:
                    ids.append(u)
                    vals.append(tu | FBIT)
        nt = torch.tensor(nxt, dtype=torch.int32)
        return (nt, len(nxt), torch.tensor(ids, dtype=torch.int32),
                torch.tensor(vals, dtype=torch.int64).to(torch.int32), len(ids), conf)

    def apply(self, X, ids, vals):
        x = X.numpy().view(np.uint32)
        for u, v in zip(ids.tolist(), vals.tolist()):
            x[u] = v & 0xFFFFFFFF

    def colors(self, X, lo, hi):
        x = X.numpy().view(np.uint32)
        return torch.from_numpy((x[lo:hi] & CMASK).astype(np.int64))
