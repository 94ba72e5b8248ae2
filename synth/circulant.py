"""Circulant graphs C_n(1..k) for checks at the maximum CSR size: node i is joined to
i+1, ..., i+k (mod n).  Every node has degree 2k and row i of the canonical CSR is known in
closed form, so the builder can be checked without a CPU CSR of ~2^31 entries.  Holds none of
the method's arithmetic (input synthesis only)."""
from __future__ import annotations

import numpy as np


def circulant_edges(n: int, k: int, device="cpu"):
    """int32 [n*k, 2] edge list (u, (u + o) mod n), o = 1..k, as a torch tensor on ``device``
    (generated there: at n*k ~ 2^30 the list is 8.6 GB).  Requires 2k < n (no duplicates)."""
    import torch

    if not 0 < 2 * k < n or n >= 2**31 - k:
        raise ValueError("need 0 < 2k < n < 2^31 - k")
    e = torch.empty((n, k, 2), dtype=torch.int32, device=device)
    i = torch.arange(n, dtype=torch.int32, device=device)
    e[:, :, 0] = i[:, None]
    for o in range(1, k + 1):
        v = i + o
        v[n - o:] -= n
        e[:, o - 1, 1] = v
    return e.view(n * k, 2)


def circulant_row(n: int, k: int, i: int) -> np.ndarray:
    """The canonical (sorted) neighbour list of node i."""
    return np.array(sorted({(i + o) % n for o in range(-k, k + 1) if o != 0}), dtype=np.int32)
