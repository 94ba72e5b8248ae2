"""Seeded layer states Z (float32 [N, d]) for layer-by-layer checks (igp_embed_opts.d_z0 on the
CUDA side, oracle.embed(..., Z0=...) on the oracle side).  Holds none of the method's
arithmetic: plain random matrices shaped like the states a layer consumes."""
from __future__ import annotations

import numpy as np


def layer_state(n: int, d: int, seed: int, kind: str = "normal") -> np.ndarray:
    """'normal': i.i.d. N(0, 1) (a generic standardised column); 'bimodal': values near +-1 with
    small jitter (the shape of columns after saturated tanh units, e.g. at tau = -80)."""
    rng = np.random.default_rng(seed)
    if kind == "normal":
        z = rng.standard_normal((n, d))
    elif kind == "bimodal":
        z = np.where(rng.random((n, d)) < 0.5, -1.0, 1.0) + 0.05 * rng.standard_normal((n, d))
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(z, dtype=np.float32)
