"""Write a degree-sorted relabelled CSR of a DC-SBM config to binary files for layer_lab (tooling).

    python tools/lab/prep_csr.py headline /tmp/lab      -> /tmp/lab.rp (int32[N+1]), /tmp/lab.ci (int32[nnz])
Optional 3rd arg 'planted': order rows by planted block (degree-descending within) instead.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from synth.dcsbm import CONFIGS, generate  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
prefix = sys.argv[2]
order_kind = sys.argv[3] if len(sys.argv) > 3 else "degree"
edges, labels = generate(cfg)
n = cfg.num_nodes
u, v = edges[:, 0].astype(np.int64), edges[:, 1].astype(np.int64)
keep = u != v
u, v = u[keep], v[keep]
a, b = np.minimum(u, v), np.maximum(u, v)
key = np.unique(a * n + b)
a, b = key // n, key % n
rows = np.concatenate([a, b])
cols = np.concatenate([b, a])
deg = np.bincount(rows, minlength=n)
if order_kind == "planted":
    order = np.lexsort((np.arange(n), -deg, labels))
else:
    order = np.lexsort((np.arange(n), -deg))
inv = np.empty(n, np.int64)
inv[order] = np.arange(n)
r2, c2 = inv[rows], inv[cols]
o = np.lexsort((c2, r2))
r2, c2 = r2[o], c2[o]
rp = np.zeros(n + 1, np.int64)
np.cumsum(np.bincount(r2, minlength=n), out=rp[1:])
rp.astype(np.int32).tofile(prefix + ".rp")
c2.astype(np.int32).tofile(prefix + ".ci")
print(f"N={n} nnz={c2.size} written to {prefix}.rp/.ci")
