"""Parity of the GPU path vs the fp64 oracle at the paper's own (tau, L, d) settings (Table II),
layer by layer (tooling: decides which settings the tests can gate at 1e-4)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2508_19737_b200 as igp  # noqa: E402
from synth.dcsbm import PAPER_CONFIGS, generate  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["paper_5k", "paper_10k", "paper_50k", "paper_100k"]
nt = len(os.sched_getaffinity(0))
for name in names:
    c = PAPER_CONFIGS[name]
    edges, _ = generate(c)
    e = torch.from_numpy(edges).cuda()
    g = igp.build_graph(e, c.num_nodes)
    rp, ci, _ = oracle.build_csr(edges, c.num_nodes)
    Ls = sorted({1, 2, 3, 5, 10, c.steps} & set(range(1, c.steps + 1)))
    for L in Ls:
        z = igp.embed(g, c.tau, c.d, L, 0).cpu().numpy().astype(np.float64)
        ref = oracle.embed(rp, ci, c.num_nodes, c.d, L, c.tau, seed=0, nthreads=nt)
        err = float(np.max(np.abs(z - ref) / np.linalg.norm(ref, axis=1, keepdims=True)))
        print(f"{name} tau={c.tau} d={c.d} L={L:3d}: row-rel err {err:.3e}", flush=True)
    g.close()
