"""Full-L parity of one config against the fp64 oracle (tooling: a one-off evidence run for sizes
whose full oracle is too slow for the test suite, e.g. Large: 60 layers x ~35 s on 16 cores).

    python tools/full_parity.py large [L] > gpurun_out/full_parity_large.json
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: this is a parity check)
import paper_2508_19737_b200 as igp  # noqa: E402
from synth.dcsbm import ALL_CONFIGS, generate  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
c = ALL_CONFIGS[name]
L = int(sys.argv[2]) if len(sys.argv) > 2 else c.steps
edges, _ = generate(c)
e = torch.from_numpy(edges).cuda()
g = igp.build_graph(e, c.num_nodes)
t0 = time.time()
z = igp.embed(g, c.tau, c.d, L, c.seed).cpu().numpy().astype(np.float64)
gpu_s = time.time() - t0
rp, ci, _ = oracle.build_csr(edges, c.num_nodes)
nt = len(os.sched_getaffinity(0))
t0 = time.time()
ref = oracle.embed(rp, ci, c.num_nodes, c.d, L, c.tau, seed=c.seed, nthreads=nt)
oracle_s = time.time() - t0
nrm = np.linalg.norm(ref, axis=1, keepdims=True)
err = float(np.max(np.abs(z - ref) / np.where(nrm > 0, nrm, 1.0)))
print(json.dumps({"config": name, "N": c.num_nodes, "nnz": int(ci.size), "d": c.d, "L": L, "tau": c.tau,
                  "row_rel_err": err, "bar": 1e-4, "pass": err <= 1e-4, "oracle_seconds": oracle_s,
                  "oracle_threads": nt}))
