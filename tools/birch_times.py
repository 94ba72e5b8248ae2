"""BIRCH (igp_birch_*) device times on a config's GPU embedding (tooling).

    python tools/birch_times.py headline [T1,T2,...] [--oracle-rows R]
For each threshold: fit (igp_birch_partial_fit, host-timed: synchronous call), predict on both paths
(tensor cores, certified, and all-fp64; CUDA events; labels must agree),
K / depth / nodes, us per inserted row; the oracle's fit + predict on the first R rows (one thread).
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402
from ncu_embed import cached_edges  # noqa: E402
from synth.dcsbm import ALL_CONFIGS  # noqa: E402

argv = sys.argv[1:]
orows = 0
if "--oracle-rows" in argv:
    k = argv.index("--oracle-rows")
    orows = int(argv[k + 1])
    del argv[k:k + 2]
cfg = ALL_CONFIGS[argv[0] if argv else "headline"]
thresholds = [float(x) for x in (argv[1].split(",") if len(argv) > 1 else ["1.0"])]
e = torch.from_numpy(cached_edges(cfg)).cuda()
g = igp.build_graph(e, cfg.num_nodes)
Z = igp.embed(g, cfg.tau, cfg.d, cfg.steps, cfg.seed)
torch.cuda.synchronize()
for T in thresholds:
    b = igp.Birch(cfg.d, T, 50)
    t0 = time.perf_counter()
    b.partial_fit(Z)
    fit = time.perf_counter() - t0
    pt = {}
    for path in ("tensor", "fp64"):
        b.predict(Z, path=path)  # warm
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record()
        lab = b.predict(Z, path=path)
        p1.record()
        torch.cuda.synchronize()
        pt[path] = (p0.elapsed_time(p1), lab)
    _, amb = b.predict(Z, path="tensor", return_ambiguous=True)
    assert torch.equal(pt["tensor"][1], pt["fp64"][1])
    K, dep, nodes, pts = b.info()
    line = (f"{cfg.name} T={T}: K={K} depth={dep} nodes={nodes}  fit {fit * 1e3:9.1f} ms "
            f"({fit / pts * 1e6:.2f} us/row)  predict tensor {pt['tensor'][0]:8.2f} ms ({amb} rows to fp64) "
            f"fp64 {pt['fp64'][0]:8.2f} ms")
    if orows:
        import oracle
        X = Z[:orows].cpu().numpy().astype(np.float64)
        t0 = time.perf_counter()
        ob = oracle.Birch(cfg.d, T, 50).fit(X)
        ob.predict(X)
        ot = time.perf_counter() - t0
        line += f"  | oracle (1 thread) fit+predict {orows} rows: {ot:.2f} s ({ot / orows * 1e6:.1f} us/row)"
    print(line, flush=True)
    b.close()
