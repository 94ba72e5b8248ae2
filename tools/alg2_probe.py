"""Alg. 2 BIRCH steps on the streaming config, each library call host-timed with a sync (tooling).

    python tools/alg2_probe.py [stages]
Per stage: merge + embed, row extraction, partial_fit, info (cluster-list refresh), predict twice
(first = after the fit, second = warm), with the uncertified row count.
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402
from synth.dcsbm import ALL_CONFIGS, generate, stream_batches  # noqa: E402

stages = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = ALL_CONFIGS["streaming"]
edges, _ = generate(cfg)
dev = torch.device("cuda", 0)
batches = [torch.from_numpy(b).to(dev) for b in stream_batches(edges, 10)]
N, d = cfg.num_nodes, cfg.d
out = torch.empty((N, d), dtype=torch.float32, device=dev)
kept = torch.empty((N, d), dtype=torch.float32, device=dev)
seen = torch.zeros(N, dtype=torch.bool, device=dev)
bt = igp.Birch(d, 1.0, 50)
g = igp.build_graph(batches[0], N)
n_kept = 0


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


for t in range(stages):
    if t > 0:
        g.add_edges(batches[t])
    igp.embed(g, cfg.tau, d, cfg.steps, cfg.seed, out=out, subsequence=t)
    _, _, deg = g.csr(degrees=True)
    new = torch.nonzero((deg > 0) & ~seen).flatten()
    seen[new] = True
    kept[n_kept:n_kept + new.numel()] = out[new]
    _, fit_ms = timed(lambda: bt.partial_fit(kept[n_kept:n_kept + new.numel()]))
    n_kept += new.numel()
    info, info_ms = timed(lambda: bt.info())
    (lab, amb), p1 = timed(lambda: bt.predict(kept[:n_kept], return_ambiguous=True))
    _, p2 = timed(lambda: bt.predict(kept[:n_kept]))
    _, p3 = timed(lambda: bt.predict(kept[:n_kept], path="fp64")) if t == 0 else (None, float("nan"))
    print(f"stage {t}: new {new.numel()} fit {fit_ms:.1f} ms  info {info_ms:.2f} ms (K={info[0]}, depth {info[1]}, "
          f"nodes {info[2]})  predict first {p1:.1f} ms, again {p2:.1f} ms, fp64 {p3:.1f} ms  ({amb} rows by fp64)",
          flush=True)
