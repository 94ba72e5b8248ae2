"""The fp64 oracle's per-config FFP rate on the host cores: 1 thread and all allowed cores (tooling;
BASELINE.md §4 "oracle 1-core / all-core").  Each config times `layers` filter steps (+ Philox input
and sigmoid output) on its full graph and reports GEdge·feat/s (a rate, independent of L) and the
implied full-L embed seconds.

    python tools/oracle_times.py [tiny,medium,headline,streaming,large] [--json out.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: tooling may time it)
from synth.dcsbm import CONFIGS, generate  # noqa: E402

argv = sys.argv[1:]
out_json = None
if "--json" in argv:
    k = argv.index("--json")
    out_json = argv[k + 1]
    del argv[k:k + 2]
names = argv[0].split(",") if argv else ["tiny", "medium", "headline", "streaming", "large"]
cores = len(os.sched_getaffinity(0))
res = {}
for name in names:
    cfg = CONFIGS[name]
    edges, _ = generate(cfg)
    rp, ci, _ = oracle.build_csr(edges, cfg.num_nodes)
    nnz = int(ci.size)
    layers = {"tiny": cfg.steps, "medium": 4, "headline": 1, "streaming": 2, "large": 1}[name]
    row = {"nnz": nnz, "layers_timed": layers, "L": cfg.steps}
    for nt in (1, cores):
        t0 = time.perf_counter()
        oracle.embed(rp, ci, cfg.num_nodes, cfg.d, layers, cfg.tau, seed=cfg.seed, nthreads=nt)
        s = time.perf_counter() - t0
        rate = nnz * cfg.d * layers / s / 1e9
        row[f"threads_{nt}"] = {"s": s, "GEdge_feat_per_s": rate,
                                "full_L_embed_s_extrapolated": nnz * cfg.d * cfg.steps / (rate * 1e9)}
    res[name] = row
    print(name, json.dumps(row), flush=True)
if out_json:
    with open(out_json, "w") as f:
        json.dump({"cores": cores, "configs": res}, f, indent=1)
