"""Embed / build time of every config with the default slice width (tooling)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402
from synth.dcsbm import CONFIGS, generate  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["tiny", "medium", "streaming", "headline", "large"]
for name in names:
    cfg = CONFIGS[name]
    t0 = time.time()
    edges, _ = generate(cfg)
    gen_s = time.time() - t0
    e = torch.from_numpy(edges).cuda()
    out = torch.empty((cfg.num_nodes, cfg.d), device="cuda")
    for _ in range(2):
        g = igp.build_graph(e, cfg.num_nodes)
        igp.embed(g, cfg.tau, cfg.d, cfg.steps, 0, out=out)
        torch.cuda.synchronize()
        g.close()
    reps = 5 if cfg.num_nodes < 2_000_000 else 2
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    bms, ems = [], []
    for _ in range(reps):
        a.record()
        g = igp.build_graph(e, cfg.num_nodes)
        b.record()
        igp.layer_timer_reset()
        igp.embed(g, cfg.tau, cfg.d, cfg.steps, 0, out=out, time_layers=True)
        c.record()
        torch.cuda.synchronize()
        bms.append(a.elapsed_time(b))
        ems.append(b.elapsed_time(c))
        lms, nl = igp.layer_timer_read()
        nnz = g.nnz
        g.close()
    em = sorted(ems)[len(ems) // 2]
    print(f"{name:10s} N={cfg.num_nodes:8d} nnz={nnz:10d} d={cfg.d} L={cfg.steps}: build {sorted(bms)[len(bms)//2]:8.2f} ms  "
          f"embed {em:8.2f} ms  ({nnz * cfg.d * cfg.steps / em / 1e6:7.1f} GEdge-feat/s)  filter launches {nl} "
          f"{lms:8.2f} ms  gen {gen_s:.1f}s", flush=True)
    del e, out
    torch.cuda.empty_cache()
