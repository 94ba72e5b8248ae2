"""Sweep slice widths on one config: embed ms and filter-step launch time (tooling)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402
from synth.dcsbm import CONFIGS, generate  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "headline"]
widths = [int(w) for w in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["16", "32", "64"])]
occs = [int(o) for o in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["2"])]
envs = [kv for kv in (sys.argv[4].split(";") if len(sys.argv) > 4 else [""])]
from ncu_embed import cached_edges  # noqa: E402
edges = cached_edges(cfg)
e = torch.from_numpy(edges).cuda()
g = igp.build_graph(e, cfg.num_nodes)
out = torch.empty((cfg.num_nodes, cfg.d), device="cuda")
ref = None
for w, occ, env in [(w, o, e) for w in widths for o in occs for e in envs]:
    if w > cfg.d:
        continue
    os.environ["IGP_SLICE_WIDTH"] = str(w)
    os.environ["IGP_LAYER_OCC"] = str(occ)
    for kv in env.split(","):
        if "=" in kv:
            k, v = kv.split("=")
            os.environ[k] = v
    for _ in range(2):
        igp.embed(g, cfg.tau, cfg.d, cfg.steps, 0, out=out)
    torch.cuda.synchronize()
    reps = 3
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(reps):
        igp.embed(g, cfg.tau, cfg.d, cfg.steps, 0, out=out)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / reps
    igp.layer_timer_reset()
    igp.embed(g, cfg.tau, cfg.d, cfg.steps, 0, out=out, time_layers=True)
    torch.cuda.synchronize()
    lms, nl = igp.layer_timer_read()
    if ref is None:
        ref = out.clone()
    diff = float((out - ref).abs().max())
    units = g.nnz * cfg.d * cfg.steps
    print(f"{cfg.name} W={w:3d} occ={occ} {env:28s}: embed {ms:8.2f} ms  {units / ms / 1e6:8.1f} GEdge-feat/s  "
          f"filter launches {nl} avg {lms / nl * 1e3:8.1f} us (per full step {lms / cfg.steps:7.3f} ms)  "
          f"max|diff vs first W| {diff:.2e}", flush=True)
