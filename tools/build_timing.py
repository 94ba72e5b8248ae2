"""Time igp_build_graph (wall clock and CUDA events) on one config (tooling)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402
from synth.dcsbm import CONFIGS, generate  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "headline"]
edges, _ = generate(cfg)
e = torch.from_numpy(edges).cuda()
for i in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g = igp.build_graph(e, cfg.num_nodes)
    t1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    t3 = time.perf_counter()
    g.close()
    t4 = time.perf_counter()
    print(f"build call {1e3*(t1-t0):7.2f} ms  to-idle {1e3*(t2-t0):7.2f} ms  events {a.elapsed_time(b):7.2f} ms  close {1e3*(t4-t3):7.2f} ms")

out = torch.empty((cfg.num_nodes, cfg.d), device="cuda")
for i in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = igp.build_graph(e, cfg.num_nodes)
    t1 = time.perf_counter()
    igp.embed(g, cfg.tau, cfg.d, cfg.steps, 0, out=out)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    g.close()
    t4 = time.perf_counter()
    print(f"[build+embed] build {1e3*(t1-t0):7.2f}  embed-enqueue {1e3*(t2-t1):7.2f}  sync {1e3*(t3-t2):7.2f}  close {1e3*(t4-t3):7.2f} ms")

for tl in (True, False, True):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = igp.build_graph(e, cfg.num_nodes)
    igp.layer_timer_reset()
    igp.embed(g, cfg.tau, cfg.d, cfg.steps, 0, out=out, time_layers=tl)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if tl:
        print("layer ms", igp.layer_timer_read())
    g.close()
    print(f"[time_layers={tl}] step {1e3*(t1-t0):7.2f} ms")
