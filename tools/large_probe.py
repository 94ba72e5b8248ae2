import os, sys, torch, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp
from synth.dcsbm import CONFIGS, generate
cfg = CONFIGS["large"]
edges, _ = generate(cfg)
e = torch.from_numpy(edges).cuda()
out = torch.empty((cfg.num_nodes, cfg.d), device="cuda")
g = igp.build_graph(e, cfg.num_nodes)
for L, tl in ((60, False), (60, True), (60, False), (30, False), (10, False)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    igp.layer_timer_reset(); a.record(); igp.embed(g, cfg.tau, cfg.d, L, 0, out=out, time_layers=tl); b.record(); torch.cuda.synchronize()
    extra = igp.layer_timer_read() if tl else ""
    print("L", L, "timed", tl, "embed ms", a.elapsed_time(b), "wall", 1e3 * (time.perf_counter() - t0), extra, flush=True)
