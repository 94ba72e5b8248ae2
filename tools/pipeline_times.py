"""InfraredGP end to end on the paper's own settings (Table II; Table I-shaped DC-SBM stand-ins):
build + FFP embedding (Alg. 1 l.1-6) + BIRCH fit (l.7) + predict, device/host times beside the
paper's Table IX Emb / Clus / Total columns (RTX 4090 + scikit-learn; context, not a target).

    python tools/pipeline_times.py [paper_5k,...,paper_1m] [--json out.json]

Threshold: T = sqrt(d / 64) (reading B1's T = 1.0 at d = 64, scaled with the embedding's
dimension: sigmoid rows in (0,1)^d).  Embed: median of 3 (CUDA events); fit: host time of the
synchronous call; predict: CUDA events.  Quality context: NMI / ARI of the labels against the
planted blocks (scikit-learn metrics).
"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402
from synth.dcsbm import PAPER_CONFIGS, generate  # noqa: E402

# PAPER.md Table IX (Emb, Clus, Total seconds) per N
PAPER = {5_000: (0.0406, 0.067, 0.1076), 10_000: (0.0469, 0.1411, 0.188), 50_000: (0.1365, 1.1113, 1.2478),
         100_000: (0.4097, 2.2593, 2.6689), 500_000: (1.8373, 14.4521, 16.2894), 1_000_000: (3.6771, 32.9939, 36.6711)}

argv = sys.argv[1:]
out_json = None
if "--json" in argv:
    k = argv.index("--json")
    out_json = argv[k + 1]
    del argv[k:k + 2]
names = argv[0].split(",") if argv else ["paper_5k", "paper_10k", "paper_50k", "paper_100k", "paper_500k", "paper_1m"]
res = {}
for name in names:
    cfg = PAPER_CONFIGS[name]
    edges, planted = generate(cfg)
    e = torch.from_numpy(edges).cuda()
    out = torch.empty((cfg.num_nodes, cfg.d), device="cuda")
    s = torch.cuda.current_stream()
    times = []
    for rep in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g = igp.build_graph(e, cfg.num_nodes, stream=s, async_build=True)
        igp.embed(g, cfg.tau, cfg.d, cfg.steps, cfg.seed, out=out, stream=s)
        g.close(stream=s)
        b.record(s)
        torch.cuda.synchronize()
        if rep:
            times.append(a.elapsed_time(b))
    emb_ms = float(np.median(times))
    T = math.sqrt(cfg.d / 64)
    t0 = time.perf_counter()
    bt = igp.Birch(cfg.d, T, 50).partial_fit(out)
    fit_s = time.perf_counter() - t0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    lab = bt.predict(out)
    b.record(s)
    torch.cuda.synchronize()
    pred_ms = a.elapsed_time(b)
    K, depth = bt.info()[:2]
    bt.close()
    from sklearn.metrics import adjusted_rand_score, normalized_mutual_info_score
    labs = lab.cpu().numpy()
    nmi = normalized_mutual_info_score(planted, labs)
    ari = adjusted_rand_score(planted, labs)
    total_s = emb_ms / 1e3 + fit_s + pred_ms / 1e3
    pe, pc, pt = PAPER[cfg.num_nodes]
    res[name] = {"N": cfg.num_nodes, "d": cfg.d, "tau": cfg.tau, "L": cfg.steps, "T": T, "clusters": K, "depth": depth,
                 "build_embed_ms": emb_ms, "fit_s": fit_s, "predict_ms": pred_ms, "total_s": total_s, "nmi": nmi,
                 "ari": ari, "paper_emb_s": pe, "paper_clus_s": pc, "paper_total_s": pt}
    print(f"{name:11s} N={cfg.num_nodes:8d} d={cfg.d} T={T:.3f}: build+embed {emb_ms:8.2f} ms  BIRCH fit {fit_s:7.3f} s "
          f"predict {pred_ms:7.2f} ms (K={K}, depth {depth})  total {total_s:7.3f} s  | paper Emb {pe} Clus {pc} "
          f"Total {pt} s | NMI {nmi:.3f} ARI {ari:.3f}", flush=True)
if out_json:
    with open(out_json, "w") as f:
        json.dump(res, f, indent=1)
