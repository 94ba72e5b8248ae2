"""BIRCH predict at scale: the tensor-core path (birch_tc.cu) vs the all-fp64 path (tooling).

    python tools/birch_predict_bench.py [fit_rows] [rows] [d] [T] [--reps R] [--profile]
A tree fitted on `fit_rows` synthetic embedding-like rows (sigmoid of N(0, 1.5^2), the FFP's
output distribution; threshold T small enough that most rows stay singleton clusters, the regime
of the streaming Alg. 2 leg where K ~ 1.5e5) predicts `rows` rows (the fitted rows + fresh ones).
Prints per path: device time (CUDA events, median of R), rows left to fp64, and for the tensor
kernel the tensor throughput (3 tf32 products per (row, centroid, k): 6 m Kpad d flop) and its
share of the call.  --profile: one predict per path only (for ncu).
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402

argv = sys.argv[1:]
reps, profile = 5, False
if "--reps" in argv:
    k = argv.index("--reps")
    reps = int(argv[k + 1])
    del argv[k:k + 2]
if "--profile" in argv:
    argv.remove("--profile")
    profile = True
fit_rows = int(argv[0]) if len(argv) > 0 else 150_000
rows = int(argv[1]) if len(argv) > 1 else 200_000
d = int(argv[2]) if len(argv) > 2 else 64
T = float(argv[3]) if len(argv) > 3 else 0.05

g = torch.Generator().manual_seed(7)
Xf = torch.sigmoid(torch.randn((fit_rows, d), generator=g) * 1.5).cuda()
Q = torch.cat([Xf, torch.sigmoid(torch.randn((max(rows - fit_rows, 0), d), generator=g) * 1.5).cuda()])[:rows]
b = igp.Birch(d, T, 50).partial_fit(Xf)
K = b.info()[0]
res = {"fit_rows": fit_rows, "rows": rows, "d": d, "threshold": T, "clusters": K}
labs = {}
if not profile:  # the process's first predict (module load, pool growth) timed apart
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record()
    b.predict(Q, path="tensor")
    p1.record()
    torch.cuda.synchronize()
    res["tensor_first_call_ms"] = p0.elapsed_time(p1)
for path in ("tensor", "fp64"):
    if profile:
        labs[path] = b.predict(Q, path=path)
        torch.cuda.synchronize()
        continue
    b.predict(Q, path=path)  # warm
    ts = []
    for _ in range(reps if path == "tensor" else 1):
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record()
        labs[path] = b.predict(Q, path=path)
        p1.record()
        torch.cuda.synchronize()
        ts.append(p0.elapsed_time(p1))
    res[f"{path}_ms"] = float(np.median(ts))
assert torch.equal(labs["tensor"], labs["fp64"]), "tensor and fp64 labels differ"
_, amb = b.predict(Q, path="tensor", return_ambiguous=True)
res["rows_to_fp64"] = amb
if not profile:
    kpad = -(-K // 128) * 128
    mpad = -(-rows // 128) * 128
    res["tensor_TFLOPs_whole_call"] = 6.0 * mpad * kpad * d / (res["tensor_ms"] * 1e-3) / 1e12
    res["speedup"] = res["fp64_ms"] / res["tensor_ms"]
print(json.dumps(res), flush=True)
b.close()
