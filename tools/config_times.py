"""Device times of every BASELINE.json config (tooling; results go to profiles/ and DESIGN.md).

    python tools/config_times.py [tiny,medium,headline,streaming,large,large_noreorder] [--json out.json]

static configs: build (igp_build_graph, async) + embed, median of reps, CUDA events on one stream;
streaming: stage 0 build + 9 igp_graph_add_edges merges, each followed by a re-embed (Philox
subsequence t), all enqueued without a host sync; per-stage merge and embed times.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402
from synth.dcsbm import ALL_CONFIGS as CONFIGS, generate, stream_batches  # noqa: E402

argv = sys.argv[1:]
out_json = None
if "--json" in argv:
    k = argv.index("--json")
    out_json = argv[k + 1]
    del argv[k:k + 2]
names = argv[0].split(",") if argv else ["tiny", "medium", "headline", "headline_degree", "streaming", "large",
                                         "large_degree", "large_noreorder"]
results = {}


def ev():
    return torch.cuda.Event(enable_timing=True)


def static(name):
    base, suffix = name, ""
    for sfx in ("_degree", "_noreorder", "_community"):
        if name.endswith(sfx):
            base, suffix = name[: -len(sfx)], sfx[1:]
    order = {"": "auto", "degree": "degree", "noreorder": "none", "community": "community"}[suffix]
    reorder = order != "none"
    cfg = CONFIGS[base]
    edges, _ = generate(cfg)
    e = torch.from_numpy(edges).cuda()
    out = torch.empty((cfg.num_nodes, cfg.d), device="cuda")
    s = torch.cuda.current_stream()
    g = igp.build_graph(e, cfg.num_nodes, order=order)
    nnz = g.nnz
    g.close()
    reps = 7 if cfg.num_nodes < 2_000_000 else 3
    for _ in range(2):  # warm-up
        g = igp.build_graph(e, cfg.num_nodes, stream=s, order=order, async_build=True)
        igp.embed(g, cfg.tau, cfg.d, cfg.steps, 0, out=out, stream=s)
        g.close(stream=s)
    igp.layer_timer_reset()
    marks = []
    for _ in range(reps):
        a, b, c = ev(), ev(), ev()
        a.record(s)
        g = igp.build_graph(e, cfg.num_nodes, stream=s, order=order, async_build=True)
        b.record(s)
        igp.embed(g, cfg.tau, cfg.d, cfg.steps, 0, out=out, stream=s, time_layers=True)
        c.record(s)
        g.close(stream=s)
        marks.append((a, b, c))
    torch.cuda.synchronize()
    lms, nl = igp.layer_timer_read()
    bms = sorted(a.elapsed_time(b) for a, b, _ in marks)[reps // 2]
    ems = sorted(b.elapsed_time(c) for _, b, c in marks)[reps // 2]
    units = nnz * cfg.d * cfg.steps
    r = {"N": cfg.num_nodes, "nnz": nnz, "d": cfg.d, "L": cfg.steps, "tau": cfg.tau, "order": order,
         "build_ms": bms, "embed_ms": ems, "step_ms": bms + ems,
         "GEdge_feat_per_s_embed": units / ems / 1e6, "GEdge_feat_per_s_step": units / (bms + ems) / 1e6,
         "filter_step_ms": lms / reps / cfg.steps,  # all column slices of one filter step
         "filter_launches_per_embed": nl // reps}
    print(f"{name:16s} N={cfg.num_nodes:8d} nnz={nnz:10d} d={cfg.d:3d} L={cfg.steps}: build {bms:8.2f} ms  "
          f"embed {ems:8.2f} ms  step {units / (bms + ems) / 1e6:8.1f} GEdge-feat/s  filter step "
          f"{r['filter_step_ms']:.3f} ms", flush=True)
    return r


def streaming():
    cfg = CONFIGS["streaming"]
    edges, _ = generate(cfg)
    batches = [torch.from_numpy(b).cuda() for b in stream_batches(edges, 10)]
    out = torch.empty((cfg.num_nodes, cfg.d), device="cuda")
    s = torch.cuda.current_stream()
    rows = None
    for rep in range(3):  # last repetition is reported (the first ones warm the pool)
        marks = []
        for t, b in enumerate(batches):
            a, m, c = ev(), ev(), ev()
            a.record(s)
            if t == 0:
                g = igp.build_graph(b, cfg.num_nodes, stream=s, async_build=True)
            else:
                g.add_edges(b, stream=s)
            m.record(s)
            igp.embed(g, cfg.tau, cfg.d, cfg.steps, 0, out=out, stream=s, subsequence=t)
            c.record(s)
            marks.append((a, m, c))
        torch.cuda.synchronize()
        nnz = g.nnz
        g.close()
        rows = [(a.elapsed_time(m), m.elapsed_time(c)) for a, m, c in marks]
    tot = sum(x + y for x, y in rows)
    for t, (x, y) in enumerate(rows):
        print(f"streaming stage {t}: {'build' if t == 0 else 'merge'} {x:7.3f} ms  embed {y:7.3f} ms", flush=True)
    print(f"streaming total (10 stages, final nnz {nnz}): {tot:.2f} ms", flush=True)
    return {"N": cfg.num_nodes, "final_nnz": nnz, "d": cfg.d, "L": cfg.steps, "stages": 10,
            "stage_build_or_merge_ms": [x for x, _ in rows], "stage_embed_ms": [y for _, y in rows],
            "total_ms": tot}


for name in names:
    results[name] = streaming() if name == "streaming" else static(name)
    torch.cuda.empty_cache()
if out_json:
    with open(out_json, "w") as f:
        json.dump(results, f, indent=1)
