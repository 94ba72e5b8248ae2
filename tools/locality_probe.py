"""Upper-bound probe for locality reordering (tooling, not product): how fast is the
filter step when rows/columns are numbered so that gathers stay local?

Relabels the headline graph's node ids with several orderings, builds with
IGP_BUILD_NO_REORDER (filter steps run in the given id order) and times the
filter-step launches.  The 'planted' orderings use the generator's block labels and
are an experiment-only upper bound; a product ordering must come from the graph alone.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402
from synth.dcsbm import CONFIGS, generate  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "headline"]
widths = [int(w) for w in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["32", "64"])]
edges, labels = generate(cfg)
n = cfg.num_nodes
deg = np.bincount(edges[:, 0], minlength=n) + np.bincount(edges[:, 1], minlength=n)
rng = np.random.default_rng(1)


def new_ids(order):
    inv = np.empty(n, dtype=np.int32)
    inv[order] = np.arange(n, dtype=np.int32)
    return inv


orders = {
    "identity(random ids)": np.arange(n),
    "degree-desc": np.lexsort((np.arange(n), -deg)),
    "planted block, degree-desc within": np.lexsort((-deg, labels)),
    "planted block, random within": np.lexsort((rng.random(n), labels)),
}
out = torch.empty((n, cfg.d), device="cuda")
for name, order in orders.items():
    inv = new_ids(order)
    e = torch.from_numpy(inv[edges]).cuda()
    g = igp.build_graph(e, n, reorder=False)
    for w in widths:
        os.environ["IGP_SLICE_WIDTH"] = str(w)
        igp.embed(g, cfg.tau, cfg.d, cfg.steps, 0, out=out)
        igp.layer_timer_reset()
        igp.embed(g, cfg.tau, cfg.d, cfg.steps, 0, out=out, time_layers=True)
        torch.cuda.synchronize()
        lms, nl = igp.layer_timer_read()
        print(f"{name:38s} W={w:3d}: filter step {lms / cfg.steps:7.3f} ms  "
              f"gather {4 * g.nnz * cfg.d / (lms / cfg.steps / 1e3) / 1e12:6.2f} TB/s", flush=True)
    g.close()
