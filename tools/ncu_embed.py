"""One embed of a config (for ncu captures of the filter-step kernel; tooling).

    python tools/ncu_embed.py headline [L]
Edge lists are cached under /tmp/igp_edges_<config>.npy (regenerated if absent; the
generator is deterministic, so the cache never changes a result).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402
from synth.dcsbm import ALL_CONFIGS, generate  # noqa: E402


def cached_edges(cfg):
    path = f"/tmp/igp_edges_{cfg.name}_{cfg.seed}.npy"
    if os.path.exists(path):
        return np.load(path)
    edges, _ = generate(cfg)
    np.save(path, edges)
    return edges


if __name__ == "__main__":
    cfg = ALL_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "headline"]
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    e = torch.from_numpy(cached_edges(cfg)).cuda()
    g = igp.build_graph(e, cfg.num_nodes)
    out = igp.embed(g, cfg.tau, cfg.d, L, cfg.seed)
    torch.cuda.synchronize()
    print("ok", float(out.mean()))
