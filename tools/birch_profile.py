"""One BIRCH fit of the first R rows of a config's GPU embedding (for ncu captures; tooling).

    python tools/birch_profile.py headline 20000 [threshold]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402
from ncu_embed import cached_edges  # noqa: E402
from synth.dcsbm import ALL_CONFIGS  # noqa: E402

cfg = ALL_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "headline"]
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
T = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
e = torch.from_numpy(cached_edges(cfg)).cuda()
g = igp.build_graph(e, cfg.num_nodes)
Z = igp.embed(g, cfg.tau, cfg.d, cfg.steps, cfg.seed)
b = igp.Birch(cfg.d, T, 50).partial_fit(Z[:rows].contiguous())
print("ok", b.info())
