"""Three headline builds (default row order) for an ncu launch list of the builder (tooling)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402
from synth.dcsbm import ALL_CONFIGS, generate  # noqa: E402

cfg = ALL_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "headline"]
order = sys.argv[2] if len(sys.argv) > 2 else "auto"
edges, _ = generate(cfg)
e = torch.from_numpy(edges).cuda()
for _ in range(3):
    g = igp.build_graph(e, cfg.num_nodes, order=order)
    g.close()
torch.cuda.synchronize()
print("ok")
