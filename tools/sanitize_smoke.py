"""Small end-to-end exercise of every kernel for compute-sanitizer (memcheck / racecheck / initcheck)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402
from synth.dcsbm import CONFIGS, generate, stream_batches  # noqa: E402

rng = np.random.default_rng(0)
cases = [(generate(CONFIGS["tiny"])[0], 1000),
         (rng.integers(0, 777, (5000, 2)).astype(np.int32), 777),
         (np.zeros((0, 2), np.int32), 5),
         (np.stack([np.zeros(3000, np.int32), np.arange(1, 3001, dtype=np.int32)], 1), 3001)]  # star hub
for edges, n in cases:
    e = torch.from_numpy(np.ascontiguousarray(edges)).cuda()
    for order in ("none", "degree", "community"):
        g = igp.build_graph(e, n, order=order)
        g.csr()
        for d in (16, 32, 64, 128):
            for mode in ("full", "pre_sigmoid", "linear"):
                igp.embed(g, -1.0, d, 3, 0, mode=mode)
        g.close()
# streaming merges, async
c = CONFIGS["tiny"]
bs = [torch.from_numpy(b).cuda() for b in stream_batches(generate(c)[0], 4)]
g = igp.build_graph(bs[0], c.num_nodes, async_build=True, order="community")
for b in bs[1:]:
    g.add_edges(b)
igp.embed(g, -1.0, 64, 5, 0, time_layers=True)
g.status()
g.close()
igp.embed_host(generate(c)[0], c.num_nodes, -1.0, 64, 4, 0)
igp.philox_normal(1, 2, 4096)
igp.philox_bits(1, 2, 4097)
torch.cuda.synchronize()
print("sanitize smoke ok", igp.kernel_launch_count(), "launches")
