"""The streaming config's stage-9 merge vs a fresh build of the same graph, for an ncu launch list
(tooling).  Phases are separated by a torch fill kernel (a marker in the launch list):

    fresh build of stages 0-8 | MARK | merge of stage 9 | MARK | fresh build of stages 0-9 | MARK
    python tools/merge_launches.py [reps]      (plain run: prints device ms of both, CUDA events)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402
from synth.dcsbm import ALL_CONFIGS, generate, stream_batches  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = ALL_CONFIGS["streaming"]
edges, _ = generate(cfg)
b = [torch.from_numpy(x).cuda() for x in stream_batches(edges, 10)]
first9 = torch.cat(b[:9])
allb = torch.cat(b)
N = cfg.num_nodes
mark = torch.zeros(1024, device="cuda")


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


tm, tf = [], []
for _ in range(reps):
    g = igp.build_graph(first9, N)
    mark.fill_(1.0)
    a = ev()
    g.add_edges(b[9])
    c = ev()
    mark.fill_(2.0)
    d = ev()
    f = igp.build_graph(allb, N)
    e = ev()
    mark.fill_(3.0)
    torch.cuda.synchronize()
    tm.append(a.elapsed_time(c))
    tf.append(d.elapsed_time(e))
    assert g.nnz == f.nnz
    g.close()
    f.close()
tm.sort()
tf.sort()
print(f"stage-9 merge {tm[len(tm) // 2]:.3f} ms   fresh build {tf[len(tf) // 2]:.3f} ms   ratio "
      f"{tm[len(tm) // 2] / tf[len(tf) // 2]:.3f}  (median of {reps})")
