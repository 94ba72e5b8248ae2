import os, sys, torch, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from cuda.bindings import runtime as cudart
import paper_2508_19737_b200 as igp
from synth.dcsbm import CONFIGS, generate
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "large"]
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
edges, _ = generate(cfg)
e = torch.from_numpy(edges).cuda()
out = torch.empty((cfg.num_nodes, cfg.d), device="cuda")
def pool():
    _, p = cudart.cudaDeviceGetDefaultMemPool(0)
    _, r = cudart.cudaMemPoolGetAttribute(p, cudart.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)
    _, u = cudart.cudaMemPoolGetAttribute(p, cudart.cudaMemPoolAttr.cudaMemPoolAttrUsedMemCurrent)
    return int(r) >> 20, int(u) >> 20
for i in range(int(os.environ.get("ITERS", "5"))):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g = igp.build_graph(e, cfg.num_nodes); torch.cuda.synchronize(); t1 = time.perf_counter()
    igp.embed(g, cfg.tau, cfg.d, L, 0, out=out); torch.cuda.synchronize(); t2 = time.perf_counter()
    g.close(); t3 = time.perf_counter()
    print(f"iter {i}: build {1e3*(t1-t0):8.1f} embed {1e3*(t2-t1):8.1f} close {1e3*(t3-t2):6.1f} ms  pool reserved/used MB {pool()}", flush=True)
