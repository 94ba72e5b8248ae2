"""Host-side cost of each call in bench.py's asynchronous step (tooling, not product).

Prints, per step, the host time spent inside build_graph / embed / close and the device
time between events recorded around them, to find where the GPU waits on the host.
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19737_b200 as igp  # noqa: E402
from synth.dcsbm import CONFIGS, generate  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "headline"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
mode = sys.argv[3] if len(sys.argv) > 3 else ""  # "smi": nvidia-smi -lms 100 running; "nvml": pynvml polling
if mode == "smi":
    import subprocess
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks_event_reasons.active", "--format=csv",
                            "-lms", "100", "-i", "0"], stdout=subprocess.DEVNULL)
    time.sleep(1.0)
elif mode == "nvml":
    import threading
    import pynvml
    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
    stop = []

    def poll():
        while not stop:
            pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(hnd)
            time.sleep(0.1)
    threading.Thread(target=poll, daemon=True).start()
edges, _ = generate(cfg)
e = torch.from_numpy(edges).cuda()
N, d, L, tau = cfg.num_nodes, cfg.d, cfg.steps, cfg.tau
out = torch.empty((N, d), device="cuda")
s = torch.cuda.current_stream()
rows = []
for k in range(steps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t0 = time.perf_counter()
    ev[0].record(s)
    g = igp.build_graph(e, N, stream=s, async_build=True)
    t1 = time.perf_counter()
    ev[1].record(s)
    igp.embed(g, tau, d, L, 0, out=out, stream=s, time_layers=(mode != ""))
    t2 = time.perf_counter()
    ev[2].record(s)
    g.close(stream=s)
    t3 = time.perf_counter()
    rows.append((ev, (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3))
torch.cuda.synchronize()
for k, (ev, hb, he, hc) in enumerate(rows):
    print(f"step {k}: host build {hb:7.2f} embed {he:6.2f} close {hc:5.2f} ms | device build "
          f"{ev[0].elapsed_time(ev[1]):7.2f} embed {ev[1].elapsed_time(ev[2]):7.2f} ms"
          + (f" | gap to next {rows[k][0][2].elapsed_time(rows[k + 1][0][0]):6.2f} ms" if k + 1 < len(rows) else ""))
