#!/usr/bin/env python
"""bench.py — InfraredGP FFP embed throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config headline] [--impl igp|reference]

One step = one pass of the whole hot path over the
config's synthetic DC-SBM graph: igp_build_graph (device CSR from the raw edge
list) + igp_embed (Eq. (1) scale, Philox input, L filter steps, sigmoid output).
Inputs (edge list 160 MB, feature buffers 256 MB at Headline) are larger than the
126 MB L2 and already resident in HBM when the timed region starts.

value   = nnz * d * L * K * n_gpus / max-over-ranks device time   (GEdge·feat/s)
e2e     = same metric through igp_embed_host (pinned host edges in, host Z~ out)
roofline= the filter-step kernel, per launch: algorithmic bytes B_step / (column-slice launches
          per step), SURVEY.md §8(d) B_step = 4(N+1) + 4 nnz + 4N + 8 N d, over its average
          CUDA-event launch time, vs the measured HBM copy bandwidth (MEASURED_PEAKS.json);
          traffic = ncu DRAM bytes of one launch (profiles/ncu_traffic.json)
cpu_baseline = the fp64 oracle (oracle/, test infrastructure) on a bounded sample.

--impl reference times the oracle itself as the reference arm (rank 0 only).
Multi-GPU: replicas only: each rank embeds its own graph (seed =
rank), no data-path collective; NCCL is used only for the barrier and the
max-over-ranks timing reduction.  `--gpus N` without a torchrun environment
re-launches itself under torch.distributed.run with N processes.

--config streaming: one step = the 10 cumulative stages of BASELINE.json config 4
(stage 0 build, stages 1-9 igp_graph_add_edges merges, each followed by a re-embed
with Philox subsequence t, Alg. 2 l.1-7); per-stage merge / embed ms are reported.
The default headline run also reports the streaming config's per-stage merge / re-embed ms
("streaming_stages", measured after the timed region; --no-side skips it).
After the timed region the downstream BIRCH (Alg. 1 l.7) is timed once on the step's
embedding and reported beside the FFP ("birch"), with the oracle's BIRCH time.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth.dcsbm import ALL_CONFIGS as CONFIGS, generate, stream_batches  # noqa: E402

FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- helpers
def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def aggregate(per_rank_ms, per_rank_units):
    """Whole-job throughput: all ranks' units over the slowest rank's time (weak scaling)."""
    t = max(per_rank_ms)
    return sum(per_rank_units) / (t / 1e3), t


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def tf32_peak():
    """TF32 dense tensor peak for the tensor-core BIRCH predict: the measured bf16 peak x the guide's
    nominal TF32/bf16 ratio (1.1 / 2.25 PFLOP/s), and the nominal 1.1 PFLOP/s beside it."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["bf16_tflops"]) * 1.1 / 2.25, "measured bf16 x 1.1/2.25 (MEASURED_PEAKS.json)"
    except Exception:
        return 1100.0, "nominal (B200_PROFILING.md)"


def step_bytes(n, nnz, d):
    """compulsory bytes of one filter step (fp32, int32)."""
    return 4 * (n + 1) + 4 * nnz + 4 * n + 8 * n * d


def embed_bytes(n, nnz, d, L):
    """B_embed = L B_step + (4(N+1) + 4 nnz + 12 N) [a4] + (4Nd + 4N) [a5] + (8Nd + 4N) [a8]."""
    return L * step_bytes(n, nnz, d) + (4 * (n + 1) + 4 * nnz + 12 * n) + (4 * n * d + 4 * n) + (8 * n * d + 4 * n)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)), "reasons": sorted(reasons),
                "samples": len(sm)}


TRAFFIC_JSON = os.path.join(ROOT, "profiles", "ncu_traffic.json")
KERNEL_SRC = os.path.join(ROOT, "paper_2508_19737_b200", "csrc", "embed.cu")


def layer_kernel_name(n, width):
    """The filter-step kernel embed.cu launches for this slice (run_embed_w's rule): layer_kernel,
    or the warp-specialised layer_ws_kernel when IGP_LAYER_WS=1 opts in (W >= 32)."""
    env = os.environ.get("IGP_LAYER_WS")
    ws = env is not None and env != "0"
    return "layer_ws_kernel" if ws and width >= 32 else "layer_kernel"


def kernel_source_sha():
    """sha256 of the filter-step kernel's source (the ncu traffic numbers are tied to it)."""
    with open(KERNEL_SRC, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def load_traffic_entry(config_name):
    try:
        with open(TRAFFIC_JSON) as f:
            return json.load(f).get(config_name) or {}
    except Exception:
        return {}


def load_gather_ceiling(config_name):
    """Measured random-gather ceiling (GB/s) of this workload's index stream, if profiled."""
    return load_traffic_entry(config_name).get("gather_ceiling_GBps")


def load_traffic(config_name):
    """DRAM bytes (read + write) of one filter-step launch from the committed ncu --set full
    capture (profiles/ncu_traffic.json), ONLY if it was captured from the current kernel source
    (its kernel_source_sha matches embed.cu); otherwise (None, reason)."""
    v = load_traffic_entry(config_name)
    if "dram_bytes_per_launch" not in v:
        return None, "no ncu capture for this config"
    if v.get("kernel_source_sha") != kernel_source_sha():
        return None, "ncu capture predates the current embed.cu (sha mismatch): not reported"
    return float(v["dram_bytes_per_launch"]), v.get("source")


def l2_policy(cfg, nnz, l2_bytes):
    """How the timing rule on L2 is met for this config (stated in config.l2): inputs larger than
    L2, or an explicit L2 flush between timed steps."""
    edges_b = 8 * cfg.num_edges  # int32 (u, v) pairs (streaming: all 10 stages' batches stay resident)
    z_b = 4 * cfg.num_nodes * cfg.d
    csr_b = 4 * nnz + 4 * (cfg.num_nodes + 1)
    foot = edges_b + z_b + csr_b
    big = foot > 2 * l2_bytes
    desc = (f"footprint {foot / 1e6:.0f} MB (edges {edges_b / 1e6:.0f} MB, CSR {csr_b / 1e6:.0f} MB, "
            f"Z {z_b / 1e6:.0f} MB) vs L2 {l2_bytes / 1e6:.0f} MB: ")
    desc += "inputs > 2 x L2, no flush" if big else "L2 flushed (256 MB write) before every timed step, untimed"
    return (not big), desc


# ---------------------------------------------------------------- CPU oracle leg
def oracle_sample(cfg, edges, layers, nthreads):
    """The fp64 oracle as it stands: CSR (untimed setup), then Alg. 1 l.1-6 with
    `layers` filter steps, timed.  Returns (seconds, nnz)."""
    import oracle
    rp, ci, _ = oracle.build_csr(edges, cfg.num_nodes)
    t0 = time.perf_counter()
    oracle.embed(rp, ci, cfg.num_nodes, cfg.d, layers, cfg.tau, seed=cfg.seed, nthreads=nthreads)
    return time.perf_counter() - t0, int(ci.size)


def oracle_single_thread(cfg, edges, layers=1):
    """The oracle on ONE thread, `layers` filter steps (+ input, output) of the same graph."""
    secs, onnz = oracle_sample(cfg, edges, layers, 1)
    return {"value": onnz * cfg.d * layers / secs / 1e9, "unit": "GEdge·feat/s", "cores": 1, "kind": "oracle",
            "sample": f"{cfg.name} graph, {layers} of L={cfg.steps} filter steps (+ Philox input, sigmoid), fp64, "
                      f"1 thread, {secs:.1f} s"}


def birch_oracle_time(Z, threshold, branching, max_rows=None):
    """The oracle's BIRCH (fit + predict) on the same fp32 rows, single thread (the reference
    for the downstream clustering step)."""
    import oracle
    X = Z if max_rows is None else Z[:max_rows]
    X = X.astype("float64")
    t0 = time.perf_counter()
    b = oracle.Birch(X.shape[1], threshold, branching).fit(X)
    b.predict(X)
    return time.perf_counter() - t0, X.shape[0]


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- reference arm
def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    edges, _ = generate(cfg, seed=cfg.seed)
    cores = cpu_cores()
    layers = args.ref_layers
    import oracle
    rp, ci, _ = oracle.build_csr(edges, cfg.num_nodes)
    nnz = int(ci.size)

    def one():
        t0 = time.perf_counter()
        oracle.embed(rp, ci, cfg.num_nodes, cfg.d, layers, cfg.tau, seed=cfg.seed, nthreads=cores)
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        one()
    ts = [one() for _ in range(args.steps)]
    tot = sum(ts)
    units = nnz * cfg.d * layers * args.steps
    value = units / tot / 1e9
    sample = (f"{cfg.name} graph (N={cfg.num_nodes}, nnz={nnz}, d={cfg.d}), {layers} of L={cfg.steps} filter "
              f"steps per step incl. Philox input + sigmoid, fp64, {cores} threads")
    line = {"metric": "FFP embed throughput (GEdge·feat/s)", "value": value, "unit": "GEdge·feat/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic DC-SBM (synth/dcsbm.py)",
            "config": {"workload": cfg.name, "num_nodes": cfg.num_nodes, "nnz": nnz, "d": cfg.d, "tau": cfg.tau,
                       "L": cfg.steps, "L_sampled": layers,
                       "note": "a per-edge-feature RATE: each step runs the oracle on the full graph for "
                               f"{layers} of the L = {cfg.steps} filter steps (+ input, output); GEdge·feat/s "
                               "does not depend on L, so the ratio to the GPU arm is a per-layer rate ratio"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "GEdge·feat/s", "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": value, "unit": "GEdge·feat/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- distributed plumbing
def dist_init(backend, device=None):
    import torch.distributed as dist
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=device)
    else:
        dist.init_process_group(backend)


def gather_rank_values(vals, device=None):
    """all_gather of a small float64 vector per rank -> list of lists (rank order)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    allt = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(allt, t)
    return [[float(v) for v in x] for x in allt]


def relaunch_under_torchrun(n):
    """`--gpus N` outside torchrun: run this script again as N ranks (one process per GPU)."""
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def base_line(args, cfg, world, value, ms_per_step, dtype, nnz, extra_cfg):
    line = {"metric": "FFP embed throughput (GEdge·feat/s)", "value": value, "unit": "GEdge·feat/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype,
            "data": "synthetic DC-SBM (synth/dcsbm.py), seed = rank",
            "config": {"workload": cfg.name, "num_nodes": cfg.num_nodes, "nnz": nnz, "d": cfg.d, "tau": cfg.tau,
                       "L": cfg.steps, "parallelism": f"replicas x{world}"}}
    line["config"].update(extra_cfg)
    return line


# ---------------------------------------------------------------- CPU self-test of the multi-rank path
def run_selftest_cpu(args, cfg):
    """The multi-rank skeleton of the GPU arm on CPU (gloo): the same init, barrier, per-rank
    timing exchange and aggregation, with a CPU stand-in for the step.  Used by
    tests/test_multirank.py to check `--gpus N` end to end without a GPU."""
    rank, world, _ = dist_env()
    if world > 1:
        dist_init("gloo")
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    acc = 0
    for i in range(20000 * (rank + 1)):  # rank r does (r + 1) units of work
        acc += i * i
    ms = (time.perf_counter() - t0) * 1e3
    units = float(rank + 1) * 1e6
    if world > 1:
        vals = gather_rank_values([ms, units])
        per_ms, per_units = [v[0] for v in vals], [v[1] for v in vals]
    else:
        per_ms, per_units = [ms], [units]
    value, tmax = aggregate(per_ms, per_units)
    if rank == 0:
        line = base_line(args, cfg, world, value / 1e9, tmax / args.steps, "cpu-selftest", 0, {"selftest": True})
        line["per_rank_ms"] = per_ms
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def predict_times(bt, X, stream, dev, fp64=True):
    """igp_birch_predict (auto path: tensor cores where d allows) timed with CUDA events on the
    stream, the rows it left to fp64, and (fp64=True) the all-fp64 path's time beside it."""
    import torch
    rec = {}
    for path in ("auto", "fp64") if fp64 else ("auto",):
        # a tree's first predict sizes its workspaces from the library's memory pool (a pool
        # growth stalls the stream for tens of ms, once): one untimed call, then the median of 3
        bt.predict(X, stream=stream, path=path)
        ts = []
        for _ in range(3):
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record(stream)
            bt.predict(X, stream=stream, path=path)
            p1.record(stream)
            torch.cuda.synchronize(dev)
            ts.append(p0.elapsed_time(p1))
        rec["predict_ms" if path == "auto" else "predict_fp64_ms"] = sorted(ts)[1]
    _, rec["predict_rows_fp64"] = bt.predict(X, stream=stream, return_ambiguous=True)
    return rec


def birch_leg(args, igp, out, stream, dev, N, d, oracle_ref):
    """igp_birch_partial_fit + igp_birch_predict on the step's embedding (Alg. 1 l.7)."""
    import torch
    torch.cuda.synchronize(dev)
    b0 = time.perf_counter()
    bt = igp.Birch(d, args.birch_threshold, args.birch_branching, device=dev).partial_fit(out, stream=stream)
    fit_s = time.perf_counter() - b0
    times = predict_times(bt, out, stream, dev)
    K, depth, nodes, pts = bt.info()
    bt.close()
    rec = {"fit_s": fit_s, **times, "clusters": K, "depth": depth,
           "threshold": args.birch_threshold, "branching": args.birch_branching, "rows": pts,
           "us_per_row": fit_s / max(pts, 1) * 1e6,
           "what": "igp_birch_partial_fit (CF-tree build, one persistent CTA, fp64) + igp_birch_predict on the "
                   "step's embedding; not part of the timed step"}
    if oracle_ref:
        rows = min(N, args.birch_oracle_rows)
        secs, n_rows = birch_oracle_time(out.cpu().numpy(), args.birch_threshold, args.birch_branching, rows)
        rec["oracle"] = {"s": secs, "rows": n_rows, "cores": 1, "us_per_row": secs / n_rows * 1e6,
                         "note": "oracle fit + predict on the first rows of the same embedding"}
    return rec


def streaming_alg2_leg(args, igp, batches, N, d, L, tau, seed, stream, dev):
    """Alg. 2 end to end on the streaming config, after the timed region: per
    stage t, merge (l.1) and re-embed with a fresh draw (l.2-7), extract the rows of the nodes that
    arrived at stage t (their first edge; l.8), partially fit BIRCH with them (l.9), append them to
    the kept embeddings (l.10) and predict every arrived node (l.11).  Row extraction and appending
    are bench-side tensor plumbing; every step of the method runs in the library."""
    import torch
    out = torch.empty((N, d), dtype=torch.float32, device=dev)
    kept = torch.empty((N, d), dtype=torch.float32, device=dev)  # Z^hat: rows of arrived nodes
    seen = torch.zeros(N, dtype=torch.bool, device=dev)
    bt = igp.Birch(d, args.birch_threshold, args.birch_branching, device=dev)
    g = igp.build_graph(batches[0], N, stream=stream)
    rec = []
    n_kept = 0
    for t in range(10):
        if t > 0:
            g.add_edges(batches[t], stream=stream)
        igp.embed(g, tau, d, L, seed, out=out, stream=stream, subsequence=t)
        _, _, deg = g.csr(stream=stream, degrees=True)
        new = torch.nonzero((deg > 0) & ~seen).flatten()
        seen[new] = True
        kept[n_kept:n_kept + new.numel()] = out[new]  # l.8 + l.10 (append)
        torch.cuda.synchronize(dev)
        f0 = time.perf_counter()
        if new.numel():
            bt.partial_fit(kept[n_kept:n_kept + new.numel()], stream=stream)  # l.9 (synchronous)
        fit_ms = (time.perf_counter() - f0) * 1e3
        n_kept += new.numel()
        times = predict_times(bt, kept[:n_kept], stream, dev, fp64=(t == 9))  # l.11
        K = bt.info()[0]
        rec.append({"stage": t, "new_nodes": int(new.numel()), "partial_fit_ms": fit_ms, **times, "clusters": K})
    g.close()
    bt.close()
    # the final stage's predict against the TF32 tensor peak: 3 TF32 products per (row, cluster,
    # column) over the padded tiles (whole call: split, both tensor passes, re-checks)
    last = rec[-1]
    tile_n = 256 if d >= 48 else 128
    flops = 6.0 * (-(-n_kept // 128) * 128) * (-(-last["clusters"] // tile_n) * tile_n) * d
    peak, src = tf32_peak()
    ach = flops / (last["predict_ms"] * 1e-3) / 1e12
    roof = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
            "peak_source": src, "nominal_peak": 1100.0, "frac_of_nominal": ach / 1100.0,
            "what": "igp_birch_predict (tensor-core path) on the final stage, whole call, 6 m Kpad d flops"}
    return {"stages": rec, "threshold": args.birch_threshold, "branching": args.birch_branching,
            "predict_roofline": roof,
            "new_nodes": "nodes whose first edge arrives at stage t (edge-arrival stream)"}


# ---------------------------------------------------------------- GPU arm
def streaming_side_leg(igp, dev, stream, reps=3):
    """BASELINE.json config 4 (Alg. 2 l.1-7) measured inside the default headline
    run, after its timed region, so a driver-run line carries per-stage merge / re-embed times:
    stage 0 build, stages 1-9 igp_graph_add_edges merges, each followed by a re-embed with
    Philox subsequence t.  Medians over `reps` runs after one warm-up; CUDA events on `stream`."""
    import torch
    cfg = CONFIGS["streaming"]
    edges_np, _ = generate(cfg, seed=cfg.seed)
    batches = [torch.from_numpy(b).to(dev) for b in stream_batches(edges_np, 10)]
    N, d, L, tau = cfg.num_nodes, cfg.d, cfg.steps, cfg.tau
    out = torch.empty((N, d), dtype=torch.float32, device=dev)
    runs = []
    for r in range(reps + 1):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g = igp.build_graph(batches[0], N, stream=stream, async_build=True)
        for t in range(10):
            if t > 0:
                g.add_edges(batches[t], stream=stream)
            ev[t][0].record(stream)
            igp.embed(g, tau, d, L, cfg.seed, out=out, stream=stream, subsequence=t)
            ev[t][1].record(stream)
        torch.cuda.synchronize(dev)
        nnz = g.nnz
        g.close()
        starts = [e0] + [ev[t - 1][1] for t in range(1, 10)]
        if r > 0:  # r == 0 warms up
            runs.append(([starts[t].elapsed_time(ev[t][0]) for t in range(10)],
                         [a.elapsed_time(b) for a, b in ev], e0.elapsed_time(ev[9][1])))
    fb = []
    all_edges = torch.cat(batches)
    for _ in range(reps + 1):
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        gf = igp.build_graph(all_edges, N, stream=stream, async_build=True)
        f1.record(stream)
        torch.cuda.synchronize(dev)
        gf.close()
        fb.append(f0.elapsed_time(f1))
    med = lambda xs: float(np.median(xs))  # noqa: E731
    merge = [med([r[0][t] for r in runs]) for t in range(10)]
    emb = [med([r[1][t] for r in runs]) for t in range(10)]
    fresh = med(fb[1:])
    return {"workload": "streaming (BASELINE.json config 4): N=200,000, 10 cumulative stages",
            "final_nnz": int(nnz), "d": d, "L": L, "tau": tau, "reps": reps,
            "build_or_merge_ms": merge, "embed_ms": emb, "ten_stage_ms": med([r[2] for r in runs]),
            "fresh_build_of_final_graph_ms": fresh, "merge_stage9_vs_fresh_build": merge[9] / fresh}


def run_gpu(args, cfg):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist_init("nccl", dev)
    import paper_2508_19737_b200 as igp

    seed = cfg.seed + rank  # replicas: independent graphs
    t0 = time.perf_counter()
    edges_np, _ = generate(cfg, seed=seed)
    log(f"[rank {rank}] generated {cfg.name}: E={edges_np.shape[0]} in {time.perf_counter() - t0:.1f}s")
    edges = torch.from_numpy(edges_np).to(dev)
    stream = torch.cuda.current_stream(dev)
    N, d, L, tau = cfg.num_nodes, cfg.d, cfg.steps, cfg.tau
    out = torch.empty((N, d), dtype=torch.float32, device=dev)
    streaming = cfg.name == "streaming"
    batches = [torch.from_numpy(b).to(dev) for b in stream_batches(edges_np, 10)] if streaming else None
    stage_ev = None

    def step(timed, record_stages=False):
        # the whole step is enqueued without a host sync: asynchronous build (range errors are
        # checked on the warm-up graphs), embed, stream-ordered release of the graph
        if not streaming:
            g = igp.build_graph(edges, N, stream=stream, async_build=True)
            igp.embed(g, tau, d, L, seed, out=out, stream=stream, time_layers=timed)
            g.close(stream=stream)
            return
        # Alg. 2 l.1-7 over the 10 cumulative stages: stage 0 build, then merge + re-embed
        g = igp.build_graph(batches[0], N, stream=stream, async_build=True)
        for t in range(10):
            if t > 0:
                g.add_edges(batches[t], stream=stream)
            if record_stages:
                stage_ev[t][0].record(stream)
            igp.embed(g, tau, d, L, seed, out=out, stream=stream, time_layers=timed, subsequence=t)
            if record_stages:
                stage_ev[t][1].record(stream)
        g.close(stream=stream)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize(dev)

    # units of one step: nnz x d x L (streaming: summed over the 10 stages' graphs)
    if streaming:
        g = igp.build_graph(batches[0], N, stream=stream)
        stage_nnz = [g.nnz]
        for t in range(1, 10):
            g.add_edges(batches[t], stream=stream)
            stage_nnz.append(g.nnz)
        g.close()
        nnz = stage_nnz[-1]
        units_step = sum(stage_nnz) * d * L
    else:
        g = igp.build_graph(edges, N, stream=stream)  # synchronous build: validates the input, gives nnz
        nnz = g.nnz
        g.close()
        units_step = nnz * d * L
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    flush, l2_desc = l2_policy(cfg, nnz, l2_bytes)
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev) if flush else None

    for _ in range(args.warmup):
        step(True)  # same calls as the timed steps (the timer's events are created here)
    torch.cuda.synchronize(dev)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    step(True)  # the GPU idled while the sampler started: one more untimed step brings it back up
    igp.layer_timer_reset()
    launches0 = igp.kernel_launch_count()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if streaming:
        stage_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for k in range(args.steps):
        if flush:
            flush_buf.fill_(float(k))  # untimed: outside the step's events
        ev[k][0].record(stream)
        step(True, record_stages=streaming and k == args.steps - 1)
        ev[k][1].record(stream)
    barrier()
    per_step = [a.elapsed_time(b) for a, b in ev]
    log(f"[rank {rank}] per-step ms: " + " ".join(f"{x:.2f}" for x in per_step))
    launches = igp.kernel_launch_count() - launches0
    clock_rec = clocks.stop()
    ms_total = sum(per_step)
    tot_layer_ms, tot_launches = igp.layer_timer_read()
    stages = None
    if streaming:
        st_embed = [a.elapsed_time(b) for a, b in stage_ev]
        # stage t's build / merge = from the previous stage's embed end (or the step start) to this embed
        starts = [ev[-1][0]] + [stage_ev[t - 1][1] for t in range(1, 10)]
        st_merge = [starts[t].elapsed_time(stage_ev[t][0]) for t in range(10)]
        stages = [{"stage": t, "nnz": stage_nnz[t], "build_or_merge_ms": st_merge[t], "embed_ms": st_embed[t]}
                  for t in range(10)]
        # reference for the merges: a fresh build of the final (stage-9) graph from all its edges
        all_edges = torch.cat(batches)
        fb = []
        for _ in range(4):
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            gf = igp.build_graph(all_edges, N, stream=stream, async_build=True)
            f1.record(stream)
            gf.close(stream=stream)
            torch.cuda.synchronize(dev)
            fb.append(f0.elapsed_time(f1))
        fresh_build_ms = float(np.median(fb[1:]))

    # embed-only timing (no build), same stream, for the breakdown (static configs)
    embed_ms = None
    if not streaming:
        g = igp.build_graph(edges, N, stream=stream)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            igp.embed(g, tau, d, L, seed, out=out, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        embed_ms = e0.elapsed_time(e1) / args.steps
        g.close()

    units = units_step * args.steps
    if world > 1:
        vals = gather_rank_values([ms_total, float(units)], dev)
        per_ms, per_units = [v[0] for v in vals], [v[1] for v in vals]
    else:
        per_ms, per_units = [ms_total], [float(units)]
    value, t_max = aggregate(per_ms, per_units)
    value /= 1e9

    # roofline of the dominant kernel (the filter step).  One filter step over all d
    # columns is d/W launches of layer_kernel<W> (column slices); the
    # algorithmic bytes are those of the whole step (SURVEY.md §8(d) B_step), so
    # achieved = B_step / (time of the d/W launches that make up one step).
    n_embeds = 10 if streaming else 1
    slices = max(1, tot_launches // max(1, L * args.steps * n_embeds))
    width = d // slices
    avg_launch_s = tot_layer_ms / 1e3 / max(tot_launches, 1)
    step_s = avg_launch_s * slices
    b_step = step_bytes(N, nnz, d)
    peak, peak_src = hbm_peak()
    achieved = b_step / step_s / 1e9
    traffic, traffic_src = load_traffic(cfg.name)
    # per launch (the contract's unit): one filter step is `slices` column-slice launches, so a
    # launch's algorithmic bytes are B_step / slices and achieved = that / the average launch
    # time (identical to B_step / step time); traffic is the ncu DRAM bytes of one launch
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_source": traffic_src, "kernel_source_sha": kernel_source_sha()[:16],
            "kernel": f"{layer_kernel_name(N, width)}<{width}> ({slices} column-slice launches per filter step)",
            "per": "launch", "algorithmic_bytes": b_step / slices, "algorithmic_bytes_per_step": b_step,
            "traffic_per_step": None if traffic is None else traffic * slices,
            "step_us": step_s * 1e6, "avg_launch_us": avg_launch_s * 1e6, "peak_source": peak_src,
            "gather_bytes_per_step": 4 * nnz * d, "gather_GBps": 4 * nnz * d / step_s / 1e9,
            "gather_ceiling_GBps": load_gather_ceiling(cfg.name),
            "share_of_step": tot_layer_ms / ms_total}
    if streaming:
        roof["note"] = "streaming: the final stage's nnz (the largest graph) is the byte basis of B_step"
    if embed_ms is not None:
        # whole-embed compulsory bytes over the embed time (SURVEY.md §8(d) "B_embed/(t HBM)")
        roof.update({"embed_algorithmic_bytes": embed_bytes(N, nnz, d, L),
                     "embed_frac": embed_bytes(N, nnz, d, L) / (embed_ms / 1e3) / 1e9 / peak,
                     "embed_frac_8TBs": embed_bytes(N, nnz, d, L) / (embed_ms / 1e3) / 8e12})

    step_desc = ("10 stages: igp_build_graph (stage 0) / igp_graph_add_edges (stages 1-9) + igp_embed "
                 "(subsequence t)" if streaming else "igp_build_graph + igp_embed")
    extra = {"step": step_desc, "l2": l2_desc}
    if embed_ms is not None:
        extra.update({"embed_ms": embed_ms, "build_ms": t_max / args.steps - embed_ms})
    if stages is not None:
        if not args.no_birch:
            try:
                extra["alg2_birch"] = streaming_alg2_leg(args, igp, batches, N, d, L, tau, seed, stream, dev)
            except Exception as exc:  # noqa: BLE001
                extra["alg2_birch"] = {"error": f"{type(exc).__name__}: {exc}"}
        extra["stages"] = stages
        extra["fresh_build_of_final_graph_ms"] = fresh_build_ms
        extra["merge_stage9_vs_fresh_build"] = stages[9]["build_or_merge_ms"] / fresh_build_ms
        extra["units_per_step"] = "sum over the 10 stages of nnz_t x d x L"
    line = base_line(args, cfg, world, value, t_max / args.steps, "f32", nnz, extra)
    line.update({"roofline": roof, "gpu_launches": launches, "clocks": clock_rec})

    # e2e through the public host-buffer API (pinned host memory in and out); static configs
    if not args.no_e2e and not streaming:
        h_edges = torch.from_numpy(edges_np).pin_memory()
        h_out = torch.empty((N, d), dtype=torch.float32, pin_memory=True)
        igp.embed_host(h_edges, N, tau, d, L, seed, out=h_out, stream=stream)  # warm
        ke = max(1, min(args.steps, 3))
        barrier()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record(stream)
        for _ in range(ke):
            igp.embed_host(h_edges, N, tau, d, L, seed, out=h_out, stream=stream)
        x1.record(stream)
        barrier()
        e2e_ms = x0.elapsed_time(x1) / ke
        if world > 1:
            e2e_ms = max(v[0] for v in gather_rank_values([e2e_ms], dev))
        line["e2e"] = {"value": nnz * d * L * world / (e2e_ms / 1e3) / 1e9, "unit": "GEdge·feat/s",
                       "ms_per_step": e2e_ms, "h2d_bytes_per_step": int(h_edges.numel() * 4),
                       "d2h_bytes_per_step": int(h_out.numel() * 4)}

    # the downstream BIRCH (Alg. 1 l.7) on this step's embedding: reported beside the FFP, not
    # part of the step; the oracle's BIRCH on the same rows (one thread) is its reference
    if not args.no_birch:
        try:  # a failure here must not cost the bench line: it is reported instead
            line["birch"] = birch_leg(args, igp, out, stream, dev, N, d,
                                      oracle_ref=rank == 0 and world == 1 and not args.no_cpu_baseline)
        except Exception as exc:  # noqa: BLE001
            line["birch"] = {"error": f"{type(exc).__name__}: {exc}"}

    # the streaming config's per-stage merge / re-embed times beside the headline (not part of
    # the headline step or its value)
    if rank == 0 and world == 1 and cfg.name == "headline" and not args.no_side:
        try:
            line["streaming_stages"] = streaming_side_leg(igp, dev, stream)
        except Exception as exc:  # noqa: BLE001
            line["streaming_stages"] = {"error": f"{type(exc).__name__}: {exc}"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = cpu_cores()
        secs, onnz = oracle_sample(cfg, edges_np if not streaming else np.concatenate(stream_batches(edges_np, 10)),
                                   args.cpu_layers, cores)
        line["cpu_baseline"] = {"value": onnz * d * args.cpu_layers / secs / 1e9, "unit": "GEdge·feat/s",
                                "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                                "sample": f"{cfg.name} graph, {args.cpu_layers} of L={L} filter steps "
                                          f"(+ Philox input, sigmoid), fp64, {secs:.1f} s",
                                "single_thread": oracle_single_thread(cfg, edges_np, 1)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="igp", choices=["igp", "reference"])
    ap.add_argument("--config", default="headline", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-layers", type=int, default=2)
    ap.add_argument("--ref-layers", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-birch", action="store_true")
    ap.add_argument("--no-side", action="store_true", help="skip the streaming per-stage leg of the headline run")
    ap.add_argument("--birch-threshold", type=float, default=1.0)  # reading B1
    ap.add_argument("--birch-branching", type=int, default=50)
    ap.add_argument("--birch-oracle-rows", type=int, default=200_000)
    ap.add_argument("--selftest-cpu", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: fewer than 3 warm-up steps")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args.gpus)
    cfg = CONFIGS[args.config]
    if args.selftest_cpu:
        return run_selftest_cpu(args, cfg)
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_gpu(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
