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
max-over-ranks timing reduction.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth.dcsbm import ALL_CONFIGS as CONFIGS, generate  # noqa: E402

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


def load_gather_ceiling(config_name):
    """Measured random-gather ceiling (GB/s) of this workload's index stream, if profiled."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            v = json.load(f).get(config_name) or {}
        return v.get("gather_ceiling_GBps")
    except Exception:
        return None


def load_traffic(config_name):
    """DRAM bytes (read + write) of one filter-step launch, from the committed ncu --set full
    capture of the bench command (profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        v = t.get(config_name)
        return None if v is None else float(v["dram_bytes_per_launch"])
    except Exception:
        return None


# ---------------------------------------------------------------- CPU oracle leg
def oracle_sample(cfg, edges, layers, nthreads):
    """The fp64 oracle as it stands: CSR (untimed setup), then Alg. 1 l.1-6 with
    `layers` filter steps, timed.  Returns (seconds, nnz)."""
    import oracle
    rp, ci, _ = oracle.build_csr(edges, cfg.num_nodes)
    t0 = time.perf_counter()
    oracle.embed(rp, ci, cfg.num_nodes, cfg.d, layers, cfg.tau, seed=cfg.seed, nthreads=nthreads)
    return time.perf_counter() - t0, int(ci.size)


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
                       "L": cfg.steps, "L_sampled": layers},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "GEdge·feat/s", "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": value, "unit": "GEdge·feat/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm
def run_gpu(args, cfg):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    import paper_2508_19737_b200 as igp

    seed = cfg.seed + rank  # replicas: independent graphs
    t0 = time.perf_counter()
    edges_np, _ = generate(cfg, seed=seed)
    log(f"[rank {rank}] generated {cfg.name}: E={edges_np.shape[0]} in {time.perf_counter() - t0:.1f}s")
    edges = torch.from_numpy(edges_np).to(dev)
    stream = torch.cuda.current_stream(dev)
    N, d, L, tau = cfg.num_nodes, cfg.d, cfg.steps, cfg.tau
    out = torch.empty((N, d), dtype=torch.float32, device=dev)

    def step(timed):
        # the whole step is enqueued without a host sync: asynchronous build (range errors
        # are checked on the warm-up graphs), embed, stream-ordered release of the graph
        g = igp.build_graph(edges, N, stream=stream, async_build=True)
        igp.embed(g, tau, d, L, seed, out=out, stream=stream, time_layers=timed)
        g.close(stream=stream)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize(dev)

    g = igp.build_graph(edges, N, stream=stream)  # synchronous build: validates the input, gives nnz
    nnz = g.nnz
    g.close()
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
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev0.record(stream)
    for k in range(args.steps):
        step(True)
        step_ev[k].record(stream)
    ev1.record(stream)
    barrier()
    log(f"[rank {rank}] per-step ms: " + " ".join(
        f"{(ev0 if k == 0 else step_ev[k - 1]).elapsed_time(step_ev[k]):.2f}" for k in range(args.steps)))
    launches = igp.kernel_launch_count() - launches0
    clock_rec = clocks.stop()
    ms_total = ev0.elapsed_time(ev1)
    tot_layer_ms, tot_launches = igp.layer_timer_read()

    # embed-only timing (no build), same stream, for the breakdown
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

    units = nnz * d * L * args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms_total, float(units)], dtype=torch.float64, device=dev)
        all_t = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(all_t, t)
        per_ms = [float(x[0]) for x in all_t]
        per_units = [float(x[1]) for x in all_t]
    else:
        per_ms, per_units = [ms_total], [float(units)]
    value, t_max = aggregate(per_ms, per_units)
    value /= 1e9

    # roofline of the dominant kernel (the filter step).  One filter step over all d
    # columns is d/W launches of layer_kernel<W> (column slices); the
    # algorithmic bytes are those of the whole step (SURVEY.md §8(d) B_step), so
    # achieved = B_step / (time of the d/W launches that make up one step).
    slices = max(1, tot_launches // max(1, L * args.steps))
    width = d // slices
    avg_launch_s = tot_layer_ms / 1e3 / max(tot_launches, 1)
    step_s = avg_launch_s * slices
    b_step = step_bytes(N, nnz, d)
    peak, peak_src = hbm_peak()
    achieved = b_step / step_s / 1e9
    traffic = load_traffic(cfg.name)
    # per launch (the contract's unit): one filter step is `slices` column-slice launches, so a
    # launch's algorithmic bytes are B_step / slices and achieved = that / the average launch
    # time (identical to B_step / step time); traffic is the ncu DRAM bytes of one launch
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": f"layer_kernel<{width}> ({slices} column-slice launches per filter step)",
            "per": "launch", "algorithmic_bytes": b_step / slices, "algorithmic_bytes_per_step": b_step,
            "traffic_per_step": None if traffic is None else traffic * slices,
            "step_us": step_s * 1e6, "avg_launch_us": avg_launch_s * 1e6, "peak_source": peak_src,
            "gather_bytes_per_step": 4 * nnz * d, "gather_GBps": 4 * nnz * d / step_s / 1e9,
            "gather_ceiling_GBps": load_gather_ceiling(cfg.name),
            "share_of_step": tot_layer_ms / ms_total,
            # whole-embed compulsory bytes over the embed time (SURVEY.md §8(d) "B_embed/(t HBM)")
            "embed_algorithmic_bytes": embed_bytes(N, nnz, d, L),
            "embed_frac": embed_bytes(N, nnz, d, L) / (embed_ms / 1e3) / 1e9 / peak,
            "embed_frac_8TBs": embed_bytes(N, nnz, d, L) / (embed_ms / 1e3) / 8e12}

    line = {"metric": "FFP embed throughput (GEdge·feat/s)", "value": value, "unit": "GEdge·feat/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic DC-SBM (synth/dcsbm.py), seed = rank",
            "config": {"workload": cfg.name, "num_nodes": N, "nnz": nnz, "d": d, "tau": tau, "L": L,
                       "step": "igp_build_graph + igp_embed", "embed_ms": embed_ms,
                       "build_ms": t_max / args.steps - embed_ms,
                       "l2": "inputs > L2: edge list 160 MB, Z 256 MB per buffer, no flush needed",
                       "parallelism": f"replicas x{world}"},
            "roofline": roof, "gpu_launches": launches, "clocks": clock_rec}

    # e2e through the public host-buffer API (pinned host memory in and out)
    if not args.no_e2e:
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
            import torch.distributed as dist
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t)
        line["e2e"] = {"value": nnz * d * L * world / (e2e_ms / 1e3) / 1e9, "unit": "GEdge·feat/s",
                       "ms_per_step": e2e_ms, "h2d_bytes_per_step": int(h_edges.numel() * 4),
                       "d2h_bytes_per_step": int(h_out.numel() * 4)}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = cpu_cores()
        secs, onnz = oracle_sample(cfg, edges_np, args.cpu_layers, cores)
        line["cpu_baseline"] = {"value": onnz * d * args.cpu_layers / secs / 1e9, "unit": "GEdge·feat/s",
                                "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                                "sample": f"{cfg.name} graph, {args.cpu_layers} of L={L} filter steps "
                                          f"(+ Philox input, sigmoid), fp64, {secs:.1f} s"}
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
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: fewer than 3 warm-up steps")
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_gpu(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
