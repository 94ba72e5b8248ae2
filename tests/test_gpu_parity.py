"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Bars (north star):
  - CSR: bit-exact (row_ptr, col_idx) on adversarial lists and the DC-SBM configs;
  - Philox raw words: bit-exact; normals: within 1 fp32 ulp of the fp64 value;
  - embeddings: max_i max_c |gpu - oracle| / ||oracle_i||_2 <= 1e-4 (fp32 vs fp64).
All inputs are seeded and synthetic (synth/dcsbm.py).
"""
import os

import numpy as np
import pytest
import torch

import oracle
from conftest import record, row_rel_err
from synth.dcsbm import CONFIGS, generate

pytestmark = pytest.mark.gpu

TOL = 1e-4  # north-star row-relative tolerance
NTHREADS = max(1, len(os.sched_getaffinity(0)))


@pytest.fixture(scope="module")
def igp():
    if not torch.cuda.is_available():
        pytest.fail("GPU test requires CUDA (no CPU fallback)")
    import paper_2508_19737_b200 as m
    return m


def gpu_graph(igp, edges, n):
    e = torch.from_numpy(np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))).cuda()
    return igp.build_graph(e, n)


def check_csr(igp, edges, n):
    g = gpu_graph(igp, edges, n)
    rp, ci = g.csr()
    torch.cuda.synchronize()
    rp_o, ci_o, m_o = oracle.build_csr(edges, n)
    assert g.num_edges == m_o and g.nnz == 2 * m_o
    assert np.array_equal(rp.cpu().numpy(), rp_o), "row_ptr differs"
    assert np.array_equal(ci.cpu().numpy(), ci_o), "col_idx differs"
    return g, rp_o, ci_o


# ------------------------------------------------------------------ CSR
def adversarial_edge_lists():
    rng = np.random.default_rng(0)
    cases = {
        "empty": (np.zeros((0, 2), np.int32), 3),
        "single_node": (np.zeros((0, 2), np.int32), 1),
        "self_loops_only": (np.array([[0, 0], [1, 1], [2, 2]], np.int32), 3),
        "dups_both_orient": (np.array([[0, 1], [1, 0], [0, 1], [1, 1], [2, 0], [0, 2]], np.int32), 4),
        "random_small": (rng.integers(0, 50, (400, 2)).astype(np.int32), 50),
        "ragged_tail": (rng.integers(0, 2049, (30000, 2)).astype(np.int32), 2049),
    }
    # stars: hub rows that take the block-sort (1024 < len <= 16384) and bitmap (> 16384) paths
    for name, leaves in [("star_1500", 1500), ("star_20000", 20000)]:
        n = leaves + 1
        e = np.stack([np.zeros(leaves, np.int32), np.arange(1, n, dtype=np.int32)], 1)
        e = np.concatenate([e, e[::3, ::-1], rng.integers(0, n, (2000, 2)).astype(np.int32)])
        cases[name] = (e[rng.permutation(e.shape[0])], n)
    # a dense core: many rows with raw length > 1024 (duplicates included)
    n = 3000
    core = rng.integers(0, 64, (80000, 2)).astype(np.int32)
    cases["dense_core"] = (np.concatenate([core, rng.integers(0, n, (5000, 2)).astype(np.int32)]), n)
    return cases


@pytest.mark.parametrize("name", list(adversarial_edge_lists()))
def test_csr_bit_exact_adversarial(igp, name):
    edges, n = adversarial_edge_lists()[name]
    check_csr(igp, edges, n)


@pytest.mark.parametrize("cfg", ["tiny", "medium", "streaming"])
def test_csr_bit_exact_configs(igp, cfg):
    c = CONFIGS[cfg]
    edges, _ = generate(c)
    check_csr(igp, edges, c.num_nodes)


def test_csr_out_of_range_is_input_error(igp):
    with pytest.raises(igp.IGPError) as ei:
        gpu_graph(igp, np.array([[0, 1], [2, 5]], np.int32), 5)
    assert ei.value.status == 2
    with pytest.raises(igp.IGPError):
        gpu_graph(igp, np.array([[0, -1]], np.int32), 5)


# ------------------------------------------------------------------ Philox
@pytest.mark.parametrize("seed,sub", [(0, 0), (1234, 5), (2**40 + 17, 3)])
def test_philox_bits_bit_exact(igp, seed, sub):
    count = 4 * 100_003
    got = igp.philox_bits(seed, sub, count).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, oracle.philox_bits(seed, sub, count))


def test_philox_normal_within_one_ulp(igp):
    count = 1 << 20
    got = igp.philox_normal(7, 2, count).cpu().numpy()
    ref = oracle.normal(7, 2, count)
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(got.astype(np.float64) - ref) <= ulp)


# ------------------------------------------------------------------ embeddings
def run_parity(igp, edges, n, d, L, tau, seed=0, mode="full", sub=0, floor=None, **kw):
    """GPU embed vs the fp64 oracle on the same seeded input.  With floor=<name>, the oracle's
    fp32 twin (same steps in float) is run too and its drift from the fp64
    oracle is recorded as <name>_fp32_floor beside the GPU error (the irreducible fp32 part)."""
    g = gpu_graph(igp, edges, n)
    z = igp.embed(g, tau, d, L, seed, mode=mode, subsequence=sub, **kw).cpu().numpy()
    rp, ci, _ = oracle.build_csr(edges, n)
    omode = {"full": oracle.MODE_FULL, "pre_sigmoid": oracle.MODE_PRE_SIGMOID, "linear": oracle.MODE_LINEAR}[mode]
    ref = oracle.embed(rp, ci, n, d, L, tau, seed=seed, sub=sub, mode=omode, nthreads=NTHREADS, **kw)
    if floor is not None:
        twin = oracle.embed(rp, ci, n, d, L, tau, seed=seed, sub=sub, mode=omode, nthreads=NTHREADS,
                            fp32_twin=True, **kw)
        record(f"{floor}_fp32_floor", row_rel_err(twin, ref))
    return z, ref


def test_embed_tiny_config(igp):
    c = CONFIGS["tiny"]
    edges, _ = generate(c)
    z, ref = run_parity(igp, edges, c.num_nodes, c.d, c.steps, c.tau, floor="tiny")
    err = row_rel_err(z, ref)
    record("tiny", err)
    assert err <= TOL
    assert z.min() > 0 and z.max() < 1


@pytest.mark.parametrize("tau", [-1.5, -1.0, 0.0])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_embed_medium_config(igp, tau, seed):
    c = CONFIGS["medium"]
    edges, _ = generate(c, seed=seed)
    z, ref = run_parity(igp, edges, c.num_nodes, c.d, c.steps, tau, seed=seed, floor=f"medium_tau{tau}_seed{seed}")
    err = row_rel_err(z, ref)
    record(f"medium_tau{tau}_seed{seed}", err)
    assert err <= TOL


@pytest.mark.parametrize("d", [16, 32, 48, 64, 96, 128, 192, 256])
@pytest.mark.parametrize("n", [1, 7, 777, 4099])
def test_embed_dims_and_ragged_sizes(igp, d, n):
    rng = np.random.default_rng(n + d)
    edges = rng.integers(0, n, (6 * n, 2)).astype(np.int32)
    for mode in ["full", "pre_sigmoid"]:
        z, ref = run_parity(igp, edges, n, d, 6, -1.0, seed=3, mode=mode)
        err = row_rel_err(z, ref)
        record(f"ragged_n{n}_d{d}_{mode}", err)
        assert err <= TOL, (mode, d, n)


@pytest.mark.parametrize("w", [32, 64, 128])
@pytest.mark.parametrize("mode", ["full", "linear"])
def test_layer_ws_kernel_bit_identical(igp, w, mode, monkeypatch):
    """The warp-specialised filter step (layer_ws_kernel: gather warps hand row sums to epilogue
    warps; the default for DRAM-bound slices) computes the same arithmetic in the
    same order as layer_kernel: bit-identical outputs at every slice width, a ragged N (partial
    last row batch), and within the tolerance of the oracle."""
    n, d, L = 40961, 128, 8
    rng = np.random.default_rng(w)
    edges = rng.integers(0, n, (20 * n, 2)).astype(np.int32)
    g = gpu_graph(igp, edges, n)
    monkeypatch.setenv("IGP_SLICE_WIDTH", str(w))
    outs = []
    for ws in ("0", "1"):
        monkeypatch.setenv("IGP_LAYER_WS", ws)
        outs.append(igp.embed(g, -1.0, d, L, 5, mode=mode))
    assert torch.equal(outs[0], outs[1])
    rp, ci, _ = oracle.build_csr(edges, n)
    omode = oracle.MODE_FULL if mode == "full" else oracle.MODE_LINEAR
    ref = oracle.embed(rp, ci, n, d, L, -1.0, seed=5, mode=omode, nthreads=NTHREADS)
    err = row_rel_err(outs[1].cpu().numpy(), ref)
    record(f"layer_ws_w{w}_{mode}", err)
    assert err <= TOL


@pytest.mark.parametrize("d", [1008, 1024])
def test_embed_maximum_d(igp, d):
    """The largest d (include/igp.h: a multiple of 16 up to 1024): 1024 = 8 slices of 128 columns,
    1008 = 63 slices of 16 (the slice count limit is 64); ragged N, every slice checked."""
    rng = np.random.default_rng(d)
    n = 1531
    edges = rng.integers(0, n, (8 * n, 2)).astype(np.int32)
    for mode in ["full", "pre_sigmoid"]:
        z, ref = run_parity(igp, edges, n, d, 4, -1.0, seed=5, mode=mode)
        err = row_rel_err(z, ref)
        record(f"max_d{d}_{mode}", err)
        assert err <= TOL, (mode, d)


def test_embed_linear_mode(igp):
    rng = np.random.default_rng(9)
    n = 500
    edges = rng.integers(0, n, (3000, 2)).astype(np.int32)
    z, ref = run_parity(igp, edges, n, 32, 3, -0.5, seed=1, mode="linear")
    assert row_rel_err(z, ref) <= TOL


@pytest.mark.parametrize("tau", [-1.0, 0.0, 2.0])
def test_embed_isolated_nodes_and_empty_graph(igp, tau):
    rng = np.random.default_rng(4)
    n = 1000
    edges = rng.integers(0, 600, (2000, 2)).astype(np.int32)  # nodes 600..999 isolated
    z, ref = run_parity(igp, edges, n, 64, 8, tau, seed=2)
    assert row_rel_err(z, ref) <= TOL
    z, ref = run_parity(igp, np.zeros((0, 2), np.int32), 300, 16, 5, tau, seed=2)
    assert row_rel_err(z, ref) <= TOL


def test_embed_single_node_is_one_half(igp):
    z, _ = run_parity(igp, np.zeros((0, 2), np.int32), 1, 64, 4, -1.0)
    assert np.all(z == 0.5)


def test_embed_star_hub_and_theta_alpha_subsequence(igp):
    n = 5000
    e = np.stack([np.zeros(n - 1, np.int32), np.arange(1, n, dtype=np.int32)], 1)
    z, ref = run_parity(igp, e, n, 64, 10, -1.0, seed=5, sub=3, theta=0.3, alpha=0.7, eps=1e-2)
    err = row_rel_err(z, ref)
    record("star_hub_theta0.3_alpha0.7", err)
    assert err <= TOL


def test_embed_deterministic_and_stream_safe(igp):
    c = CONFIGS["tiny"]
    edges, _ = generate(c)
    g = gpu_graph(igp, edges, c.num_nodes)
    a = igp.embed(g, -1.0, 64, 10, 0).clone()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        b = igp.embed(g, -1.0, 64, 10, 0, stream=s1)
    with torch.cuda.stream(s2):
        c2 = igp.embed(g, -1.0, 64, 10, 0, stream=s2)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(a, c2)


def test_embed_host_matches_device_path(igp):
    c = CONFIGS["tiny"]
    edges, _ = generate(c)
    g = gpu_graph(igp, edges, c.num_nodes)
    dev = igp.embed(g, -1.0, 64, 10, 0).cpu()
    host = igp.embed_host(torch.from_numpy(edges).pin_memory(), c.num_nodes, -1.0, 64, 10, 0)
    assert torch.equal(dev, host)


def test_embed_argument_errors(igp):
    g = gpu_graph(igp, np.array([[0, 1]], np.int32), 2)
    for bad_d in (40, 8, 2048):  # d must be a multiple of 16 in [16, 1024]
        with pytest.raises(igp.IGPError) as ei:
            igp.embed(g, -1.0, bad_d, 3, 0)
        assert ei.value.status == 7
    with pytest.raises(igp.IGPError):
        igp.embed(g, float("nan"), 64, 3, 0)
    with pytest.raises(igp.IGPError):
        igp.embed(g, -1.0, 64, -1, 0)


# ------------------------------------------------------------------ full size (bench launch configuration)
@pytest.fixture(scope="module")
def headline(igp):
    c = CONFIGS["headline"]
    edges, _ = generate(c)
    return c, edges


def test_headline_csr_bit_exact(igp, headline):
    c, edges = headline
    check_csr(igp, edges, c.num_nodes)


def test_headline_dynamic_schedule_bit_identical(igp, headline, monkeypatch):
    """layer_kernel's dynamic row-batch schedule (atomic counters; on at the headline size,
    DESIGN.md §5) changes only which warp finishes which rows: the embedding is bit-identical to
    the static striding's (IGP_DYN=0), full size, both row orders that use it."""
    c, edges = headline
    e = torch.from_numpy(edges).cuda()
    for order in ("community", "degree"):
        g = igp.build_graph(e, c.num_nodes, order=order)
        outs = []
        for dyn in ("0", "1"):
            monkeypatch.setenv("IGP_DYN", dyn)
            outs.append(igp.embed(g, c.tau, c.d, 6, 0))
        g.close()
        assert torch.equal(outs[0], outs[1]), order


def test_dynamic_schedule_ragged_tail(igp, monkeypatch):
    """The dynamic row-batch schedule where it is on (>= 4 batches and >= 2048 CSR entries per
    warp) with a ragged N (a partial last batch) and rows of every length: bit-identical to the
    static striding, and within the tolerance of the oracle."""
    n, d, L = 300_007, 32, 3
    rng = np.random.default_rng(11)
    m = 4_000_000
    u = rng.integers(0, n, m)
    v = (u + rng.integers(1, 2000, m)) % n  # banded: neighbours near in id (community-like)
    hubs = rng.integers(0, 64, 20_000)      # a few long rows (fold path)
    edges = np.concatenate([np.stack([u, v], 1), np.stack([hubs, rng.integers(0, n, hubs.size)], 1)])
    edges = edges.astype(np.int32)
    g = gpu_graph(igp, edges, n)
    outs = []
    for dyn in ("0", "1"):
        monkeypatch.setenv("IGP_DYN", dyn)
        outs.append(igp.embed(g, -1.0, d, L, 9))
    assert torch.equal(outs[0], outs[1])
    rp, ci, _ = oracle.build_csr(edges, n)
    ref = oracle.embed(rp, ci, n, d, L, -1.0, seed=9, mode=oracle.MODE_FULL, nthreads=NTHREADS)
    err = row_rel_err(outs[1].cpu().numpy(), ref)
    record("dyn_schedule_ragged", err)
    assert err <= TOL


QUICK = os.environ.get("IGP_QUICK") == "1"  # development runs: reduced L at the full sizes
# The oracle's fp32 twin at the full headline size and L = 60 costs ~150 s of host time and gates
# nothing (it is a reported floor): opt-in.  The recorded value (4.0e-6, beside the GPU's 4.1e-6)
# is in profiles/r02/parity_gpu_full_suite.json and profiles/r02/final_s4/.
FULL_FLOORS = os.environ.get("IGP_FULL_FLOORS") == "1"


def test_headline_parity_full_steps(igp, headline):
    """The bench workload itself: full N / nnz / d / L = 60, the same kernels and grid as
    bench.py, element by element against the fp64 oracle (IGP_QUICK=1: L = 3;
    IGP_FULL_FLOORS=1 also runs the oracle's fp32 twin and records its drift)."""
    c, edges = headline
    L = 3 if QUICK else c.steps
    z, ref = run_parity(igp, edges, c.num_nodes, c.d, L, c.tau,
                        floor=f"headline_L{L}" if (FULL_FLOORS or QUICK) else None)
    err = row_rel_err(z, ref)
    record(f"headline_L{L}", err)
    assert err <= TOL


def test_headline_full_steps_properties(igp, headline):
    """L = 60 at full size: properties that hold at any size (range, determinism,
    standardised pre-sigmoid columns)."""
    c, edges = headline
    g = gpu_graph(igp, edges, c.num_nodes)
    z1 = igp.embed(g, c.tau, c.d, c.steps, 0)
    z2 = igp.embed(g, c.tau, c.d, c.steps, 0)
    assert torch.equal(z1, z2)
    assert float(z1.min()) > 0 and float(z1.max()) < 1
    pre = igp.embed(g, c.tau, c.d, c.steps, 0, mode="pre_sigmoid").double()
    assert torch.allclose(pre.mean(0), torch.zeros(c.d, dtype=torch.float64, device=pre.device), atol=1e-4)
    assert torch.allclose(pre.std(0, unbiased=False), torch.ones(c.d, dtype=torch.float64, device=pre.device),
                          atol=1e-4)


# ------------------------------------------------------------------ community row order (IGP_BUILD_REORDER_COMMUNITY)
@pytest.mark.parametrize("cfg", ["tiny", "medium"])
def test_embed_community_order(igp, cfg):
    """The label-propagation row order changes only where rows sit (and so fp32 summation
    order): the canonical CSR is unchanged and the embedding matches the oracle."""
    c = CONFIGS[cfg]
    edges, _ = generate(c)
    e = torch.from_numpy(edges).cuda()
    g = igp.build_graph(e, c.num_nodes, order="community")
    rp, ci = g.csr()
    rp_o, ci_o, _ = oracle.build_csr(edges, c.num_nodes)
    assert np.array_equal(rp.cpu().numpy(), rp_o) and np.array_equal(ci.cpu().numpy(), ci_o)
    z = igp.embed(g, c.tau, c.d, c.steps, 0).cpu().numpy()
    z2 = igp.embed(igp.build_graph(e, c.num_nodes, order="community"), c.tau, c.d, c.steps, 0).cpu().numpy()
    assert np.array_equal(z, z2)  # the order (and so the output) is deterministic
    ref = oracle.embed(rp_o, ci_o, c.num_nodes, c.d, c.steps, c.tau, seed=0, nthreads=NTHREADS)
    err = row_rel_err(z, ref)
    record(f"{cfg}_community_order", err)
    assert err <= TOL


def test_community_order_flag_conflict(igp):
    import ctypes
    h = ctypes.c_void_p()
    e = torch.zeros((1, 2), dtype=torch.int32, device="cuda")
    st = igp.lib().igp_build_graph_ex(ctypes.c_void_p(e.data_ptr()), 1, 2, igp.BUILD_NO_REORDER |
                                      igp.BUILD_REORDER_COMMUNITY, None, ctypes.byref(h))
    assert st == 2


# ------------------------------------------------------------------ row order (IGP_BUILD_NO_REORDER)
@pytest.mark.parametrize("cfg", ["tiny", "medium"])
def test_embed_without_relabelling(igp, cfg):
    """The filter steps on the original row order (no degree-sorted relabelling) meet the
    same bar; the two orders differ only by fp32 summation order."""
    c = CONFIGS[cfg]
    edges, _ = generate(c)
    e = torch.from_numpy(edges).cuda()
    g0 = igp.build_graph(e, c.num_nodes, reorder=False)
    g1 = igp.build_graph(e, c.num_nodes)
    rp0, ci0 = g0.csr()
    rp1, ci1 = g1.csr()
    assert torch.equal(rp0, rp1) and torch.equal(ci0, ci1)  # the canonical CSR is the same
    z0 = igp.embed(g0, c.tau, c.d, c.steps, 0).cpu().numpy()
    z1 = igp.embed(g1, c.tau, c.d, c.steps, 0).cpu().numpy()
    rp, ci, _ = oracle.build_csr(edges, c.num_nodes)
    ref = oracle.embed(rp, ci, c.num_nodes, c.d, c.steps, c.tau, seed=0, nthreads=NTHREADS)
    err0 = row_rel_err(z0, ref)
    record(f"{cfg}_no_reorder", err0)
    assert err0 <= TOL
    assert row_rel_err(z0, z1) <= TOL


def test_build_flags_rejected(igp):
    import ctypes
    h = ctypes.c_void_p()
    e = torch.zeros((1, 2), dtype=torch.int32, device="cuda")
    st = igp.lib().igp_build_graph_ex(ctypes.c_void_p(e.data_ptr()), 1, 2, 0x80, None, ctypes.byref(h))
    assert st == 2


# ------------------------------------------------------------------ streaming (device CSR merge, Alg. 2 l.1-7)
def test_streaming_merge_csr_bit_exact_and_embed(igp):
    """Stage t's graph = union of batches 0..t (uniform edge sampling, 10 stages).
    igp_graph_add_edges must give the canonical CSR of the cumulative edge list after
    every stage, and the stage's re-embed (fresh Philox subsequence t, Alg. 2 l.3)
    matches the oracle on the cumulative graph."""
    from synth.dcsbm import stream_batches
    c = CONFIGS["streaming"]
    edges, _ = generate(c)
    batches = stream_batches(edges, 10)
    g = None
    cum = []
    for t, b in enumerate(batches):
        cum.append(b)
        eb = torch.from_numpy(b).cuda()
        if g is None:
            g = igp.build_graph(eb, c.num_nodes)
        else:
            g.add_edges(eb)
        rp, ci = g.csr()
        torch.cuda.synchronize()
        allc = np.concatenate(cum)
        rp_o, ci_o, m_o = oracle.build_csr(allc, c.num_nodes)
        assert g.num_edges == m_o
        assert np.array_equal(rp.cpu().numpy(), rp_o) and np.array_equal(ci.cpu().numpy(), ci_o), f"stage {t}"
        if t in (0, 4, 9):
            z = igp.embed(g, c.tau, c.d, c.steps, 0, subsequence=t).cpu().numpy()
            ref = oracle.embed(rp_o, ci_o, c.num_nodes, c.d, c.steps, c.tau, seed=0, sub=t, nthreads=NTHREADS)
            err = row_rel_err(z, ref)
            record(f"streaming_stage{t}", err)
            assert err <= TOL


def test_add_edges_errors_leave_graph_unchanged(igp):
    g = gpu_graph(igp, np.array([[0, 1], [1, 2]], np.int32), 4)
    with pytest.raises(igp.IGPError):
        g.add_edges(torch.tensor([[0, 9]], dtype=torch.int32, device="cuda"))
    rp, ci = g.csr()
    assert rp.cpu().tolist() == [0, 1, 3, 4, 4] and ci.cpu().tolist() == [1, 0, 2, 1]
    g.add_edges(torch.tensor([[3, 0], [0, 1]], dtype=torch.int32, device="cuda"))  # one new, one duplicate
    rp, ci = g.csr()
    assert rp.cpu().tolist() == [0, 2, 4, 5, 6] and ci.cpu().tolist() == [1, 3, 0, 2, 1, 0]
    g.add_edges(torch.zeros((0, 2), dtype=torch.int32, device="cuda"))
    assert g.num_edges == 3


# ------------------------------------------------------------------ asynchronous build / release, layer timer
def test_async_build_same_csr_and_embed(igp):
    """IGP_BUILD_ASYNC enqueues the whole build with no host sync: the CSR and the embed
    behind it are identical to the synchronous build's."""
    c = CONFIGS["medium"]
    edges, _ = generate(c)
    e = torch.from_numpy(edges).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ga = igp.build_graph(e, c.num_nodes, stream=s, async_build=True)
        za = igp.embed(ga, c.tau, c.d, 5, 0, stream=s)
        rpa, cia = ga.csr(stream=s)
    s.synchronize()
    gs = igp.build_graph(e, c.num_nodes)
    zs = igp.embed(gs, c.tau, c.d, 5, 0)
    rps, cis = gs.csr()
    torch.cuda.synchronize()
    assert ga.nnz == gs.nnz
    assert torch.equal(rpa, rps) and torch.equal(cia, cis)
    assert torch.equal(za, zs)  # bitwise: same kernels, same order
    ga.close(stream=s)
    gs.close()


def test_async_build_reports_range_error_lazily(igp):
    e = torch.tensor([[0, 1], [2, 7], [1, 2]], dtype=torch.int32, device="cuda")
    g = igp.build_graph(e, 5, async_build=True)  # returns before the range check is read
    with pytest.raises(igp.IGPError) as ei:
        g.status()
    assert ei.value.status == 2
    with pytest.raises(igp.IGPError):
        _ = g.nnz
    g.close(stream=torch.cuda.current_stream())
    # an asynchronous merge of a bad batch is reported the same way
    g = igp.build_graph(torch.tensor([[0, 1]], dtype=torch.int32, device="cuda"), 4, async_build=True)
    g.status()
    g.add_edges(torch.tensor([[0, 9]], dtype=torch.int32, device="cuda"))
    with pytest.raises(igp.IGPError):
        g.status()
    g.close()


def test_async_streaming_merge_matches_oracle(igp):
    """The streaming config's 10 merges, all asynchronous (no host sync until the end)."""
    from synth.dcsbm import stream_batches
    c = CONFIGS["streaming"]
    edges, _ = generate(c)
    batches = [torch.from_numpy(b).cuda() for b in stream_batches(edges, 10)]
    g = igp.build_graph(batches[0], c.num_nodes, async_build=True)
    for b in batches[1:]:
        g.add_edges(b)
    rp, ci = g.csr()
    rp_o, ci_o, m_o = oracle.build_csr(edges, c.num_nodes)
    assert g.num_edges == m_o
    assert np.array_equal(rp.cpu().numpy(), rp_o) and np.array_equal(ci.cpu().numpy(), ci_o)
    g.close()


def test_layer_timer_accumulates_without_sync(igp):
    c = CONFIGS["tiny"]
    edges, _ = generate(c)
    e = torch.from_numpy(edges).cuda()
    igp.layer_timer_reset()
    assert igp.layer_timer_read() == (0.0, 0)
    s = torch.cuda.current_stream()
    for k in range(3):
        g = igp.build_graph(e, c.num_nodes, stream=s, async_build=True)
        igp.embed(g, c.tau, c.d, c.steps, k, stream=s, time_layers=True)
        g.close(stream=s)
    ms, launches = igp.layer_timer_read()
    assert launches % c.steps == 0  # L launches per timed column slice
    assert launches >= 3 * c.steps and ms > 0.0
    igp.layer_timer_reset()
    assert igp.layer_timer_read() == (0.0, 0)


# ------------------------------------------------------------------ Large config (5M nodes, d = 128)
@pytest.fixture(scope="module")
def large(igp):
    c = CONFIGS["large"]
    edges, _ = generate(c)
    return c, edges


def test_large_csr_bit_exact(igp, large):
    c, edges = large
    check_csr(igp, edges, c.num_nodes)


def test_large_parity_reduced_steps(igp, large):
    """Full N = 5M / nnz ~ 200M / d = 128 with the bench's kernels and grid; L = 5 (SURVEY.md
    §8(d): the fp64 oracle does ~10x the headline's work per layer)."""
    c, edges = large
    L = 2 if QUICK else 5
    z, ref = run_parity(igp, edges, c.num_nodes, c.d, L, c.tau)
    err = row_rel_err(z, ref)
    record(f"large_L{L}", err)
    assert err <= TOL


def test_large_full_steps_with_and_without_reordering(igp, large):
    """L = 60 at full size with the community order (the default here), the degree-sorted
    relabelling and no relabelling (config 5): every run is deterministic, in (0, 1),
    standardised before the sigmoid, and they agree with each other to the parity tolerance
    (they differ only in fp32 summation order)."""
    c, edges = large
    e = torch.from_numpy(edges).cuda()
    zs = []
    for order in ("community", "degree", "none"):
        g = igp.build_graph(e, c.num_nodes, order=order)
        z1 = igp.embed(g, c.tau, c.d, c.steps, 0)
        z2 = igp.embed(g, c.tau, c.d, c.steps, 0)
        assert torch.equal(z1, z2)
        assert float(z1.min()) > 0 and float(z1.max()) < 1
        pre = igp.embed(g, c.tau, c.d, c.steps, 0, mode="pre_sigmoid").double()
        assert torch.allclose(pre.mean(0), torch.zeros(c.d, dtype=torch.float64, device=pre.device), atol=1e-4)
        assert torch.allclose(pre.std(0, unbiased=False), torch.ones(c.d, dtype=torch.float64, device=pre.device),
                              atol=1e-4)
        del pre
        g.close()
        zs.append(z1.cpu().numpy())
        del z1, z2
    for name, z in (("degree", zs[1]), ("none", zs[2])):
        err = row_rel_err(z, zs[0].astype(np.float64))
        record(f"large_L60_{name}_vs_community", err)
        assert err <= TOL


# ------------------------------------------------------------------ the paper's own settings (Table II)
@pytest.mark.parametrize("cfg", ["paper_5k", "paper_10k"])
def test_paper_settings_full_parity(igp, cfg):
    """Table II: N=5K tau=-6 L=10 d=64 and N=10K tau=-3 L=9 d=64 on DC-SBM
    graphs of Table I's shape; full-L parity at the north-star bar."""
    from synth.dcsbm import PAPER_CONFIGS
    c = PAPER_CONFIGS[cfg]
    edges, _ = generate(c)
    z, ref = run_parity(igp, edges, c.num_nodes, c.d, c.steps, c.tau, floor=cfg)
    err = row_rel_err(z, ref)
    record(cfg, err)
    assert err <= TOL


FLOOR_MARGIN = 2.0  # DESIGN.md reading A16: the GPU error may not exceed twice the fp32-twin floor


@pytest.mark.parametrize("cfg", ["paper_50k", "paper_stream_100k", "paper_1m"])
def test_paper_settings_chaotic_tau_layerwise(igp, cfg):
    """Table II's tau = -80 / -100 clamp every node of degree <= |tau| to D = eps (Eq. (1)), so
    s^2 = 1/eps = 1000 and each layer amplifies fp32 rounding ~10^3 times: the fp32 and fp64
    trajectories separate after 2-3 layers (reading A16).  Checked instead: layer 1 from the
    exact Philox input at the 1e-4 bar; one layer from seeded layer states Z (synth/states.py,
    generic and tanh-saturated shapes; the same fp32 values go to the CUDA path via d_z0 and to
    the oracle via Z0) at FLOOR_MARGIN x the oracle's fp32-twin error on the same state (measured:
    the GPU error equals that floor to 5 digits, so it is fp32 itself, not the kernel's deferred
    z-score algebra); full-L properties."""
    from synth.dcsbm import PAPER_CONFIGS
    from synth.states import layer_state
    c = PAPER_CONFIGS[cfg]
    edges, _ = generate(c)
    e = torch.from_numpy(edges).cuda()
    g = igp.build_graph(e, c.num_nodes)
    rp, ci, _ = oracle.build_csr(edges, c.num_nodes)
    z1 = igp.embed(g, c.tau, c.d, 1, 0).cpu().numpy()
    ref1 = oracle.embed(rp, ci, c.num_nodes, c.d, 1, c.tau, seed=0, nthreads=NTHREADS)
    err1 = row_rel_err(z1, ref1)
    record(f"{cfg}_L1", err1)
    assert err1 <= TOL
    for k, kind in enumerate(("normal", "bimodal")):
        zs = layer_state(c.num_nodes, c.d, seed=100 + k, kind=kind)
        for mode, om in (("full", oracle.MODE_FULL), ("pre_sigmoid", oracle.MODE_PRE_SIGMOID)):
            zl = igp.embed(g, c.tau, c.d, 1, 0, mode=mode, z0=torch.from_numpy(zs).cuda()).cpu().numpy()
            ref = oracle.embed(rp, ci, c.num_nodes, c.d, 1, c.tau, Z0=zs.astype(np.float64), mode=om,
                               nthreads=NTHREADS)
            twin = oracle.embed(rp, ci, c.num_nodes, c.d, 1, c.tau, Z0=zs.astype(np.float64), mode=om,
                                nthreads=NTHREADS, fp32_twin=True)
            err = row_rel_err(zl, ref)
            floor = row_rel_err(twin, ref)
            record(f"{cfg}_one_layer_from_{kind}_state_{mode}", err)
            record(f"{cfg}_one_layer_from_{kind}_state_{mode}_fp32_floor", floor)
            assert err <= max(TOL, FLOOR_MARGIN * floor), (kind, mode, err, floor)
    za = igp.embed(g, c.tau, c.d, c.steps, 0)
    zb = igp.embed(g, c.tau, c.d, c.steps, 0)
    assert torch.equal(za, zb)
    assert float(za.min()) > 0 and float(za.max()) < 1
    pre = igp.embed(g, c.tau, c.d, c.steps, 0, mode="pre_sigmoid").double()
    assert torch.allclose(pre.mean(0), torch.zeros(c.d, dtype=torch.float64, device=pre.device), atol=1e-4)
    assert torch.allclose(pre.std(0, unbiased=False), torch.ones(c.d, dtype=torch.float64, device=pre.device),
                          atol=1e-4)
    g.close()


# ------------------------------------------------------------------ downstream sanity report (not a gate)
@pytest.mark.parametrize("cfg", ["medium", "paper_5k"])
def test_birch_sanity_report(igp, cfg):
    """north_star: 'as a sanity report only, both embeddings fed to the same CPU BIRCH must give
    an equal NMI against the planted blocks' (Alg. 1 l.7; sklearn Birch, K-agnostic,
    threshold 1.0 -- the paper does not state its threshold).  BIRCH's threshold
    decisions can flip on 1e-5 perturbations, so 'equal' is checked to 0.02 and both recorded."""
    from sklearn.cluster import Birch
    from sklearn.metrics import adjusted_rand_score, normalized_mutual_info_score
    from synth.dcsbm import ALL_CONFIGS
    c = ALL_CONFIGS[cfg]
    edges, labels = generate(c)
    z, ref = run_parity(igp, edges, c.num_nodes, c.d, c.steps, c.tau)
    scores = {}
    for name, emb in (("gpu", z.astype(np.float64)), ("oracle", ref)):
        pred = Birch(n_clusters=None, threshold=1.0).fit_predict(emb)
        scores[name] = (normalized_mutual_info_score(labels, pred), adjusted_rand_score(labels, pred))
        record(f"{cfg}_birch_{name}_nmi", scores[name][0])
        record(f"{cfg}_birch_{name}_ari", scores[name][1])
    assert scores["oracle"][0] > 0.5  # the embedding carries the planted blocks at all
    assert abs(scores["gpu"][0] - scores["oracle"][0]) <= 0.02


def test_concurrent_host_threads(igp):
    """Two host threads, each with its own stream, build and embed different graphs at the same
    time (thread-safe handles, pools, caches and error strings): results equal the sequential run."""
    import threading
    cfgs = [CONFIGS["tiny"], CONFIGS["medium"]]
    inputs = [torch.from_numpy(generate(c)[0]).cuda() for c in cfgs]
    seq = []
    for c, e in zip(cfgs, inputs):
        g = igp.build_graph(e, c.num_nodes)
        seq.append(igp.embed(g, c.tau, c.d, c.steps, 3).cpu())
        g.close()
    out = [None, None]
    errs = []

    def work(k):
        try:
            c, e = cfgs[k], inputs[k]
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    g = igp.build_graph(e, c.num_nodes, stream=s, async_build=True)
                    z = igp.embed(g, c.tau, c.d, c.steps, 3, stream=s)
                    g.close(stream=s)
                s.synchronize()
                out[k] = z.cpu()
        except Exception as ex:  # surfaced below
            errs.append(ex)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for k in range(2):
        assert torch.equal(out[k], seq[k])


# ------------------------------------------------------------------ optional row-L2 post-op (IGP_FLAG_ROW_L2, reading A12)
@pytest.mark.parametrize("cfg,d", [("tiny", 16), ("tiny", 128), ("medium", 64)])
def test_row_l2_flag(igp, cfg, d):
    """Off by default (the paper ends with the sigmoid); with the flag each output row is the
    oracle's sigmoid row scaled to unit L2 norm.  Also through the host-buffer path."""
    c = CONFIGS[cfg]
    edges, _ = generate(c)
    g = gpu_graph(igp, edges, c.num_nodes)
    z = igp.embed(g, c.tau, d, c.steps, 0, row_l2=True).cpu().numpy()
    rp, ci, _ = oracle.build_csr(edges, c.num_nodes)
    ref = oracle.row_l2(oracle.embed(rp, ci, c.num_nodes, d, c.steps, c.tau, seed=0, nthreads=NTHREADS))
    err = row_rel_err(z, ref)
    record(f"{cfg}_d{d}_row_l2", err)
    assert err <= TOL
    assert np.allclose(np.linalg.norm(z.astype(np.float64), axis=1), 1.0, atol=1e-6)
    if cfg == "tiny":
        host = igp.embed_host(torch.from_numpy(edges).pin_memory(), c.num_nodes, c.tau, d, c.steps, 0,
                              row_l2=True).numpy()
        assert np.array_equal(host, z)


def test_embed_unknown_flags_rejected(igp):
    import ctypes
    g = gpu_graph(igp, np.array([[0, 1]], np.int32), 2)
    o = igp.make_opts(-1.0, 16, 2)
    o.flags = 0x100
    out = torch.empty((2, 16), device="cuda")
    assert igp.lib().igp_embed_ex(g.handle, ctypes.byref(o), ctypes.c_void_p(out.data_ptr()), None) == 2


@pytest.mark.parametrize("L", [0, 1])
def test_embed_zero_and_one_step(igp, L):
    """L = 0: the output is sigmoid(Theta) (Alg. 1 with an empty layer loop); L = 1: one layer."""
    c = CONFIGS["tiny"]
    edges, _ = generate(c)
    for mode in ("full", "pre_sigmoid", "linear"):
        z, ref = run_parity(igp, edges, c.num_nodes, 32, L, c.tau, seed=11, mode=mode)
        err = row_rel_err(z, ref)
        record(f"tiny_L{L}_{mode}", err)
        assert err <= TOL, mode


def test_plain_c_consumer(igp):
    """The C ABI used from C alone (examples/embed_c.c): host and device paths agree bitwise,
    outputs in (0, 1), pre-sigmoid columns standardised."""
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples", "embed_c")
    for args in (["3000", "30000", "64", "10"], ["777", "5000", "16", "3"], ["20000", "400000", "128", "5"]):
        res = subprocess.run([exe, *args], capture_output=True, text=True, timeout=300)
        assert res.returncode == 0, res.stderr
        assert res.stdout.startswith("ok "), res.stdout


def test_bitwise_reproducible_across_processes(igp):
    """Same graph, arguments and seed give bitwise-identical embeddings in a fresh process
    (no dependence on allocation addresses, scheduling or atomics order)."""
    import hashlib
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, hashlib, torch; sys.path.insert(0, %r); import paper_2508_19737_b200 as igp; "
            "from synth.dcsbm import CONFIGS, generate; c = CONFIGS['medium']; "
            "e = torch.from_numpy(generate(c)[0]).cuda(); g = igp.build_graph(e, c.num_nodes); "
            "z = igp.embed(g, c.tau, c.d, 12, 5).cpu().numpy(); print(hashlib.sha256(z.tobytes()).hexdigest())" % root)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    c = CONFIGS["medium"]
    e = torch.from_numpy(generate(c)[0]).cuda()
    g = igp.build_graph(e, c.num_nodes)
    z = igp.embed(g, c.tau, c.d, 12, 5).cpu().numpy()
    assert hashlib.sha256(z.tobytes()).hexdigest() == out.stdout.strip()


@pytest.mark.parametrize("cfg", ["tiny", "medium"])
def test_initial_state_hook(igp, cfg):
    """igp_embed_opts.d_z0: a caller-provided Z^(0) (seeded, synth/states.py) replaces Theta;
    row i of z0 is node id i whatever the internal row order.  Several layers at the 1e-4 bar."""
    from synth.states import layer_state
    c = CONFIGS[cfg]
    edges, _ = generate(c)
    zs = layer_state(c.num_nodes, c.d, seed=7)
    rp, ci, _ = oracle.build_csr(edges, c.num_nodes)
    e = torch.from_numpy(edges).cuda()
    for order in ("degree", "community", "none"):
        g = igp.build_graph(e, c.num_nodes, order=order)
        z = igp.embed(g, c.tau, c.d, 5, 0, z0=torch.from_numpy(zs).cuda()).cpu().numpy()
        ref = oracle.embed(rp, ci, c.num_nodes, c.d, 5, c.tau, Z0=zs.astype(np.float64), nthreads=NTHREADS)
        err = row_rel_err(z, ref)
        record(f"{cfg}_z0_{order}", err)
        assert err <= TOL, order
        g.close()


@pytest.mark.parametrize("tau,theta,alpha,L", [(-1.0, 0.1, 1.0, 200),   # many layers: no drift to NaN/inf
                                               (1e6, 0.1, 1.0, 10),     # huge positive correction: s ~ 1e-3
                                               (-1.0, 0.0, 0.0, 5),     # phi* = 0: constant columns -> 0.5
                                               (-1.0, 1.0, -1.0, 8),    # alpha < 0 (Eq. (2) allows [-1, 1])
                                               (-2.5, 0.0, 1.0, 8)])    # no self term
def test_parameter_extremes(igp, tau, theta, alpha, L):
    c = CONFIGS["tiny"]
    edges, _ = generate(c)
    z, ref = run_parity(igp, edges, c.num_nodes, 32, L, tau, seed=9, theta=theta, alpha=alpha)
    assert np.all(np.isfinite(z))
    err = row_rel_err(z, ref)
    record(f"extreme_tau{tau}_theta{theta}_alpha{alpha}_L{L}", err)
    assert err <= TOL


@pytest.mark.parametrize("case", ["empty", "star", "two_cliques_bridge", "ragged"])
def test_community_order_adversarial(igp, case):
    """The label-propagation order on graphs where communities are degenerate (no edges, one hub,
    two dense blocks, random): canonical CSR unchanged, embeddings match the oracle."""
    rng = np.random.default_rng(4)
    if case == "empty":
        n, edges = 300, np.zeros((0, 2), np.int32)
    elif case == "star":
        n = 3000
        edges = np.stack([np.zeros(n - 1, np.int32), np.arange(1, n, dtype=np.int32)], 1)
    elif case == "two_cliques_bridge":
        a = np.array([(i, j) for i in range(40) for j in range(i + 1, 40)], np.int32)
        edges = np.concatenate([a, a + 40, [[0, 40]]]).astype(np.int32)
        n = 80
    else:
        n = 2049
        edges = rng.integers(0, n, (9000, 2)).astype(np.int32)
    e = torch.from_numpy(np.ascontiguousarray(edges)).cuda()
    g = igp.build_graph(e, n, order="community")
    rp, ci = g.csr()
    rp_o, ci_o, _ = oracle.build_csr(edges, n)
    assert np.array_equal(rp.cpu().numpy(), rp_o) and np.array_equal(ci.cpu().numpy(), ci_o)
    z = igp.embed(g, -1.0, 32, 8, 2).cpu().numpy()
    ref = oracle.embed(rp_o, ci_o, n, 32, 8, -1.0, seed=2, nthreads=NTHREADS)
    err = row_rel_err(z, ref)
    record(f"community_{case}", err)
    assert err <= TOL


def test_streaming_merges_in_community_order(igp):
    """igp_graph_add_edges keeps the graph's row order mode: merges of a community-ordered graph
    stay canonical and embed like the oracle."""
    from synth.dcsbm import stream_batches
    c = CONFIGS["medium"]
    edges, _ = generate(c)
    batches = stream_batches(edges, 4)
    g = igp.build_graph(torch.from_numpy(batches[0]).cuda(), c.num_nodes, order="community")
    for b in batches[1:]:
        g.add_edges(torch.from_numpy(b).cuda())
    rp, ci = g.csr()
    rp_o, ci_o, _ = oracle.build_csr(edges, c.num_nodes)
    assert np.array_equal(rp.cpu().numpy(), rp_o) and np.array_equal(ci.cpu().numpy(), ci_o)
    z = igp.embed(g, c.tau, c.d, 10, 0).cpu().numpy()
    ref = oracle.embed(rp_o, ci_o, c.num_nodes, c.d, 10, c.tau, seed=0, nthreads=NTHREADS)
    err = row_rel_err(z, ref)
    record("streaming_community_merged", err)
    assert err <= TOL


# ------------------------------------------------------------------ maximum CSR size
def test_maximum_csr_size_circulant(igp):
    """The largest graph the int32 CSR admits (include/igp.h: 2E <= INT32_MAX - 64): the circulant
    C_n(1..32) with n = 2^25 - 2 has 2E = 64n = 2^31 - 128 directed entries (synth/circulant.py).
    CSR: bit-exact on every row against its closed form.  One LINEAR filter step (Eq. 3):
    sampled rows against oracle.propagate over each row's neighbourhood with the oracle's own
    Philox inputs.  Two FULL layers: the ZNorm properties (column mean 0, population std 1) that
    hold at any size."""
    from synth.circulant import circulant_edges, circulant_row
    k, n = 32, 2**25 - 2
    assert 2 * n * k <= 2**31 - 1 - 64
    e = circulant_edges(n, k, "cuda")
    g = igp.build_graph(e, n)
    del e
    assert g.nnz == 2 * n * k and g.num_edges == n * k
    rp, ci = g.csr()
    assert torch.equal(rp, torch.arange(n + 1, device="cuda", dtype=torch.int32) * (2 * k))
    ci2 = ci.view(n, 2 * k)
    offs = torch.cat([torch.arange(-k, 0), torch.arange(1, k + 1)]).to(device="cuda", dtype=torch.int32)
    step = 1 << 22
    for r0 in range(k, n - k, step):
        r1 = min(r0 + step, n - k)
        rows = torch.arange(r0, r1, device="cuda", dtype=torch.int32)
        assert torch.equal(ci2[r0:r1] - rows[:, None], offs.expand(r1 - r0, -1)), f"rows {r0}..{r1}"
    wrap = list(range(k)) + list(range(n - k, n))
    ci_w = ci2[wrap].cpu().numpy()
    for t, i in enumerate(wrap):
        assert np.array_equal(ci_w[t], circulant_row(n, k, i)), f"row {i}"
    del rp, ci, ci2

    d, tau, seed = 16, -1.0, 3
    z = igp.embed(g, tau, d, 1, seed, mode="linear")
    sample = np.concatenate([[0, 1, k, n // 2, n - k - 1, n - 1], np.random.default_rng(0).integers(0, n, 10)])
    zs = z[torch.from_numpy(sample).cuda()].cpu().numpy().astype(np.float64)
    del z
    Dt = oracle.corrected_degree([2 * k], tau)[0]
    rp_l = np.array([0] + [2 * k] * (2 * k + 1), np.int32)  # row 0 = the sampled node, others empty
    ci_l = np.arange(1, 2 * k + 1, dtype=np.int32)
    worst = 0.0
    for t, i in enumerate(sample):
        ids = np.concatenate([[i], circulant_row(n, k, int(i))]).astype(np.int64)
        X = oracle.normal_at(seed, 0, (ids[:, None] * d + np.arange(d)[None, :]).ravel()).reshape(-1, d)
        P = oracle.propagate(rp_l, ci_l, np.full(ids.size, Dt), X / np.sqrt(d))[0]
        worst = max(worst, float(np.max(np.abs(zs[t] - P)) / np.linalg.norm(P)))
    record("max_size_linear_sampled", worst)
    assert worst <= 1e-5, worst

    zp = igp.embed(g, tau, d, 2, seed, mode="pre_sigmoid").double()
    mu, sd = zp.mean(0), zp.std(0, correction=0)
    assert float(mu.abs().max()) < 1e-5 and float((sd - 1).abs().max()) < 1e-5, (mu, sd)
    del zp
    zf = igp.embed(g, tau, d, 2, seed)
    assert float(zf.min()) > 0.0 and float(zf.max()) < 1.0
    g.close()


# ------------------------------------------------------------------ round-2 boundary additions (§8(b))
def test_embed_sample_std_ddof(igp):
    """igp_embed_opts.ddof = 1 (sample std in ZNorm, the other reading of PAPER.md:166) against
    the oracle with the same ddof; ddof = 0 and 1 really differ."""
    c = CONFIGS["tiny"]
    edges, _ = generate(c)
    z1, ref1 = run_parity(igp, edges, c.num_nodes, c.d, c.steps, c.tau, ddof=1)
    err = row_rel_err(z1, ref1)
    record("tiny_ddof1", err)
    assert err <= TOL
    z0, _ = run_parity(igp, edges, c.num_nodes, c.d, c.steps, c.tau)
    assert np.abs(z1 - z0).max() > 1e-6


def test_embed_rejects_misaligned_buffers(igp):
    c = CONFIGS["tiny"]
    edges, _ = generate(c)
    g = gpu_graph(igp, edges, c.num_nodes)
    buf = torch.empty(c.num_nodes * c.d + 4, dtype=torch.float32, device="cuda")
    with pytest.raises(igp.IGPError):
        igp.embed(g, c.tau, c.d, 2, 0, out=buf[1:1 + c.num_nodes * c.d].view(c.num_nodes, c.d))
    z0 = torch.zeros(c.num_nodes * c.d + 4, dtype=torch.float32, device="cuda")[2:2 + c.num_nodes * c.d]
    with pytest.raises(igp.IGPError):
        igp.embed(g, c.tau, c.d, 2, 0, z0=z0.view(c.num_nodes, c.d))
    g.close()


def test_copy_csr_degrees(igp):
    c = CONFIGS["tiny"]
    edges, _ = generate(c)
    g = gpu_graph(igp, edges, c.num_nodes)
    rp, ci, deg = g.csr(degrees=True)
    torch.cuda.synchronize()
    rp_o, ci_o, _ = oracle.build_csr(edges, c.num_nodes)
    assert np.array_equal(deg.cpu().numpy(), np.diff(rp_o))
    g.close()


def test_destroy_waits_for_embeds_on_other_streams_and_trim(igp):
    """igp_destroy_graph waits for the graph's own uses (embeds on any stream), not the device:
    destroying right after enqueueing an embed on a side stream leaves that embed intact."""
    c = CONFIGS["medium"]
    edges, _ = generate(c)
    g = gpu_graph(igp, edges, c.num_nodes)
    ref = igp.embed(g, c.tau, c.d, 5, 0).clone()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        z = igp.embed(g, c.tau, c.d, 5, 0, stream=side)
    g.close()  # must not free the CSR under the side-stream embed
    side.synchronize()
    assert torch.equal(z, ref)
    igp.trim_memory()
