"""GPU BIRCH (igp_birch_*, csrc/birch.cu) against the oracle's BIRCH (oracle/birch_oracle.c).

The bar: bit-exact.  Both sides build the CF tree by the same sequential insertions with the
same fp64 operation order (readings B1-B6), so the clusters (n, LS, SS, centroid,
|centroid|^2 of every leaf entry, in label order) and every predicted label must be
identical, not merely close.  Inputs are the same fp32 values on both sides (the GPU widens
them to fp64 exactly; the oracle receives the widened values).
"""
import numpy as np
import pytest
import torch

import oracle
from conftest import record
from synth.dcsbm import CONFIGS, generate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def igp():
    if not torch.cuda.is_available():
        pytest.fail("GPU test requires CUDA (no CPU fallback)")
    import paper_2508_19737_b200 as m
    return m


@pytest.fixture(scope="module")
def headline(igp):
    c = CONFIGS["headline"]
    edges, _ = generate(c)
    return c, edges


def f32(X):
    return np.ascontiguousarray(np.asarray(X, dtype=np.float32))


def check_same_tree(igp, X, T, B, pieces=1):
    """fit (in `pieces` partial fits) on both sides; clusters and labels bit-identical."""
    X = f32(X)
    n, d = X.shape
    g = igp.Birch(d, T, B)
    o = oracle.Birch(d, T, B)
    cuts = np.linspace(0, n, pieces + 1).astype(int)
    Xg = torch.from_numpy(X).cuda()
    for a, b in zip(cuts[:-1], cuts[1:]):
        g.partial_fit(Xg[a:b])
        o.partial_fit(X[a:b].astype(np.float64))
        if pieces > 1:  # the cached cluster list is rebuilt after every fit
            assert g.info()[0] == o.clusters()[0].shape[0]
            assert np.array_equal(g.clusters()[0].cpu().numpy(), o.clusters()[0])
    K, dep, nodes, pts = g.info()
    ocen, osqn, on, ols, oss = o.clusters()
    assert K == ocen.shape[0] and pts == n
    odep, onodes, opts = o.shape()
    assert dep == odep and nodes == onodes
    cen, sqn, cnt, ls, ss = (t.cpu().numpy() for t in g.clusters())
    for name, a, b in (("n", cnt, on), ("LS", ls, ols), ("SS", ss, oss), ("centroid", cen, ocen), ("sqn", sqn, osqn)):
        assert np.array_equal(a, b), f"{name} differs (max |diff| {np.abs(a - b).max():.3e})"
    olab = oracle.birch_predict(ocen, osqn, X.astype(np.float64))
    lab = g.predict(Xg, path="fp64").cpu().numpy()
    assert np.array_equal(lab, olab)
    if tensor_eligible(d):  # the tensor-core search, certified: the same labels
        lab, amb = g.predict(Xg, path="tensor", return_ambiguous=True)
        assert np.array_equal(lab.cpu().numpy(), olab)
        record(f"birch_tc_ambiguous_{n}x{d}_K{K}", amb)
    g.close()
    return K, dep


def tensor_eligible(d):
    return d % 8 == 0 and 8 <= d <= 64


def datasets():
    rng = np.random.default_rng(11)
    C = rng.random((12, 8))
    return [
        ("blobs8", C[rng.integers(0, 12, 2000)] + rng.normal(0, 0.05, (2000, 8)), 0.1, 50),
        ("uniform_deep_B3", rng.random((1500, 8)), 0.01, 3),  # every point a leaf entry; many splits
        ("sigmoid64_T1", 1 / (1 + np.exp(-rng.normal(0, 1, (3000, 64)))), 1.0, 50),
        ("sigmoid64_T05_B10", 1 / (1 + np.exp(-rng.normal(0, 1, (2000, 64)))), 0.5, 10),
        ("sigmoid16_B5", 1 / (1 + np.exp(-rng.normal(0, 1, (3000, 16)))), 0.3, 5),
        ("odd_width_d37", 1 / (1 + np.exp(-rng.normal(0, 1, (1200, 37)))), 0.4, 7),
        ("wide_d200_B63", rng.random((800, 200)), 2.0, 63),
        ("wide_d256", rng.random((700, 256)), 3.0, 20),     # predict: fewer rows per block
        ("max_d1024", rng.random((300, 1024)), 6.0, 10),    # predict rows from global memory; no shared pool
        ("single_point", np.array([[0.25, -0.5, 0.75]]), 0.5, 50),
        ("duplicates", np.repeat(rng.random((5, 6)), 40, axis=0), 0.05, 4),
    ]


@pytest.mark.parametrize("name,X,T,B", datasets(), ids=[d[0] for d in datasets()])
def test_birch_bit_exact(igp, name, X, T, B):
    K, dep = check_same_tree(igp, X, T, B)
    record(f"birch_{name}_K", K)


def test_birch_partial_fit_pieces_and_pool_growth(igp):
    """Alg. 2 l.9: partial fits in stages equal the oracle's; the uniform B = 3 case outgrows the
    initial pools (1024 entries / 256 nodes) several times."""
    rng = np.random.default_rng(5)
    X = rng.random((6000, 8))
    K, dep = check_same_tree(igp, X, 0.005, 3, pieces=7)
    assert K > 4000 and dep >= 6


def test_birch_on_embeddings_medium(igp):
    """The paper's pipeline at the Medium config: GPU embed (Alg. 1 l.1-6), then BIRCH on the
    same fp32 rows on both sides (T = 1.0, B = 50, reading B1)."""
    c = CONFIGS["medium"]
    edges, labels = generate(c)
    e = torch.from_numpy(edges).cuda()
    g = igp.build_graph(e, c.num_nodes)
    Z = igp.embed(g, c.tau, c.d, c.steps, c.seed).cpu().numpy()
    K, dep = check_same_tree(igp, Z, 1.0, 50)
    record("birch_medium_T1_K", K)
    K2, dep2 = check_same_tree(igp, Z[:8000], 0.5, 50)  # the library default threshold: many clusters
    record("birch_medium8k_T05_K", K2)


def fit_clusters(igp, X, T, B):
    """fit on both sides (bit-exact trees are checked elsewhere); returns (gpu tree, centroids, sqn)"""
    g = igp.Birch(X.shape[1], T, B).partial_fit(torch.from_numpy(f32(X)).cuda())
    o = oracle.Birch(X.shape[1], T, B).fit(f32(X).astype(np.float64))
    ocen, osqn = o.clusters()[:2]
    return g, ocen, osqn


def test_birch_tensor_predict_ties_fall_back_to_fp64(igp):
    """Rows exactly between two clusters (and duplicate centroids) cannot be certified by the
    tensor-core pass (gap 0 < 2M): they are listed and solved in fp64; the labels are the
    oracle's first minimum."""
    rng = np.random.default_rng(3)
    C = np.round(rng.random((40, 16)) * 8) / 8  # dyadic values: midpoints and distances are exact
    X = np.concatenate([C, C[:5]])  # duplicates collapse into the same leaf entries
    g, ocen, osqn = fit_clusters(igp, X, 1e-3, 50)
    assert ocen.shape[0] == 40
    Q = np.concatenate([(C[:-1] + C[1:]) / 2, C, rng.random((300, 16))])
    Qg = torch.from_numpy(f32(Q)).cuda()
    lab, amb = g.predict(Qg, path="tensor", return_ambiguous=True)
    olab = oracle.birch_predict(ocen, osqn, f32(Q).astype(np.float64))
    assert np.array_equal(lab.cpu().numpy(), olab)
    assert amb >= 1  # at least the exact ties among the midpoints went to fp64
    record("birch_tc_ties_ambiguous", amb)
    g.close()


def test_birch_tensor_predict_lattice_ties(igp):
    """Rows on an integer lattice against lattice clusters, queried at half-integer offsets: exact
    ties by the dozen (up to 2^8 equidistant clusters), so the tensor path takes all three routes —
    in-kernel re-check, the candidate pass, and rows with more than 32 candidates through the
    all-cluster fp64 pass — and must still return the oracle's first minimum."""
    rng = np.random.default_rng(9)
    X = np.unique(rng.integers(0, 3, (3000, 8)), axis=0).astype(np.float64)
    g, ocen, osqn = fit_clusters(igp, X, 0.1, 50)
    assert ocen.shape[0] == X.shape[0]
    Q = f32(np.concatenate([X, X[:400] + 0.5, X[:400] + rng.integers(0, 2, (400, 8)) * 0.5, rng.random((400, 8)) * 2]))
    Qg = torch.from_numpy(Q).cuda()
    lab, amb = g.predict(Qg, path="tensor", return_ambiguous=True)
    assert np.array_equal(lab.cpu().numpy(), oracle.birch_predict(ocen, osqn, Q.astype(np.float64)))
    assert amb > 400
    record("birch_tc_lattice_ambiguous", amb)
    g.close()


def test_birch_tensor_predict_huge_values_all_fp64(igp):
    """Magnitudes outside the certified fp32 range (M = inf): every row is solved in fp64."""
    rng = np.random.default_rng(4)
    X = rng.normal(0, 1, (500, 8)) * 1e16
    g, ocen, osqn = fit_clusters(igp, X, 1e15, 50)
    Xg = torch.from_numpy(f32(X)).cuda()
    lab, amb = g.predict(Xg, path="tensor", return_ambiguous=True)
    assert amb == X.shape[0]
    assert np.array_equal(lab.cpu().numpy(), oracle.birch_predict(ocen, osqn, f32(X).astype(np.float64)))
    g.close()


@pytest.mark.parametrize("d", [8, 24, 32, 40, 48, 56, 64])
def test_birch_tensor_predict_many_clusters(igp, d):
    """Thousands of clusters (many centroid tiles, a ragged last tile) and a ragged last row tile,
    every tile shape: N = 128 (d < 48) and 256 (d >= 48), one K stage (d <= 32) or two, full or
    partial (d = 40, 48, 56): tensor path == fp64 path == oracle; almost every row certified."""
    rng = np.random.default_rng(10 + d)
    X = 1 / (1 + np.exp(-rng.normal(0, 1, (6000, d))))
    g, ocen, osqn = fit_clusters(igp, X, 0.35 * np.sqrt(d / 64), 50)
    K = ocen.shape[0]
    assert K > 300
    Q = f32(1 / (1 + np.exp(-rng.normal(0, 1, (3001, d)))))
    Qg = torch.from_numpy(Q).cuda()
    olab = oracle.birch_predict(ocen, osqn, Q.astype(np.float64))
    lab, amb = g.predict(Qg, path="tensor", return_ambiguous=True)
    assert np.array_equal(lab.cpu().numpy(), olab)
    assert np.array_equal(g.predict(Qg, path="fp64").cpu().numpy(), olab)
    assert amb < Q.shape[0] // 10
    record(f"birch_tc_many_d{d}", {"K": K, "rows": Q.shape[0], "ambiguous": amb})
    g.close()


def test_birch_tensor_predict_streaming_scale(igp):
    """The streaming leg's regime (tens of thousands of clusters): tensor path == fp64 path
    (the fp64 path is pinned to the oracle above) on 100K rows x 40K clusters; times recorded."""
    rng = np.random.default_rng(21)
    X = torch.from_numpy(f32(1 / (1 + np.exp(-rng.normal(0, 1.5, (40000, 64)))))).cuda()
    g = igp.Birch(64, 0.05, 50).partial_fit(X)
    K = g.info()[0]
    assert K > 30000
    Q = torch.cat([X, torch.from_numpy(f32(1 / (1 + np.exp(-rng.normal(0, 1.5, (60000, 64)))))).cuda()])
    times = {}
    for path in ("fp64", "tensor"):
        g.predict(Q, path=path)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lab = g.predict(Q, path=path)
        b.record()
        torch.cuda.synchronize()
        times[path] = a.elapsed_time(b)
        if path == "fp64":
            ref = lab.clone()
    lab, amb = g.predict(Q, path="tensor", return_ambiguous=True)
    assert torch.equal(lab, ref)
    record("birch_tc_streaming_scale", {"K": K, "rows": Q.shape[0], "ambiguous": amb,
                                        "fp64_ms": times["fp64"], "tensor_ms": times["tensor"]})
    g.close()


def test_birch_tensor_predict_degenerate_sizes(igp):
    """One cluster (K = 1: every row's second-best is the +inf padding), one row, and K just
    past a tile boundary (257 clusters: a 1-centroid ragged tile), on the tensor path."""
    b = igp.Birch(16, 0.5, 50).partial_fit(torch.full((10, 16), 0.25, device="cuda"))
    assert b.info()[0] == 1
    lab, amb = b.predict(torch.rand((300, 16), device="cuda"), path="tensor", return_ambiguous=True)
    assert torch.all(lab == 0) and amb == 0
    assert b.predict(torch.rand((1, 16), device="cuda"), path="tensor").tolist() == [0]
    b.close()
    rng = np.random.default_rng(12)
    X = rng.random((257, 64)) * 4  # well separated: every row its own cluster
    g, ocen, osqn = fit_clusters(igp, X, 1e-3, 50)
    assert ocen.shape[0] == 257
    Q = f32(np.concatenate([X, rng.random((100, 64)) * 4]))
    lab = g.predict(torch.from_numpy(Q).cuda(), path="tensor").cpu().numpy()
    assert np.array_equal(lab, oracle.birch_predict(ocen, osqn, Q.astype(np.float64)))
    g.close()


def test_birch_tensor_predict_row_chunks(igp):
    """More rows than one tensor-core pass takes (2^22 per chunk; the chunks share the centroid
    split and the uncertified-row list): tensor path == fp64 path on 2^22 + 1000 rows."""
    g = torch.Generator().manual_seed(8)
    fit = torch.rand((3000, 8), generator=g).cuda()
    b = igp.Birch(8, 0.15, 50).partial_fit(fit)
    Q = torch.rand(((1 << 22) + 1000, 8), generator=g).cuda()
    lab, amb = b.predict(Q, path="tensor", return_ambiguous=True)
    ref = b.predict(Q, path="fp64")
    assert torch.equal(lab, ref)
    record("birch_tc_chunks", {"K": b.info()[0], "rows": Q.shape[0], "ambiguous": amb})
    b.close()


def test_birch_errors(igp):
    with pytest.raises(igp.IGPError):
        igp.Birch(8, 0.0, 50)
    with pytest.raises(igp.IGPError):
        igp.Birch(8, 0.5, 64)  # branching above the device limit (B + 1 entries <= 64)
    b = igp.Birch(4, 0.5, 50)
    with pytest.raises(igp.IGPError):
        b.predict(torch.zeros((3, 4), device="cuda"))  # empty tree
    bad = torch.zeros((5, 4), device="cuda")
    bad[2, 1] = float("nan")
    with pytest.raises(igp.IGPError):
        b.partial_fit(bad)
    assert b.info()[3] == 0  # unchanged
    b.partial_fit(torch.zeros((0, 4), device="cuda"))
    b.partial_fit(torch.ones((2, 4), device="cuda"))
    assert b.info()[:1] == (1,)
    with pytest.raises(igp.IGPError):
        b.predict(torch.ones((2, 4), device="cuda"), path="tensor")  # d = 4: not a multiple of 8
    with pytest.raises(ValueError):
        b.predict(torch.ones((2, 4), device="cuda"), path="bf16")
    b.close()


def test_birch_headline_full_size(igp, headline):
    """The bench's clustering step at the Headline size (N = 1M): GPU fit + predict on the GPU
    embedding vs the oracle on the same rows, bit-exact; times recorded."""
    c, edges = headline
    e = torch.from_numpy(edges).cuda()
    g = igp.build_graph(e, c.num_nodes)
    Zg = igp.embed(g, c.tau, c.d, c.steps, c.seed)
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    b = igp.Birch(c.d, 1.0, 50).partial_fit(Zg)
    lab = b.predict(Zg)
    torch.cuda.synchronize()
    record("birch_headline_gpu_s", time.perf_counter() - t0)
    Z = Zg.cpu().numpy().astype(np.float64)
    t0 = time.perf_counter()
    o = oracle.Birch(c.d, 1.0, 50).fit(Z)
    ocen, osqn, on, ols, oss = o.clusters()
    olab = oracle.birch_predict(ocen, osqn, Z)
    record("birch_headline_oracle_s", time.perf_counter() - t0)
    cen, sqn, cnt, ls, ss = (t.cpu().numpy() for t in b.clusters())
    record("birch_headline_K", int(cen.shape[0]))
    assert np.array_equal(cen, ocen) and np.array_equal(cnt, on) and np.array_equal(ss, oss)
    assert np.array_equal(lab.cpu().numpy(), olab)
