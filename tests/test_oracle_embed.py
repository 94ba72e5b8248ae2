"""Composite pins for the oracle's full FFP, Alg. 1 lines 1-6 (no GPU).

The paper prints no worked FFP example, so the composite is pinned by:
  - LINEAR mode == U phi(Lambda~)^L U^T Theta from eigh (north star, N <= 200);
  - a spectral twin: propagate replaced by the eigh form, tanh/ZNorm/sigmoid kept;
  - relabelling equivariance;
  - special cases: M = 0 reduces to a per-column scalar recurrence; N = 1 gives 0.5;
  - ranges and moments: sigmoid output in (0,1), Z^(L) columns
    standardised, |Z| <= sqrt(N - 1) (z-score bound);
  - determinism and thread-count independence.
"""
import numpy as np
import pytest

import oracle
from test_oracle_filter import dense_adjacency, random_graph, spectral_filter


def _graph(seed, n, p):
    rng = np.random.default_rng(seed)
    edges = random_graph(rng, n, p)
    rp, ci, _ = oracle.build_csr(edges, n)
    return edges, rp, ci


def np_zscore(T):
    mu = T.mean(0)
    sd = T.std(0)
    return np.where(sd < 1e-8, 0.0, (T - mu) / np.where(sd < 1e-8, 1.0, sd))


@pytest.mark.parametrize("tau,L", [(-1.0, 1), (-1.0, 5), (0.0, 10), (-1.5, 3), (2.0, 4)])
def test_linear_mode_equals_spectral_power(tau, L):
    n, d = 120, 8
    edges, rp, ci = _graph(3, n, 0.06)
    th = oracle.input_theta(9, 0, n, d)
    out = oracle.embed(rp, ci, n, d, L, tau, seed=9, mode=oracle.MODE_LINEAR)
    ref = spectral_filter(dense_adjacency(edges, n), tau, th, power=L)
    assert np.max(np.abs(out - ref)) < 1e-10 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("tau", [-1.0, -1.5, 0.0])
def test_spectral_twin_full_ffp(tau):
    n, d, L = 150, 16, 6
    edges, rp, ci = _graph(4, n, 0.05)
    A = dense_adjacency(edges, n)
    Z = oracle.input_theta(1, 0, n, d)
    for _ in range(L):
        Z = np_zscore(np.tanh(spectral_filter(A, tau, Z)))
    ref = 1.0 / (1.0 + np.exp(-Z))
    out = oracle.embed(rp, ci, n, d, L, tau, seed=1)
    assert np.max(np.abs(out - ref)) < 1e-10


def test_relabel_equivariance():
    n, d, L = 300, 16, 8
    edges, rp, ci = _graph(5, n, 0.03)
    rng = np.random.default_rng(6)
    perm = rng.permutation(n)  # new id of old node i is perm[i]
    Z0 = rng.standard_normal((n, d)) / 4.0
    out = oracle.embed(rp, ci, n, d, L, -1.0, Z0=Z0)
    rp2, ci2, _ = oracle.build_csr(perm[edges], n)
    Z0p = np.empty_like(Z0)
    Z0p[perm] = Z0
    out2 = oracle.embed(rp2, ci2, n, d, L, -1.0, Z0=Z0p)
    assert np.max(np.abs(out2[perm] - out)) < 1e-12


def test_empty_graph_reduces_to_column_recurrence():
    n, d, L = 64, 8, 5
    rp = np.zeros(n + 1, dtype=np.int32)
    ci = np.zeros(0, dtype=np.int32)
    th = oracle.input_theta(2, 0, n, d)
    Z = th.copy()
    for _ in range(L):
        Z = np_zscore(np.tanh(0.1 * Z))  # phi*Z = theta Z when A = 0
    out = oracle.embed(rp, ci, n, d, L, -1.0, seed=2)
    assert np.max(np.abs(out - 1 / (1 + np.exp(-Z)))) < 1e-12


def test_single_node_is_one_half():
    out = oracle.embed(np.zeros(2, dtype=np.int32), np.zeros(0, dtype=np.int32), 1, 16, 3, -1.0, seed=0)
    assert np.all(out == 0.5)


def test_ranges_moments_and_bounds():
    from synth.dcsbm import CONFIGS, generate
    cfg = CONFIGS["tiny"]
    edges, _ = generate(cfg)
    rp, ci, _ = oracle.build_csr(edges, cfg.num_nodes)
    out = oracle.embed(rp, ci, cfg.num_nodes, cfg.d, cfg.steps, cfg.tau, seed=0)
    assert out.min() > 0 and out.max() < 1
    Z = oracle.embed(rp, ci, cfg.num_nodes, cfg.d, cfg.steps, cfg.tau, seed=0, mode=oracle.MODE_PRE_SIGMOID)
    assert np.allclose(Z.mean(0), 0, atol=1e-12) and np.allclose(Z.std(0), 1, atol=1e-12)
    assert np.abs(Z).max() <= np.sqrt(cfg.num_nodes - 1) + 1e-9
    assert np.allclose(out, 1 / (1 + np.exp(-Z)), rtol=0, atol=1e-15)


def test_determinism_threads_and_input():
    from synth.dcsbm import CONFIGS, generate
    cfg = CONFIGS["tiny"]
    edges, _ = generate(cfg)
    rp, ci, _ = oracle.build_csr(edges, cfg.num_nodes)
    a = oracle.embed(rp, ci, cfg.num_nodes, 32, 6, -1.0, seed=5)
    b = oracle.embed(rp, ci, cfg.num_nodes, 32, 6, -1.0, seed=5, nthreads=4)
    c = oracle.embed(rp, ci, cfg.num_nodes, 32, 6, -1.0, Z0=oracle.input_theta(5, 0, cfg.num_nodes, 32))
    assert np.array_equal(a, b) and np.array_equal(a, c)
    e = oracle.embed(rp, ci, cfg.num_nodes, 32, 6, -1.0, seed=6)
    assert np.mean(a != e) > 0.99


def test_negative_tau_changes_the_embedding():
    """tau enters only through D_tau: tau = -1 and tau = 0 differ; all isolated-node
    rows still evolve by the theta-only recurrence."""
    n = 200
    edges, rp, ci = _graph(8, n, 0.04)
    a = oracle.embed(rp, ci, n, 16, 5, -1.0, seed=0)
    b = oracle.embed(rp, ci, n, 16, 5, 0.0, seed=0)
    assert np.abs(a - b).max() > 1e-3


# ------------------------------------------------------------------ optional row-L2 post-op (reading A12)
def test_row_l2_closed_forms():
    """Pythagorean rows have exact unit-norm images; zero rows are unchanged."""
    Z = np.array([[3.0, 4.0], [0.0, 0.0], [5.0, 12.0], [-8.0, 15.0]])
    out = oracle.row_l2(Z)
    assert np.array_equal(out, np.array([[0.6, 0.8], [0.0, 0.0], [5 / 13, 12 / 13], [-8 / 17, 15 / 17]]))


def test_row_l2_unit_norm_and_direction():
    rng = np.random.default_rng(5)
    Z = rng.random((300, 64)) + 1e-3  # sigmoid outputs are positive
    out = oracle.row_l2(Z)
    assert np.allclose(np.linalg.norm(out, axis=1), 1.0, atol=1e-14)
    # each row is a positive multiple of its input: out_i * ||Z_i|| == Z_i
    assert np.allclose(out * np.linalg.norm(Z, axis=1, keepdims=True), Z, rtol=1e-14, atol=0)
    # idempotent
    assert np.allclose(oracle.row_l2(out), out, atol=1e-15)


# ---------------------------------------------------------------- fp32 twin
def _matching(n):
    """Perfect matching (2k, 2k+1): every degree 1, so D_tau = 1 and s = 1 exactly at tau = 0."""
    edges = np.array([[2 * k, 2 * k + 1] for k in range(n // 2)], dtype=np.int32)
    rp, ci, _ = oracle.build_csr(edges, n)
    return rp, ci


def test_fp32_twin_exact_on_dyadic_linear_case():
    """Closed form: on a perfect matching at tau = 0 (s = 1), theta = 0.5, alpha = 1 and integer
    Z0, every LINEAR-mode value P_i = Z_i / 2 + Z_partner is exactly representable in float, so
    the twin equals the fp64 oracle bit for bit and equals the closed form."""
    n, d, L = 40, 8, 3
    rp, ci = _matching(n)
    rng = np.random.default_rng(2)
    Z0 = rng.integers(-8, 9, size=(n, d)).astype(np.float64)
    kw = dict(theta=0.5, alpha=1.0, Z0=Z0, mode=oracle.MODE_LINEAR)
    a = oracle.embed(rp, ci, n, d, L, 0.0, **kw)
    b = oracle.embed(rp, ci, n, d, L, 0.0, fp32_twin=True, **kw)
    Z = Z0.copy()
    partner = np.arange(n) ^ 1
    for _ in range(L):
        Z = 0.5 * Z + Z[partner]
    assert np.array_equal(a, Z) and np.array_equal(b, Z)


def test_fp32_twin_is_float_and_within_fp32_bound():
    """The twin really rounds to float (it differs from fp64 on a generic graph) and stays within
    the fp32 drift bound the SURVEY probe measured for such graphs (<= 1e-5 row-relative)."""
    n, d, L = 300, 16, 8
    _, rp, ci = _graph(7, n, 0.04)
    a = oracle.embed(rp, ci, n, d, L, -1.0, seed=3)
    b = oracle.embed(rp, ci, n, d, L, -1.0, seed=3, fp32_twin=True)
    err = np.max(np.abs(a - b) / np.linalg.norm(a, axis=1, keepdims=True))
    assert 1e-9 < err < 1e-5
    assert np.all(b.astype(np.float32).astype(np.float64) == b)  # float values


def test_fp32_twin_znorm_golden():
    """M = 0, L = 1 from Z0 = tanh^-1 of [1,2,3]/4 scaled back by theta: one ZNorm of the column
    [t1, t2, t3] = [0.25, 0.5, 0.75] gives [-1.2247, 0, 1.2247], in float."""
    n, d = 3, 4
    rp = np.zeros(n + 1, dtype=np.int32)
    ci = np.zeros(0, dtype=np.int32)
    t = np.array([0.25, 0.5, 0.75])
    Z0 = np.repeat((np.arctanh(t) / 0.1)[:, None], d, axis=1)
    out = oracle.embed(rp, ci, n, d, 1, -1.0, Z0=Z0, mode=oracle.MODE_PRE_SIGMOID, fp32_twin=True)
    np.testing.assert_allclose(out[:, 0], [-np.sqrt(1.5), 0.0, np.sqrt(1.5)], atol=2e-6)
