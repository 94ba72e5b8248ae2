"""Pins for the oracle's Eq. (3) propagate, ZNorm and the spectral facts of L_tau (no GPU).

Eq. (3) (spatial form) is checked against Eq. (2)'s SPECTRAL
definition  phi * Z = U phi(Lambda) U^T Z computed from a
numpy eigendecomposition of the dense L_tau built from the RAW edge list — a
different route to the same operator — and against closed forms.  The spectral
facts pin Eq. (1) and the graph together.
"""
import numpy as np
import pytest
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import connected_components

import oracle
from conftest import golden

THETA, ALPHA = 0.1, 1.0


def dense_adjacency(edges, n):
    A = np.zeros((n, n))
    for u, v in np.asarray(edges).reshape(-1, 2).tolist():
        if u != v:
            A[u, v] = A[v, u] = 1.0
    return A


def dense_L_tau(A, tau, eps=1e-3):
    deg = A.sum(1).astype(np.int64)
    D = oracle.corrected_degree(deg, tau, eps)
    s = np.where(deg > 0, 1.0 / np.sqrt(D), 0.0)  # isolated rows: empty neighbour term
    return np.eye(A.shape[0]) - s[:, None] * A * s[None, :]


def spectral_filter(A, tau, Z, power=1):
    """U phi(Lambda~)^power U^T Z with phi(lambda) = (theta + alpha) - alpha lambda (Eq. 2)."""
    lam, U = np.linalg.eigh(dense_L_tau(A, tau))
    phi = (THETA + ALPHA) - ALPHA * lam
    return U @ (phi[:, None] ** power * (U.T @ Z))


def random_graph(rng, n, p):
    A = np.triu((rng.random((n, n)) < p).astype(float), 1)
    u, v = np.nonzero(A)
    return np.stack([u, v], 1).astype(np.int32)


@pytest.mark.parametrize("case", golden()["propagate"], ids=lambda c: f"tau{c['tau']}")
def test_propagate_golden(case):
    n = case["num_nodes"]
    rp, ci, _ = oracle.build_csr(np.array(case["edges"]), n)
    D = oracle.corrected_degree(np.diff(rp), case["tau"])
    P = oracle.propagate(rp, ci, D, np.array(case["Z"]))
    assert np.allclose(P, np.array(case["P"]), rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("trial", range(12))
def test_propagate_equals_spectral_form(trial):
    """Eq. (3) == U phi(Lambda~) U^T Z from eigh(L_tau) (north-star pin, N <= 200)."""
    rng = np.random.default_rng(trial)
    n = int(rng.integers(5, 200))
    edges = random_graph(rng, n, float(rng.uniform(0.02, 0.3)))
    tau = [-1.5, -1.0, -0.5, 0.0, 2.0, -6.0][trial % 6]
    rp, ci, _ = oracle.build_csr(edges, n)
    D = oracle.corrected_degree(np.diff(rp), tau)
    Z = rng.standard_normal((n, 8))
    P = oracle.propagate(rp, ci, D, Z)
    ref = spectral_filter(dense_adjacency(edges, n), tau, Z)
    assert np.max(np.abs(P - ref)) < 1e-10 * max(1.0, np.max(np.abs(ref)))


def test_propagate_dense_matrix_and_linearity():
    rng = np.random.default_rng(5)
    n = 50
    edges = np.concatenate([random_graph(rng, n, 0.1), random_graph(rng, n, 0.1)])  # duplicates
    rp, ci, _ = oracle.build_csr(edges, n)
    D = oracle.corrected_degree(np.diff(rp), -1.0)
    A = dense_adjacency(edges, n)
    s = 1.0 / np.sqrt(D)
    Z1, Z2 = rng.standard_normal((n, 3)), rng.standard_normal((n, 3))
    ref = THETA * Z1 + ALPHA * (s[:, None] * (A @ (s[:, None] * Z1)))
    assert np.allclose(oracle.propagate(rp, ci, D, Z1), ref, rtol=0, atol=1e-12)
    lin = oracle.propagate(rp, ci, D, 2.0 * Z1 - 3.0 * Z2)
    assert np.allclose(lin, 2.0 * oracle.propagate(rp, ci, D, Z1) - 3.0 * oracle.propagate(rp, ci, D, Z2),
                       atol=1e-12)
    assert np.all(oracle.propagate(rp, ci, D, np.zeros((n, 2))) == 0.0)


def test_propagate_closed_forms():
    rng = np.random.default_rng(11)
    n = 80
    edges = random_graph(rng, n, 0.15)
    rp, ci, _ = oracle.build_csr(edges, n)
    deg = np.diff(rp)
    assert deg.min() > 0
    # tau = 0: v = sqrt(deg) satisfies D^{-1/2} A D^{-1/2} v = v, so phi*v = 1.1 v
    D0 = oracle.corrected_degree(deg, 0.0)
    v = np.sqrt(deg.astype(float))[:, None]
    assert np.allclose(oracle.propagate(rp, ci, D0, v), 1.1 * v, rtol=1e-13)
    # k-regular graphs, clamp inactive: phi*1 = (theta + alpha k/(k+tau)) 1
    for n_c, k in [(30, 2), (12, 11)]:
        if k == 2:  # cycle
            e = np.stack([np.arange(n_c), (np.arange(n_c) + 1) % n_c], 1)
        else:  # complete graph
            e = np.array([(i, j) for i in range(n_c) for j in range(i + 1, n_c)])
        rp2, ci2, _ = oracle.build_csr(e, n_c)
        for tau in [-0.5, 0.0, 3.0]:
            D = oracle.corrected_degree(np.diff(rp2), tau)
            P = oracle.propagate(rp2, ci2, D, np.ones((n_c, 1)))
            assert np.allclose(P, THETA + ALPHA * k / (k + tau), rtol=1e-13)


@pytest.mark.parametrize("case", golden()["spectrum"], ids=lambda c: f"n{c['num_nodes']}_tau{c['tau']}")
def test_spectrum_golden(case):
    n = case["num_nodes"]
    rp, ci, _ = oracle.build_csr(np.array(case["edges"]), n)
    A = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(rp))
    A[rows, ci] = 1.0  # from the oracle CSR this time
    lam = np.linalg.eigvalsh(dense_L_tau(A, case["tau"]))
    assert np.allclose(lam, case["eigenvalues"], atol=1e-12)


@pytest.mark.parametrize("trial", range(20))
def test_spectrum_facts(trial):
    """tau=0: spectrum in [0,2], mult(0) = #components;
    tau<0: an infrared eigenvalue < 0 exists;
    tau>0: spectrum inside (0, 2); any tau: Gershgorin discs (Theorem 1)."""
    rng = np.random.default_rng(100 + trial)
    n = int(rng.integers(4, 120))
    edges = random_graph(rng, n, float(rng.uniform(0.01, 0.2)))
    rp, ci, _ = oracle.build_csr(edges, n)
    deg = np.diff(rp)
    keep = deg > 0  # the footnote's statement is about graphs without isolated nodes
    if keep.sum() < 2:
        return
    A = dense_adjacency(edges, n)[np.ix_(keep, keep)]
    lam0 = np.linalg.eigvalsh(dense_L_tau(A, 0.0))
    assert lam0.min() > -1e-10 and lam0.max() < 2 + 1e-10
    ncomp = connected_components(csr_matrix(A), directed=False)[0]
    assert int(np.sum(np.abs(lam0) < 1e-9)) == ncomp
    dk = A.sum(1)
    for tau in [-100.0, -6.0, -1.5, -1.0, -0.3, 0.5, 5.0, 10.0]:
        lam = np.linalg.eigvalsh(dense_L_tau(A, tau))
        D = oracle.corrected_degree(dk.astype(np.int64), tau)
        r = dk / D
        assert lam.min() >= 1 - r.max() - 1e-9 and lam.max() <= 1 + r.max() + 1e-9
        if tau < 0:
            assert lam.min() < 0, "no infrared eigenvalue"
        else:
            assert lam.min() > 0 and lam.max() < 2


@pytest.mark.parametrize("case", golden()["gershgorin"], ids=lambda c: f"tau{c['tau']}")
def test_gershgorin_golden(case):
    D = oracle.corrected_degree([case["deg"]], case["tau"])[0]
    r = case["deg"] / D
    assert [1 - r, 1 + r] == pytest.approx(case["interval"], rel=1e-12)


@pytest.mark.parametrize("case", golden()["zscore"], ids=lambda c: str(c["column"]))
def test_zscore_golden(case):
    out = oracle.zscore_columns(np.array(case["column"])[:, None])[:, 0]
    assert np.allclose(out, case["out"], rtol=1e-14, atol=1e-15)


def test_zscore_properties():
    rng = np.random.default_rng(2)
    T = rng.standard_normal((1000, 5)) * [1, 2, 3, 4, 5] + [0, 1, -1, 10, 100]
    Z = oracle.zscore_columns(T)
    assert np.allclose(Z.mean(0), 0, atol=1e-13)
    assert np.allclose(Z.std(0), 1, atol=1e-13)  # population std
    assert np.allclose(oracle.zscore_columns(Z), Z, atol=1e-12)  # idempotent
    assert np.all(oracle.zscore_columns(np.ones((1, 4))) == 0.0)  # N = 1 -> constant column
    # affine invariance: ZNorm(a x + b) = ZNorm(x) for a > 0, = -ZNorm(x) for a < 0
    assert np.allclose(oracle.zscore_columns(3 * T + 7), Z, atol=1e-12)
    assert np.allclose(oracle.zscore_columns(-2 * T), -Z, atol=1e-12)
    # population (1/N), not sample (1/(N-1)) — reading A2
    col = np.array([0.0, 2.0])
    assert np.allclose(oracle.zscore_columns(col)[:, 0], [-1.0, 1.0])


def test_zscore_sample_std_golden():
    """ddof = 1 (sample std, the other reading of PAPER.md:166): [1,2,3] has s = 1, so the
    column becomes [-1, 0, 1]; a single row (N = 1 <= ddof) is treated as constant (0)."""
    out = oracle.zscore_columns(np.array([1.0, 2.0, 3.0])[:, None], ddof=1)[:, 0]
    np.testing.assert_allclose(out, [-1.0, 0.0, 1.0], atol=1e-15)
    assert oracle.zscore_columns(np.array([[5.0, -2.0]]), ddof=1).tolist() == [[0.0, 0.0]]
    T = np.random.default_rng(0).standard_normal((50, 3))
    np.testing.assert_allclose(oracle.zscore_columns(T, ddof=1), (T - T.mean(0)) / T.std(0, ddof=1), atol=1e-14)
