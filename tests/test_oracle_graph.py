"""Pins for the oracle's graph construction and Eq. (1) (no GPU).

CSR: golden examples (derived from PAPER.md:127), brute force with
Python sets on random lists, and the invariants of SPEC.md:29-33.
Eq. (1): the worked substitutions in tests/golden/examples.json and the bounds
eps <= D <= deg (tau<0), D >= deg (tau>0), D == deg (tau=0).
"""
import numpy as np
import pytest

import oracle
from conftest import golden


def brute_force_csr(edges, n):
    adj = [set() for _ in range(n)]
    for u, v in edges:
        if u != v:
            adj[u].add(v)
            adj[v].add(u)
    rp = [0]
    ci = []
    for i in range(n):
        ci.extend(sorted(adj[i]))
        rp.append(len(ci))
    return np.array(rp, dtype=np.int32), np.array(ci, dtype=np.int32)


@pytest.mark.parametrize("case", golden()["build_graph"], ids=lambda c: c["cite"][:20])
def test_build_graph_golden(case):
    rp, ci, m = oracle.build_csr(np.array(case["edges"], dtype=np.int32).reshape(-1, 2), case["num_nodes"])
    assert m == case["M"]
    assert rp.tolist() == case["row_ptr"]
    assert ci.tolist() == case["col_idx"]
    assert np.diff(rp).tolist() == case["deg"]


@pytest.mark.parametrize("trial", range(40))
def test_build_graph_brute_force(trial):
    rng = np.random.default_rng(1000 + trial)
    n = int(rng.integers(1, 60))
    e = int(rng.integers(0, 300))
    edges = rng.integers(0, n, size=(e, 2)).astype(np.int32)
    # add explicit duplicates, reversed copies and self loops
    if e:
        extra = edges[rng.integers(0, e, size=e // 3)]
        edges = np.concatenate([edges, extra[:, ::-1], np.stack([edges[:5, 0]] * 2, 1)])
    rp, ci, m = oracle.build_csr(edges, n)
    rp_b, ci_b = brute_force_csr(edges.tolist(), n)
    assert np.array_equal(rp, rp_b)
    assert np.array_equal(ci, ci_b)
    assert 2 * m == rp[-1]


def test_csr_invariants_dcsbm():
    from synth.dcsbm import CONFIGS, generate
    edges, _ = generate(CONFIGS["tiny"])
    n = CONFIGS["tiny"].num_nodes
    rp, ci, m = oracle.build_csr(edges, n)
    assert rp[0] == 0 and rp[-1] == 2 * m == ci.size
    assert np.all(np.diff(rp) >= 0)
    rows = np.repeat(np.arange(n), np.diff(rp))
    assert not np.any(rows == ci), "self loop"
    for i in range(n):  # strictly ascending => no duplicates
        r = ci[rp[i]:rp[i + 1]]
        assert np.all(np.diff(r) > 0)
    # symmetry: j in row i <=> i in row j
    fwd = set(zip(rows.tolist(), ci.tolist()))
    assert all((j, i) in fwd for (i, j) in fwd)
    # M equals the count of unique unordered non-loop pairs
    e = edges[edges[:, 0] != edges[:, 1]]
    assert m == len({(min(u, v), max(u, v)) for u, v in e.tolist()})


def test_build_graph_errors():
    with pytest.raises(oracle.OracleError):
        oracle.build_csr(np.array([[0, 3]]), 3)
    with pytest.raises(oracle.OracleError):
        oracle.build_csr(np.array([[-1, 0]]), 3)
    with pytest.raises(oracle.OracleError):
        oracle.build_csr(np.zeros((0, 2)), 0)


@pytest.mark.parametrize("case", golden()["corrected_degree"], ids=lambda c: f"deg{c['deg']}_tau{c['tau']}")
def test_corrected_degree_golden(case):
    got = oracle.corrected_degree([case["deg"]], case["tau"], case["eps"])[0]
    assert got == pytest.approx(case["D"], rel=1e-12, abs=1e-15)


def test_corrected_degree_bounds():
    deg = np.arange(0, 300)
    for tau in [-100.0, -80.0, -6.0, -3.0, -1.5, -1.0, -0.5, -1e-4]:
        D = oracle.corrected_degree(deg, tau)
        assert np.all(D >= 1e-3 - 1e-12), tau  # deg - (deg - eps) rounds at ulp(deg)
        assert np.all(D[1:] <= deg[1:]), tau
        assert np.all(D > 0)
    assert np.array_equal(oracle.corrected_degree(deg, 0.0), deg.astype(float))
    for tau in [0.5, 1.0, 5.0, 10.0]:
        assert np.all(oracle.corrected_degree(deg, tau) >= deg)


@pytest.mark.parametrize("n,k", [(5, 2), (9, 1), (40, 7), (1000, 32)])
def test_circulant_generator_matches_its_closed_form(n, k):
    """synth/circulant.py (the maximum-size GPU test's input) against the oracle's CSR: every row
    is {i +- 1..k mod n}, every degree 2k."""
    from synth.circulant import circulant_edges, circulant_row
    e = circulant_edges(n, k).numpy()
    assert e.shape == (n * k, 2)
    rp, ci, m = oracle.build_csr(e, n)
    assert m == n * k and np.array_equal(np.diff(rp), np.full(n, 2 * k))
    for i in range(n):
        assert np.array_equal(ci[rp[i]:rp[i + 1]], circulant_row(n, k, i))
    with pytest.raises(ValueError):
        circulant_edges(4, 2)  # 2k >= n would repeat pairs
