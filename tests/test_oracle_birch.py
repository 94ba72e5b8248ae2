"""Pins for the oracle's BIRCH (oracle/birch_oracle.c; Alg. 1 l.7, Alg. 2 l.9-11) — no GPU.

The paper fits scikit-learn's Birch to the embeddings with no cluster count (PAPER.md:172,
:193, :427).  The oracle is pinned against:
  - that library routine itself (sklearn.cluster.Birch, test-only): the same leaf clusters
    (centroids bit for bit, as a multiset) and the same partition of the points, across
    thresholds, branching factors (deep trees with many splits) and widths;
  - hand-computed CF merges (n, LS, SS, centroid, radius) on three points;
  - SPEC.md:253-290 examples and invariants: separated clouds, a single point, fit(P1 || P2)
    == fit(P1) + partial_fit(P2), empty partial_fit, sum of leaf CFs == the data, every leaf
    radius <= T, predict ties go to the lowest id.
"""
import numpy as np
import pytest

import oracle


def sk_birch(X, T, B):
    from sklearn.cluster import Birch
    return Birch(threshold=T, branching_factor=B, n_clusters=None).fit(X)


def centroid_bijection(cen, ref):
    """index map i -> j with cen[i] == ref[j] bit for bit (None if the multisets differ)."""
    if cen.shape != ref.shape:
        return None
    m = {c.tobytes(): j for j, c in enumerate(ref)}
    if len(m) != len(ref):
        return None
    try:
        return np.array([m[c.tobytes()] for c in cen])
    except KeyError:
        return None


def datasets():
    rng = np.random.default_rng(11)
    out = []
    C = rng.random((12, 8))
    out.append(("blobs8", C[rng.integers(0, 12, 2000)] + rng.normal(0, 0.05, (2000, 8)), 0.1, 50))
    out.append(("uniform_deep", rng.random((600, 8)), 0.01, 3))  # every point a leaf entry, depth ~6
    out.append(("sigmoid64_T1", 1 / (1 + np.exp(-rng.normal(0, 1, (3000, 64)))), 1.0, 50))
    out.append(("sigmoid64_T05_B10", 1 / (1 + np.exp(-rng.normal(0, 1, (2000, 64)))), 0.5, 10))
    out.append(("sigmoid16_B5", 1 / (1 + np.exp(-rng.normal(0, 1, (3000, 16)))), 0.3, 5))
    return out


@pytest.mark.parametrize("name,X,T,B", datasets(), ids=[d[0] for d in datasets()])
def test_matches_library_birch(name, X, T, B):
    b = oracle.Birch(X.shape[1], T, B).fit(X)
    cen, sqn, n, ls, ss = b.clusters()
    sk = sk_birch(X, T, B)
    perm = centroid_bijection(cen, sk.subcluster_centers_)
    assert perm is not None, "leaf clusters differ from sklearn Birch"
    # the same partition: my label j corresponds to sklearn's label perm[j]
    assert np.array_equal(perm[b.predict(X)], sk.labels_)
    assert n.sum() == X.shape[0]


def test_hand_computed_cf_merges():
    """x1 = (0,0), x2 = (0.3,0.4) (|x2|=0.5), x3 = (3,0), T = 0.5:
    merge x2 into {x1}: n=2, LS=(0.3,0.4), SS=0.25, c=(0.15,0.2), r^2 = 0.125 - 0.0625 = 0.0625 <= 0.25;
    x3: radius^2 of {x1,x2,x3} = (0.25+9)/3 - |(3.3,0.4)/3|^2 = 3.0833 - 1.2278 > 0.25: new entry."""
    X = np.array([[0.0, 0.0], [0.3, 0.4], [3.0, 0.0]])
    b = oracle.Birch(2, 0.5, 50).fit(X)
    cen, sqn, n, ls, ss = b.clusters()
    assert n.tolist() == [2.0, 1.0]
    np.testing.assert_allclose(ls[0], [0.3, 0.4], rtol=0, atol=1e-15)
    np.testing.assert_allclose(ss, [0.25, 9.0], rtol=0, atol=1e-15)
    np.testing.assert_allclose(cen, [[0.15, 0.2], [3.0, 0.0]], rtol=0, atol=1e-15)
    np.testing.assert_allclose(sqn, [0.0625, 9.0], rtol=0, atol=1e-15)
    r2 = ss / n - sqn
    np.testing.assert_allclose(r2, [0.0625, 0.0], atol=1e-15)


def test_separated_clouds_and_single_point():
    rng = np.random.default_rng(1)
    X = np.concatenate([rng.normal(0, 0.01, (50, 4)), rng.normal(5, 0.01, (50, 4))])
    b = oracle.Birch(4, 0.5, 50).fit(X)
    assert b.clusters()[0].shape[0] == 2
    lab = b.predict(X)
    assert len(set(lab[:50])) == 1 and len(set(lab[50:])) == 1 and lab[0] != lab[50]
    one = oracle.Birch(3, 0.5, 50).fit(np.array([[0.1, 0.2, 0.3]]))
    cen = one.clusters()[0]
    assert cen.shape == (1, 3) and np.array_equal(cen[0], [0.1, 0.2, 0.3])


def test_partial_fit_equals_fit_in_the_same_order():
    rng = np.random.default_rng(2)
    X = 1 / (1 + np.exp(-rng.normal(0, 1, (1500, 16))))
    a = oracle.Birch(16, 0.4, 8).fit(X)
    b = oracle.Birch(16, 0.4, 8)
    b.partial_fit(X[:700])
    b.partial_fit(X[700:1000])
    b.partial_fit(np.zeros((0, 16)))  # empty partial fit: unchanged
    b.partial_fit(X[1000:])
    for u, v in zip(a.clusters(), b.clusters()):
        assert np.array_equal(u, v)
    assert a.shape() == b.shape()


def test_invariants_cf_sums_and_radius():
    rng = np.random.default_rng(3)
    X = 1 / (1 + np.exp(-rng.normal(0, 1.5, (2500, 32))))
    T = 0.6
    b = oracle.Birch(32, T, 6).fit(X)
    cen, sqn, n, ls, ss = b.clusters()
    assert n.sum() == X.shape[0]
    np.testing.assert_allclose(ls.sum(0), X.sum(0), rtol=1e-12)
    np.testing.assert_allclose(ss.sum(), (X * X).sum(), rtol=1e-12)
    r2 = ss / n - sqn
    assert np.all(r2 <= T * T + 1e-12)
    np.testing.assert_allclose(cen, ls / n[:, None], rtol=1e-15)
    dep, nodes, pts = b.shape()
    assert pts == X.shape[0] and dep >= 3


def test_predict_exact_and_ties():
    cen = np.array([[0.0, 0.0], [2.0, 0.0], [0.0, 2.0]])
    sqn = (cen * cen).sum(1)
    X = np.array([[2.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0], [0.1, 0.1]])
    lab = oracle.birch_predict(cen, sqn, X)
    # exact centroid -> that label; equidistant -> lowest id
    assert lab.tolist() == [1, 0, 0, 0, 0]


def test_rejects_bad_arguments():
    with pytest.raises(oracle.OracleError):
        oracle.Birch(4, 0.0, 50)
    with pytest.raises(oracle.OracleError):
        oracle.Birch(4, 0.5, 1)
    b = oracle.Birch(2, 0.5, 50)
    with pytest.raises(oracle.OracleError):
        b.partial_fit(np.array([[np.nan, 0.0]]))
