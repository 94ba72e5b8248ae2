"""Seeded synthetic inputs: degree-corrected stochastic block model (DC-SBM) edge lists.

Shared by tests/ and bench.py.  This module holds NONE of the method's
arithmetic (no degrees, corrections, propagation or normalisation): it only
draws raw edge lists (with duplicates and self loops, as a builder's realistic
input) and planted block labels.  Both the CUDA path and the oracle consume its
output unchanged.

The paper measures on the IEEE HPEC Graph Challenge graphs (PAPER.md:246-261,
Table I; generated with graph-tool), which are not in this
container.  These DC-SBM graphs stand in for them with the shape of Table I:
K blocks from Table I where it exists, average degree ~40, degrees ~10-126,
and the "hardest" within:between ratio (DESIGN.md §4 gives the recipe).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class DCSBMConfig:
    name: str
    num_nodes: int
    num_blocks: int
    ratio: float  # within : between edge ratio
    num_edges: int  # target undirected edges (Poisson mean)
    d: int
    tau: float
    steps: int  # L, filter steps (Table II; reading A8)
    seed: int = 0
    power: float = 2.1  # truncated power law exponent for degree propensities
    theta_min: float = 10.0
    theta_max: float = 100.0


# BASELINE.json configs (L per Table II, SURVEY.md D4 / DESIGN.md reading A8)
CONFIGS = {
    "tiny": DCSBMConfig("tiny", 1_000, 11, 2.5, 10_000, 64, -1.0, 10),
    "medium": DCSBMConfig("medium", 50_000, 44, 2.5, 500_000, 64, -1.0, 40),
    "headline": DCSBMConfig("headline", 1_000_000, 125, 2.5, 20_000_000, 64, -1.0, 60),
    "streaming": DCSBMConfig("streaming", 200_000, 71, 2.0, 4_000_000, 64, -1.0, 20),
    "large": DCSBMConfig("large", 5_000_000, 220, 1.5, 100_000_000, 128, -1.0, 60),
}

# The paper's own settings (Table II: tau, L, d per N) on DC-SBM graphs with
# Table I's shape (K, M ~ 20 N): SURVEY.md §8(f) rank 3.  Parity cases and
# throughput reports, not bench lines.
PAPER_CONFIGS = {
    "paper_5k": DCSBMConfig("paper_5k", 5_000, 19, 2.5, 100_000, 64, -6.0, 10),
    "paper_10k": DCSBMConfig("paper_10k", 10_000, 25, 2.5, 200_000, 64, -3.0, 9),
    "paper_50k": DCSBMConfig("paper_50k", 50_000, 44, 2.5, 1_000_000, 32, -80.0, 40),
    "paper_100k": DCSBMConfig("paper_100k", 100_000, 56, 2.5, 2_000_000, 32, -80.0, 60),
    "paper_500k": DCSBMConfig("paper_500k", 500_000, 98, 2.5, 10_000_000, 32, -80.0, 70),
    "paper_1m": DCSBMConfig("paper_1m", 1_000_000, 125, 2.5, 20_000_000, 32, -80.0, 60),
    "paper_stream_100k": DCSBMConfig("paper_stream_100k", 100_000, 56, 2.5, 2_000_000, 32, -100.0, 20),
    "paper_stream_1m": DCSBMConfig("paper_stream_1m", 1_000_000, 125, 2.5, 20_000_000, 16, -100.0, 20),
}
ALL_CONFIGS = {**CONFIGS, **PAPER_CONFIGS}


def block_sizes(rng: np.random.Generator, n: int, k: int, min_size: int = 10) -> np.ndarray:
    """Block sizes ~ Dirichlet(2·1_K)·N, each >= min_size, repaired to sum to N."""
    f = rng.dirichlet(np.full(k, 2.0))
    sizes = np.maximum(min_size, np.floor(f * n).astype(np.int64))
    while sizes.sum() > n:  # subtract from the largest block
        b = int(np.argmax(sizes))
        sizes[b] -= min(sizes.sum() - n, sizes[b] - min_size)
        if sizes[b] <= min_size and sizes.sum() > n and np.all(sizes <= min_size):
            raise ValueError("N too small for K blocks of min size")
    while sizes.sum() < n:  # add to the smallest block
        sizes[int(np.argmin(sizes))] += n - sizes.sum()
    return sizes


def propensities(rng: np.random.Generator, n: int, power: float, lo: float, hi: float) -> np.ndarray:
    """theta_i with pdf ∝ theta^-power on [lo, hi], by inverse CDF."""
    a = 1.0 - power
    u = rng.random(n)
    return (lo ** a + u * (hi ** a - lo ** a)) ** (1.0 / a)


def generate(cfg: DCSBMConfig, seed: int | None = None):
    """Returns (edges int32 [E, 2] raw with duplicates/self loops, labels int32 [N])."""
    seed = cfg.seed if seed is None else seed
    rng = np.random.default_rng(seed)
    n, k = cfg.num_nodes, cfg.num_blocks
    sizes = block_sizes(rng, n, k)
    # membership: a seeded permutation cut into blocks (ids carry no block locality)
    perm = rng.permutation(n).astype(np.int64)
    labels = np.empty(n, dtype=np.int32)
    starts = np.concatenate([[0], np.cumsum(sizes)])
    for b in range(k):
        labels[perm[starts[b]:starts[b + 1]]] = b
    theta = propensities(rng, n, cfg.power, cfg.theta_min, cfg.theta_max)
    # nodes grouped by block (in perm order) with cumulative propensity
    theta_by = theta[perm]
    cum = np.cumsum(theta_by)
    kappa = np.add.reduceat(theta_by, starts[:-1])
    cum_start = np.concatenate([[0.0], cum])[starts[:-1]]
    m_in = cfg.num_edges * cfg.ratio / (1.0 + cfg.ratio)
    m_out = cfg.num_edges / (1.0 + cfg.ratio)
    lam_in = m_in * kappa ** 2 / np.sum(kappa ** 2)
    bi, bj = np.triu_indices(k, 1)
    w = kappa[bi] * kappa[bj]
    lam_out = m_out * w / w.sum()
    cnt_in = rng.poisson(lam_in)
    cnt_out = rng.poisson(lam_out)
    bu = np.concatenate([np.repeat(np.arange(k), cnt_in), np.repeat(bi, cnt_out)])
    bv = np.concatenate([np.repeat(np.arange(k), cnt_in), np.repeat(bj, cnt_out)])

    def endpoint(blocks):
        # sample a node within each block ∝ theta (inverse CDF on the block's cumulative theta)
        x = cum_start[blocks] + rng.random(blocks.shape[0]) * kappa[blocks]
        pos = np.searchsorted(cum, x, side="right")
        pos = np.minimum(pos, starts[blocks + 1] - 1)  # guard fp edge at the block's end
        pos = np.maximum(pos, starts[blocks])
        return perm[pos]

    u = endpoint(bu)
    v = endpoint(bv)
    order = rng.permutation(u.shape[0])  # edge order carries no structure either
    edges = np.stack([u[order], v[order]], axis=1).astype(np.int32)
    return edges, labels


def stream_batches(edges: np.ndarray, stages: int = 10, seed: int = 0):
    """Streaming config (uniform edge sampling): a seeded permutation of the raw edge list
    cut into ``stages`` batches of ~1/stages each; stage t's graph is the union of batches
    0..t (cumulative)."""
    rng = np.random.default_rng(seed + 7919)
    order = rng.permutation(edges.shape[0])
    cuts = np.linspace(0, edges.shape[0], stages + 1).astype(np.int64)
    return [np.ascontiguousarray(edges[order[cuts[t]:cuts[t + 1]]]) for t in range(stages)]


def random_edges(rng: np.random.Generator, n: int, e: int) -> np.ndarray:
    """Uniform random edge list (with self loops / duplicates) for adversarial tests."""
    return rng.integers(0, n, size=(e, 2), dtype=np.int64).astype(np.int32)
