"""Pins for the oracle's random input (no GPU).

The paper fixes only the distribution, Theta ~ N(0, 1/d) (Alg. 1
l.2 PAPER.md:186); this build fixes Philox4x32-10 + Box-Muller (DESIGN.md
reading A11).  The oracle is pinned against a LIBRARY routine — cuRAND's own
Philox4_32_10 device-API code compiled for the host (tests/pins/curand_pin.cu)
— bit-exactly for the raw stream, and to float accuracy for curand_normal4,
plus closed forms of the transform at extreme draws and distribution tests.
"""
import math

import numpy as np
import pytest
from scipy import stats

import oracle
from conftest import np_ptr


def test_philox_block_matches_curand(curand_pin):
    rng = np.random.default_rng(7)
    for _ in range(2000):
        ctr = rng.integers(0, 2**32, size=4, dtype=np.uint64).astype(np.uint32)
        key = rng.integers(0, 2**32, size=2, dtype=np.uint64).astype(np.uint32)
        ref = np.zeros(4, dtype=np.uint32)
        curand_pin.pin_philox_block(np_ptr(ctr), np_ptr(key), np_ptr(ref))
        assert np.array_equal(oracle.philox4x32_10(ctr, key), ref)


@pytest.mark.parametrize("seed,sub", [(0, 0), (1234, 5), (2**40 + 17, 3), (99, 2**33 + 1)])
def test_stream_layout_matches_curand_init(curand_pin, seed, sub):
    """curand_init(seed, sub, 0) then curand4 x n  ==  oracle counter layout
    (lo b, hi b, lo sub, hi sub), key (lo seed, hi seed)."""
    n4 = 4096
    ref = np.zeros(4 * n4, dtype=np.uint32)
    curand_pin.pin_curand4(seed, sub, 0, n4, np_ptr(ref))
    assert np.array_equal(oracle.philox_bits(seed, sub, 4 * n4), ref)
    # and an offset into the stream: curand_init(seed, sub, 4*b)
    b = 123457
    ref2 = np.zeros(8, dtype=np.uint32)
    curand_pin.pin_curand4(seed, sub, 4 * b, 2, np_ptr(ref2))
    assert np.array_equal(oracle.philox_bits(seed, sub, 4 * (b + 2))[4 * b:], ref2)


def test_normal_matches_curand_normal4(curand_pin):
    n4 = 1 << 18
    ref = np.zeros(4 * n4, dtype=np.float32)
    curand_pin.pin_curand_normal4(42, 7, 0, n4, np_ptr(ref))
    x = oracle.normal(42, 7, 4 * n4)
    # cuRAND evaluates in fp32 (host libm sinf/cosf/logf); away from u -> 1
    # (where fp32 rounds u to 1) the two agree to fp32 accuracy.
    err = np.abs(x - ref.astype(np.float64))
    assert np.quantile(err, 0.999999) < 2e-5
    assert err.max() < 1e-3
    # pairing and sin/cos order (swaps would give O(1) errors)
    assert np.corrcoef(x[0::2], ref[0::2])[0, 1] > 0.999999


def test_box_muller_closed_forms():
    # r_even = 0 -> u = 2^-33 -> R = sqrt(-2 ln 2^-33) = sqrt(66 ln 2)
    R = math.sqrt(66.0 * math.log(2.0))
    # r_odd = 2^30 - 1/2 is not an integer; take r_odd = 2^30: v = (2^30 + .5) 2^-32
    v = (2**30 + 0.5) / 2**32
    n = oracle.box_muller(0, 2**30)
    assert n[0] == pytest.approx(R * math.sin(2 * math.pi * v), rel=1e-14)
    assert n[1] == pytest.approx(R * math.cos(2 * math.pi * v), rel=1e-12, abs=1e-15)
    # r_even = 2^32 - 1 -> u = 1 - 2^-33 -> R = sqrt(-2 ln(1 - 2^-33)) ~ 2^-16
    n = oracle.box_muller(2**32 - 1, 0)
    assert n[1] == pytest.approx(math.sqrt(-2.0 * math.log1p(-2.0**-33)), rel=1e-6)
    assert abs(n[0]) < 1e-13
    # r_odd = 2^31 -> v = 1/2 + 2^-33: sin(pi + tiny) < 0, cos ~ -1
    n = oracle.box_muller(2**31, 2**31)
    Rh = math.sqrt(-2.0 * math.log((2**31 + 0.5) / 2**32))
    assert n[1] == pytest.approx(-Rh, rel=1e-12)
    assert n[0] < 0


def test_normal_distribution_and_determinism():
    x = oracle.normal(3, 0, 1 << 20)
    assert abs(x.mean()) < 5.0 / math.sqrt(x.size)
    assert abs(x.var() - 1.0) < 0.01
    assert stats.kstest(x, "norm").pvalue > 1e-4
    assert np.array_equal(x, oracle.normal(3, 0, 1 << 20))
    y = oracle.normal(4, 0, 1 << 20)
    assert np.mean(x != y) > 0.99
    z = oracle.normal(3, 1, 1 << 20)  # another subsequence (streaming stage)
    assert np.mean(x != z) > 0.99


def test_theta_variance_is_one_over_d():
    """Alg. 1 l.2: Theta ~ N(0, 1/d) (reading A1); SPEC.md:179 (1/64 +- 10%)."""
    th = oracle.input_theta(0, 0, 10_000, 64)
    assert abs(th.var() - 1 / 64) < 0.1 / 64


def test_normal_at_matches_the_stream_and_curand(curand_pin):
    """normal_at (sampled elements, used at sizes where the stream is too large to draw) equals
    the pinned stream element by element, and cuRAND's curand_normal4 at an offset past 2^32 blocks."""
    x = oracle.normal(11, 2, 1 << 16)
    idx = np.random.default_rng(5).integers(0, 1 << 16, size=3000)
    assert np.array_equal(oracle.normal_at(11, 2, idx), x[idx])
    assert np.array_equal(oracle.normal_at(11, 2, np.arange(64)), x[:64])
    b = 2**32 + 12345  # block index beyond 32 bits: the counter's high word is used
    ref = np.zeros(8, dtype=np.float32)
    curand_pin.pin_curand_normal4(11, 2, 4 * b, 2, np_ptr(ref))
    got = oracle.normal_at(11, 2, 4 * b + np.arange(8))
    assert np.max(np.abs(got - ref.astype(np.float64))) < 2e-5
    with pytest.raises(oracle.OracleError):
        oracle.normal_at(11, 2, [-1])
