"""The equivalence planner: binomial tail
against exact rational arithmetic, the miss bound's examples and
monotonicity, and the bound's validity against a Monte-Carlo multinomial
simulation at the planned per-shard depth (host math, no GPU)."""
from fractions import Fraction
from math import comb

import pytest

import paper_1209_0410_b200 as H


def exact_tail(trials, p, phi):
    p = Fraction(p)
    return sum(comb(trials, k) * p ** k * (1 - p) ** (trials - k) for k in range(phi + 1, trials + 1))


@pytest.mark.parametrize("trials", [1, 2, 7, 16, 33, 64])
@pytest.mark.parametrize("shards", [2, 3, 4, 8, 16])
def test_binomial_tail_matches_exact_rationals(trials, shards):
    for phi in range(0, trials + 2):
        want = float(exact_tail(trials, Fraction(1, shards), phi))
        got = H.binomial_tail(trials, 1.0 / shards, phi)
        assert abs(got - want) <= 1e-12 + 1e-9 * want, (trials, shards, phi, got, want)


def test_spec_examples():
    assert H.binomial_tail(10, 0.3, 10) == 0.0          # phi >= Phi -> 0
    assert H.binomial_tail(1, 0.5, 0) == pytest.approx(0.5)
    assert H.miss_bound(50, 1, 50) == 0.0                # l = 1, phi = Phi
    for shards in (2, 4, 8):
        assert H.miss_bound(50, shards, 50) == 0.0       # phi = Phi: no loss
    assert H.plan_depth(128, 1, 0.02) == 128             # one shard: phi = Phi
    with pytest.raises(ValueError):
        H.binomial_tail(5, 0.0, 1)


def test_miss_bound_monotone():
    for shards in (2, 4, 8, 16):
        prev = 2.0
        for phi in range(0, 129):
            b = H.miss_bound(128, shards, phi)
            assert 0.0 <= b <= 1.0 and b <= prev + 1e-15
            prev = b
        for Phi in range(20, 200, 9):  # non-decreasing in Phi for fixed phi
            assert H.miss_bound(Phi, shards, 20) <= H.miss_bound(Phi + 9, shards, 20) + 1e-15


@pytest.mark.parametrize("shards", [2, 4, 8, 16])
def test_planned_depth_bound_holds_monte_carlo(shards):
    """Phi=128, target 2 %: phi* is minimal (phi* - 1 misses the target) and
    the empirical miss frequency at phi* is below the bound + 3 sigma."""
    phi = H.plan_depth(128, shards, 0.02)
    assert H.miss_bound(128, shards, phi) <= 0.02
    assert phi == 128 or H.miss_bound(128, shards, phi - 1) > 0.02
    trials = 400_000
    freq = H.monte_carlo_miss(128, shards, phi, trials, seed=shards)
    bound = H.miss_bound(128, shards, phi)
    sigma = (max(bound, 1e-6) * (1 - bound) / trials) ** 0.5
    assert freq <= bound + 3 * sigma, (shards, phi, freq, bound)


def test_monte_carlo_degenerate_cases():
    assert H.monte_carlo_miss(30, 4, 30, 1000) == 0.0    # phi >= Phi
    assert H.monte_carlo_miss(30, 1, 29, 100) == 1.0     # one shard always holds Phi
    assert H.monte_carlo_miss(30, 1, 30, 100) == 0.0


def test_bench_shard_depths():
    """The per-shard depths bench.py uses for configs[2] at D = 350."""
    assert [H.shard_probe_depth(350, g) for g in (2, 4, 8)] == [226, 134, 80]
