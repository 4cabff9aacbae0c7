"""Pins for the seeding oracle (Sec. 3.2; R16).

The draw stream is pinned by SplitMix64's published outputs, by the
distributional facts of uniform sampling without replacement (chi-square of
the marginal, pairwise inclusion, the hypergeometric union size of two
independent seeds) and by its structural invariants (distinct, in range,
S = V gives a permutation, prefix property).  The seed plan is pinned by the
SPEC's G = 64 group counts and the paper's policies.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "seeding.json")))


def test_mix64_is_splitmix64():
    gamma = 0x9E3779B97F4A7C15
    want = [int(x, 16) for x in GOLD["splitmix64_state0"]]
    got = [oracle.mix64((k * gamma) % 2**64) for k in range(3)]
    assert got == want


@pytest.mark.parametrize("policy", sorted(GOLD["group_counts_G64"]))
def test_group_counts_g64(policy):
    seeds, n = oracle.plan_seeds(64, policy, alpha=0.64, master_seed=7)
    assert n == GOLD["group_counts_G64"][policy]
    assert len(set(seeds)) == n


@pytest.mark.parametrize("G", [1, 2, 3, 4, 5, 8, 16, 64, 100])
@pytest.mark.parametrize("policy", oracle.SEED_POLICIES)
def test_plan_invariants(G, policy):
    seeds, n = oracle.plan_seeds(G, policy, alpha=0.64, master_seed=3)
    assert 1 <= n <= G and len(seeds) == G
    if G == 1:
        assert n == 1
    if policy == "distinct":
        assert n == G
    if policy == "same":
        assert n == 1
    # contiguous blocks of near-equal size, one seed per block
    blocks = [list(g) for _, g in __import__("itertools").groupby(seeds)]
    assert len(blocks) == n == len(set(seeds))
    sizes = [len(b) for b in blocks]
    assert max(sizes) - min(sizes) <= 1


def test_plan_monotone_in_g_and_ordered():
    """counts monotone in G; same <= log10 <= ln <= log2 <= power <= distinct for G >= 16."""
    order = ["same", "log10", "loge", "log2", "power", "distinct"]
    prev = {p: 0 for p in order}
    for G in range(1, 130):
        ns = [oracle.plan_seeds(G, p)[1] for p in order]
        for p, n in zip(order, ns):
            assert n >= prev[p]
            prev[p] = n
        if G >= 16:
            assert ns == sorted(ns), (G, ns)


def test_bad_alpha():
    with pytest.raises(ValueError):
        oracle.plan_seeds(8, "power", alpha=0.0)


@pytest.mark.parametrize("V,S", [(1, 1), (10, 10), (1000, 1), (793_000, 1024), (2**32 - 1, 300)])
def test_draw_invariants(V, S):
    x = oracle.draw_samples(11, 5, S, V)
    assert x.size == S and np.unique(x).size == S and int(x.max()) < V
    if S == V:
        np.testing.assert_array_equal(np.sort(x), np.arange(V))
    # deterministic per (seed, step); prefix property (stream order)
    np.testing.assert_array_equal(oracle.draw_samples(11, 5, S, V), x)
    np.testing.assert_array_equal(oracle.draw_samples(11, 5, max(1, S // 2), V), x[:max(1, S // 2)])


def test_draws_differ_across_steps_and_seeds():
    a = oracle.draw_samples(1, 0, 64, 10**6)
    assert not np.array_equal(a, oracle.draw_samples(1, 1, 64, 10**6))
    assert not np.array_equal(a, oracle.draw_samples(2, 0, 64, 10**6))


def test_marginal_uniform_chi_square():
    """Each word is included with probability S/V (uniform w/o replacement)."""
    V, S, n = 50, 10, 4000
    counts = np.zeros(V)
    for t in range(n):
        counts[oracle.draw_samples(99, t, S, V)] += 1
    exp = n * S / V
    chi2 = ((counts - exp) ** 2 / exp).sum()
    assert chi2 < 49 + 6 * math.sqrt(2 * 49)          # ~6 sigma of chi2(49)


def test_pairwise_inclusion_is_without_replacement():
    """P(i and j both drawn) = S(S-1)/(V(V-1)) for a uniform S-subset."""
    V, S, n = 20, 5, 6000
    both = 0
    for t in range(n):
        x = set(oracle.draw_samples(5, t, S, V).tolist())
        both += (0 in x) and (1 in x)
    p = S * (S - 1) / (V * (V - 1))
    assert abs(both / n - p) < 6 * math.sqrt(p * (1 - p) / n)


def test_union_sizes():
    """Same seed: union = S exactly; two seeds: E|A u B| = 2S - S^2/V
    (hypergeometric overlap); never more than groups * S."""
    V, S = 10_000, 1000
    a = oracle.draw_samples(123, 4, S, V)
    assert np.union1d(a, oracle.draw_samples(123, 4, S, V)).size == S
    sizes = [np.union1d(oracle.draw_samples(2 * t, 4, S, V),
                        oracle.draw_samples(2 * t + 1, 4, S, V)).size for t in range(40)]
    exp = 2 * S - S * S / V
    sd = math.sqrt(S * (S / V) * (1 - S / V) * (V - S) / (V - 1))   # hypergeometric sd
    assert abs(np.mean(sizes) - exp) < 6 * sd / math.sqrt(len(sizes))
    assert max(sizes) <= 2 * S
