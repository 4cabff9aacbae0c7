"""Pins for the CPU oracle (oracle/): the oracle is checked against what the
paper and mathematics fix -- printed examples (tests/golden/, each cited),
library routines for the special cases they cover (numpy unique / add.at /
searchsorted), brute-force dense-vs-unique equivalence, closed
forms, and invariants.  CPU only."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from tests.tolerances import check_rows

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ goldens

def _tokenise_and_vocab(text):
    """Reading R14: lowercase whitespace split; vocab by descending count,
    ties lexicographic."""
    toks = text.lower().split()
    counts = {}
    for t in toks:
        counts[t] = counts.get(t, 0) + 1
    order = sorted(counts, key=lambda w: (-counts[w], w))
    vocab = {w: i for i, w in enumerate(order)}
    return toks, vocab


def test_to_be_or_not_to_be():
    g = gold("to_be.json")
    toks, vocab = _tokenise_and_vocab(g["text"])
    assert vocab == g["vocab"]
    J = [vocab[t] for t in toks]
    assert J == g["J"]
    Jhat, counts, inverse = oracle.unique_local(J)
    assert len(J) == g["tokens"] == 6
    assert Jhat.size == g["types"] == 4
    assert Jhat.tolist() == g["Jhat"]
    assert counts.tolist() == g["counts"]
    assert inverse.tolist() == g["inverse"]


def test_fig2_repeated_word_accumulates():
    g = gold("fig2_i_want_a_pen.json")
    J = np.array(g["J"], np.uint32)
    Jhat, counts, inverse = oracle.unique_local(J)
    assert Jhat.tolist() == g["Jhat"]
    assert counts.tolist() == g["counts"]
    rng = np.random.default_rng(0)
    delta = rng.integers(-8, 8, size=(6, 5)).astype(np.float32)
    dhat = oracle.reduce_local(delta, inverse, Jhat.size)
    u = Jhat.tolist().index(g["shared_row_word"])
    p3, p6 = g["shared_positions"]
    np.testing.assert_array_equal(dhat[u], delta[p3].astype(np.float64) + delta[p6])
    # the row of 'I' (4343) is its single token's gradient
    np.testing.assert_array_equal(dhat[Jhat.tolist().index(4343)], delta[0])


def test_fig3_cross_gpu_duplicate():
    g = gold("fig3_two_gpus.json")
    J = [np.array(j, np.uint32) for j in g["J"]]
    D = 4
    delta = [np.arange(8, dtype=np.float32).reshape(2, D) + 10 * r for r in range(2)]
    E = np.zeros((10000, D), np.float32)
    out = oracle.sync_unique(J, delta, E, lr=1.0)
    assert out["Ihat"].tolist() == g["Ihat"]
    assert out["Ug"] == g["Ug"]
    r = g["Ihat"].index(1234)
    want = sum(delta[gi][p].astype(np.float64) for gi, p in g["word_1234_contributors"])
    np.testing.assert_array_equal(out["Mhat64"][r], want)


def test_spec_goldens():
    g = gold("spec_goldens.json")
    for case in g["unique_local"]:
        Jhat, counts, inverse = oracle.unique_local(case["J"])
        assert Jhat.tolist() == case["Jhat"], case["cite"]
        assert inverse.tolist() == case["inverse"], case["cite"]
    for case in g["reduce_local"]:
        Jhat, _, inverse = oracle.unique_local(case["J"])
        dh = oracle.reduce_local(np.array(case["delta"], np.float32), inverse, Jhat.size)
        assert dh.tolist() == case["dhat"], case["cite"]
    for case in g["gather"]:
        assert oracle.allgather_ids(case["J"]).tolist() == case["I"], case["cite"]
    for case in g["unique_global"]:
        Ihat, _ = oracle.unique_global(case["I"])
        assert Ihat.tolist() == case["Ihat"] and Ihat.size == case["Ug"], case["cite"]
    for case in g["scatter_expand"]:
        M = oracle.scatter_expand(np.array(case["dhat"], np.float64),
                                  np.array(case["l2g"], np.int32), case["Ug"])
        assert M.tolist() == case["M"], case["cite"]
    c = g["sync_unique_g1"]
    D = 3
    E = np.full((4, D), 0.25, np.float32)
    E0 = E.copy()
    oracle.sync_unique([np.array(c["J"], np.uint32)], [np.full((1, D), c["delta_row"], np.float32)],
                       E, lr=c["lr"])
    np.testing.assert_array_equal(E[0], E0[0] - 1.0)
    np.testing.assert_array_equal(E[1:], E0[1:])
    c = g["sync_unique_all7"]
    J = [np.full(5, c["word"], np.uint32) for _ in range(c["G"])]
    out = oracle.sync_unique(J, [np.ones((5, 2), np.float32)] * c["G"],
                             np.zeros((10, 2), np.float32), lr=1.0)
    assert out["Ug"] == c["Ug"]
    assert out["Mhat"].tolist() == [[10.0, 10.0]]


def test_worked_example_memory():
    g = gold("worked_example.json")
    plan = oracle.complexity_plan(g["G"], g["K"], g["D"], g["alpha"], g["elem_bytes"])
    assert round(plan["baseline_bytes"] / 1e9, 1) == g["baseline_GB"]
    assert round(plan["unique_grad_bytes"] / 1e9, 3) == g["unique_GB"]
    assert round(plan["saving_factor_grad_only"]) == g["saving"]


# ------------------------------------------------------ library cross-checks

@pytest.mark.parametrize("V,K", [(50, 1), (50, 300), (1000, 4096), (2**31, 777)])
def test_unique_local_vs_numpy(V, K):
    rng = np.random.default_rng(V + K)
    J = rng.integers(0, V, size=K, dtype=np.uint64).astype(np.uint32)
    Jhat, counts, inverse = oracle.unique_local(J)
    u, inv, cnt = np.unique(J, return_inverse=True, return_counts=True)
    np.testing.assert_array_equal(Jhat, u)
    np.testing.assert_array_equal(inverse, inv)
    np.testing.assert_array_equal(counts, cnt)
    assert counts.sum() == K
    np.testing.assert_array_equal(Jhat[inverse], J)
    assert np.all(np.diff(Jhat.astype(np.int64)) > 0)


def test_reduce_and_scatter_vs_numpy_add_at():
    rng = np.random.default_rng(3)
    V, K, D = 97, 513, 7
    J = rng.integers(0, V, size=K).astype(np.uint32)
    delta = rng.standard_normal((K, D)).astype(np.float32)
    Jhat, _, inverse = oracle.unique_local(J)
    dh = oracle.reduce_local(delta, inverse, Jhat.size)
    dense = np.zeros((V, D), np.float64)
    np.add.at(dense, J.astype(np.int64), delta.astype(np.float64))
    np.testing.assert_allclose(dh, dense[Jhat], rtol=1e-13, atol=1e-13)
    Ihat = np.union1d(Jhat, np.array([0, 5, 96], np.uint32)).astype(np.uint32)
    l2g, slot = oracle.remap(Jhat, Ihat, inverse)
    np.testing.assert_array_equal(l2g, np.searchsorted(Ihat, Jhat))
    np.testing.assert_array_equal(Ihat[slot], J)
    M = oracle.scatter_expand(dh, l2g, Ihat.size)
    np.testing.assert_allclose(M, dense[Ihat], rtol=1e-13, atol=1e-13)
    absent = ~np.isin(Ihat, Jhat)
    assert np.all(M[absent] == 0.0)


def test_unique_global_vs_numpy():
    rng = np.random.default_rng(5)
    I = rng.integers(0, 5000, size=20000).astype(np.uint32)
    Ihat, gc = oracle.unique_global(I)
    u, c = np.unique(I, return_counts=True)
    np.testing.assert_array_equal(Ihat, u)
    np.testing.assert_array_equal(gc, c)


# -------------------------------------------- brute force: dense == unique

def _instance(rng, mode):
    G = int(rng.choice([1, 2, 4, 8]))
    V = int(rng.integers(1, 1001))
    K = int(rng.integers(1, 65))
    D = int(rng.integers(1, 17))
    J = [rng.integers(0, V, size=K).astype(np.uint32) for _ in range(G)]
    if mode == "int":
        delta = [rng.integers(-8, 8, size=(K, D)).astype(np.float32) for _ in range(G)]
        E0 = (rng.integers(-16, 16, size=(V, D)) / 16).astype(np.float32)
    else:
        delta = [rng.uniform(-1, 1, size=(K, D)).astype(np.float32) for _ in range(G)]
        E0 = rng.uniform(-1, 1, size=(V, D)).astype(np.float32)
    return G, V, K, D, J, delta, E0


@pytest.mark.parametrize("mode", ["int", "signed"])
def test_dense_equals_unique_bruteforce(mode):
    """uniqueness 'only changes the flow of computation'; SPEC AC1
    (S:582): 200 instances, G in {1,2,4,8}, V<=1000, K<=64, D<=16."""
    rng = np.random.default_rng(181010045 if mode == "int" else 7)
    lr = 2.0 ** -4 if mode == "int" else 0.1
    for _ in range(200):
        G, V, K, D, J, delta, E0 = _instance(rng, mode)
        Ed = oracle.sync_dense(J, delta, E0.copy(), lr)
        Eu = E0.copy()
        out = oracle.sync_unique(J, delta, Eu, lr)
        if mode == "int":
            np.testing.assert_array_equal(Ed, Eu)
        else:
            # both round an fp64 result once; the fp64 sums differ only in order
            np.testing.assert_allclose(Ed, Eu, rtol=0, atol=1e-6)
        # invariants
        Ihat = out["Ihat"]
        assert len(set(Ihat.tolist())) == Ihat.size == out["Ug"]          # race-free witness
        assert out["Ug"] <= min(sum(r["Jhat"].size for r in out["ranks"]), V)
        assert max(r["Jhat"].size for r in out["ranks"]) <= out["Ug"]
        untouched = np.setdiff1d(np.arange(V), Ihat)
        np.testing.assert_array_equal(Eu[untouched], E0[untouched])


def test_conservation_of_summed_gradient():
    """Per-type conservation (definition) and global conservation:
    sum_r M^[r] == sum_{g,p} Delta_g[p]; type_gradient recomputes each row."""
    cfg = synth.CONFIGS["tiny"]
    J = [synth.ids_for(cfg, g) for g in range(cfg.G)]
    delta = [synth.grad_values(cfg.K, cfg.D, "int", rank=g).numpy() for g in range(cfg.G)]
    out = oracle.sync_unique(J, delta, np.zeros((cfg.V, cfg.D), np.float32), 2.0 ** -4)
    tot = sum(d.astype(np.float64).sum(0) for d in delta)
    np.testing.assert_array_equal(out["Mhat64"].sum(0), tot)
    gc = np.zeros(out["Ug"], np.int64)
    for r in out["ranks"]:
        np.add.at(gc, r["l2g"], r["counts"])
    np.testing.assert_array_equal(gc, out["gcounts"])
    assert out["gcounts"].sum() == cfg.G * cfg.K
    rng = np.random.default_rng(1)
    for r in rng.choice(out["Ug"], 16, replace=False):
        row, A, n = oracle.type_gradient(J, delta, out["Ihat"][r])
        np.testing.assert_array_equal(row, out["Mhat64"][r])
        assert n == out["gcounts"][r]


def test_tolerance_metric_signed():
    cfg = synth.CONFIGS["tiny"]
    J = [synth.ids_for(cfg, g) for g in range(cfg.G)]
    delta = [synth.grad_values(cfg.K, cfg.D, "signed", rank=g).numpy() for g in range(cfg.G)]
    out = oracle.sync_unique(J, delta, np.zeros((cfg.V, cfg.D), np.float32), 0.1)
    A = oracle.abs_scale(J, delta, out["Ihat"])
    # a sequential fp32 sum must sit inside the metric
    Ms = np.zeros((out["Ug"], cfg.D), np.float32)
    for g in range(cfg.G):
        for p in range(cfg.K):
            Ms[out["ranks"][g]["slot"][p]] += delta[g][p]
    check_rows(Ms, out["Mhat64"], A, "signed", "sequential fp32")


def test_lookup_vs_numpy_and_special_cases():
    """Forward lookup against numpy fancy indexing; identity ids
    give E back; equal ids repeat one row; ids >= V give zero rows."""
    rng = np.random.default_rng(4)
    E = rng.standard_normal((97, 13)).astype(np.float32)
    J = rng.integers(0, 97, 500).astype(np.uint32)
    np.testing.assert_array_equal(oracle.lookup(E, J), E[J])
    np.testing.assert_array_equal(oracle.lookup(E, np.arange(97, dtype=np.uint32)), E)
    out = oracle.lookup(E, np.full(5, 3, np.uint32))
    assert (out == E[3]).all()
    out = oracle.lookup(E, np.array([1, 97, 2**32 - 1], np.uint32))
    np.testing.assert_array_equal(out[0], E[1])
    assert (out[1:] == 0).all()


def test_threaded_oracle_is_bit_identical():
    """The all-cores timing variant (step 2 split over column blocks) computes
    the same seven steps with the same per-element order: bit-identical."""
    rng = np.random.default_rng(11)
    J = [synth.zipf_ids(4000, 1.0, 2500, rank=g) for g in range(3)]
    Dl = [rng.standard_normal((2500, 29)).astype(np.float32) for _ in range(3)]
    a = oracle.sync_unique(J, Dl, np.zeros((4000, 29), np.float32), 0.1)
    for t in (1, 4, 29, 64):
        b = oracle.sync_unique_threads(J, Dl, np.zeros((4000, 29), np.float32), 0.1, t)
        assert np.array_equal(a["Mhat64"], b["Mhat64"]) and np.array_equal(a["E"], b["E"])
