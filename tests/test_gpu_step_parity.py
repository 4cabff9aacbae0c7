"""GPU parity of the production world-1 step -- the exact launch sequence
bench.py times (lmscale_step: S1 grouping + S4 with S6 folded in, eager and
CUDA-graph replay) -- and of the world-1 collective sync, against the CPU
oracle on WHOLE matrices at BASELINE.json's full sizes.

At world 1 the paper's steps 3-6 are identities (I = J, I^ = J^, M = Delta^,
M^ = M), so the oracle side is steps 1-2 (unique_local,
reduce_local, fp64) and step 7's definition E[I^[r]] - lr * M^[r].
Every row of I^ is compared, and every other row of E must be bit-identical
to E0 (checked on the device, where synth regenerates E0 bit-exactly).
Tolerances: tests/tolerances.py (INT bit-exact; SIGNED 1e-5 * A).

Edge cases of the S4 kernel (segsum.cu): K = 1, all ids equal (one run cut
by every range edge), all distinct, ragged K, a row wider than one column
block, dims that are not a multiple of 4 (the unstaged path), and the staged
G > 1 path with zero rows.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.tolerances import check_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lm():
    from paper_1810_10045_b200 import lmscale
    return lmscale


def dev():
    return torch.device("cuda", 0)


def u32(t):
    return t.view(torch.int32).cpu().numpy().view(np.uint32)


def oracle_world1(J, Dnp):
    """Steps 1-2 in fp64: J^, counts, M^ (= Delta^ at G = 1) and
    the summation-error scale A (the same sums over |Delta|)."""
    Jhat, counts, inverse = oracle.unique_local(J)
    Mhat64 = oracle.reduce_local(Dnp, inverse, Jhat.size)
    A = oracle.reduce_local(np.abs(Dnp), inverse, Jhat.size)
    return Jhat, counts, inverse, Mhat64, A


def check_table(E, E0_dev, Jhat, Mhat64, A, cfg, mode, lr, what):
    rows = torch.from_numpy(Jhat.astype(np.int64)).to(dev())
    got = E[rows].cpu().numpy()
    E0r = synth.table_rows(cfg.V, cfg.D, mode, Jhat).numpy().astype(np.float64)
    ref = E0r - lr * Mhat64
    if mode == "int":
        check_rows(got, ref, None, "int", f"{what} E rows")
    else:
        check_rows(got, ref, np.abs(E0r) + lr * A, "signed", f"{what} E rows")
    # every row outside I^ untouched, bit for bit
    mask = torch.ones(cfg.V, dtype=torch.bool, device=dev())
    mask[rows] = False
    assert torch.equal(E[mask], E0_dev[mask]), f"{what}: an untouched row changed"


FULL = [("1b", "signed"), ("1b", "int"), ("char", "signed"), ("amazon", "signed"),
        ("tieba", "signed"), ("tieba", "int")]


@pytest.mark.parametrize("graph", [False, True], ids=["eager", "graph"])
@pytest.mark.parametrize("name,mode", FULL, ids=[f"{a}-{b}" for a, b in FULL])
def test_world1_step_whole_matrix(lm, name, mode, graph):
    cfg = synth.CONFIGS[name]
    lr = synth.default_lr(mode)
    J = synth.ids_for(cfg, 0)
    ids = torch.from_numpy(J.view(np.int32)).to(dev())
    grad = synth.grad_values(cfg.K, cfg.D, mode, device=dev())
    E0 = synth.table_values(cfg.V, cfg.D, mode, device=dev())
    E = E0.clone()
    ctx = lm.Context(cfg.V, cfg.K, cfg.D, flags=lm.FLAG_GRAPH if graph else 0)
    if graph:   # first call captures and launches; reset, then a pure replay
        ctx.step(ids, grad, E, lr)
        torch.cuda.synchronize()
        E.copy_(E0)
    ctx.step(ids, grad, E, lr)
    torch.cuda.synchronize()
    st = ctx.stats()
    Jhat, counts, _, Mhat64, A = oracle_world1(J, grad.cpu().numpy())
    assert st["u_global"] == Jhat.size and st["u_local"] == Jhat.size
    # byte accounting of the folded step (S4 reads Delta, RMW of each E row)
    assert st["bytes_scatter"] == 4 * cfg.K * cfg.D + 8 * Jhat.size * cfg.D
    assert st["bytes_update"] == 0 and st["bytes_grad_allreduce"] == 0
    check_table(E, E0, Jhat, Mhat64, A, cfg, mode, lr, f"{name} {mode} graph={graph}")
    # the borrowed view after a step that consumed M: no rows
    sg = ctx.sparse_grad()
    assert sg.rows is None and sg.num_unique == Jhat.size
    np.testing.assert_array_equal(u32(sg.ids), Jhat)
    ctx.close()


@pytest.mark.parametrize("name", ["1b", "char", "amazon", "tieba"])
def test_world1_sync_whole_matrix(lm, name):
    """lmscale_sync_embedding_grad at world 1: I^, the global counts and
    every row of M^ against the oracle."""
    cfg = synth.CONFIGS[name]
    mode = "signed"
    J = synth.ids_for(cfg, 0)
    grad = synth.grad_values(cfg.K, cfg.D, mode, device=dev())
    ctx = lm.Context(cfg.V, cfg.K, cfg.D)
    sg = ctx.sync(torch.from_numpy(J.view(np.int32)).to(dev()), grad)
    torch.cuda.synchronize()
    Jhat, counts, _, Mhat64, A = oracle_world1(J, grad.cpu().numpy())
    np.testing.assert_array_equal(u32(sg.ids), Jhat)
    np.testing.assert_array_equal(sg.counts.cpu().numpy(), counts)
    check_rows(sg.rows.cpu().numpy(), Mhat64, A, mode, f"{name} M^")
    st = ctx.stats()
    assert st["bytes_scatter"] == 4 * cfg.K * cfg.D + 4 * Jhat.size * cfg.D
    ctx.close()


def test_graph_replay_equals_eager_bit_exact(lm):
    """INT mode: every partial sum is exact, so eager and graph replays give
    the same bits in any summation order (the grouping's run order is the
    arrival order of S1's tickets: DESIGN.md R18)."""
    cfg = synth.CONFIGS["1b"]
    J = synth.ids_for(cfg, 0)
    ids = torch.from_numpy(J.view(np.int32)).to(dev())
    grad = synth.grad_values(cfg.K, cfg.D, "int", device=dev())
    E0 = synth.table_values(cfg.V, cfg.D, "int", device=dev())
    a, b = E0.clone(), E0.clone()
    eager = lm.Context(cfg.V, cfg.K, cfg.D)
    graph = lm.Context(cfg.V, cfg.K, cfg.D, flags=lm.FLAG_GRAPH)
    for _ in range(3):
        eager.step(ids, grad, a, 2.0 ** -4)
        graph.step(ids, grad, b, 2.0 ** -4)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    # a staged call between replays dirties the presence bitmap: the next
    # replay must still be exact
    graph.unique(ids, want_outputs=False)
    graph.step(ids, grad, b, 2.0 ** -4)
    eager.step(ids, grad, a, 2.0 ** -4)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    eager.close()
    graph.close()


def _small_world1(lm, V, J, D, mode, graph=False):
    lr = synth.default_lr(mode)
    K = len(J)
    grad = synth.grad_values(K, D, mode, device=dev())
    E0 = synth.table_values(V, D, mode, device=dev())
    E = E0.clone()
    ctx = lm.Context(V, K, D, flags=lm.FLAG_GRAPH if graph else 0)
    ctx.step(torch.from_numpy(np.asarray(J, np.uint32).view(np.int32)).to(dev()), grad, E, lr)
    torch.cuda.synchronize()
    Eo = E0.cpu().numpy().copy()
    ref = oracle.sync_unique([np.asarray(J, np.uint32)], [grad.cpu().numpy()], Eo, lr)
    if mode == "int":
        np.testing.assert_array_equal(E.cpu().numpy(), Eo)
    else:
        cfg = synth.Config("edge", V=V, K=K, D=D)
        A = oracle.abs_scale([np.asarray(J, np.uint32)], [grad.cpu().numpy()], ref["Ihat"])
        check_table(E, E0, ref["Ihat"], ref["Mhat64"], A, cfg, mode, lr, "edge")
    ctx.close()


EDGE = [
    ("K=1", 50, np.array([7], np.uint32), 64),
    ("K=2-same", 50, np.array([3, 3], np.uint32), 64),
    ("all-equal", 100, np.full(40_000, 42, np.uint32), 64),
    ("all-equal-wide", 100, np.full(9000, 99, np.uint32), 512),
    ("all-distinct", 70_000, np.random.default_rng(1).permutation(70_000)[:65_537].astype(np.uint32), 32),
    ("ragged", 50_000, synth.zipf_ids(50_000, 1.0, 4096 * 3 + 17), 128),
    ("two-col-blocks", 3000, synth.zipf_ids(3000, 1.0, 3001), 2052),
    ("4096-wide", 3000, synth.zipf_ids(3000, 1.0, 1500), 4096),
    ("dim-3", 3000, synth.zipf_ids(3000, 1.0, 2500), 3),
    ("dim-37", 3000, synth.zipf_ids(3000, 1.0, 2500), 37),
    ("dim-1", 300, synth.zipf_ids(300, 1.0, 5000), 1),
    ("vocab-2^32-1", 2**32 - 1, np.random.default_rng(2).integers(0, 2**32 - 1, 3000,
                                                                   dtype=np.uint64).astype(np.uint32), 16),
]


@pytest.mark.parametrize("mode", ["int", "signed"])
@pytest.mark.parametrize("name,V,J,D", EDGE, ids=[e[0] for e in EDGE])
def test_world1_step_edge_cases(lm, name, V, J, D, mode):
    if V == 2**32 - 1:
        pytest.skip("a 2^32-1 x D table does not fit; the id path is covered by the S1 tests")
    _small_world1(lm, V, J, D, mode)


def test_world1_step_edge_graph(lm):
    _small_world1(lm, 100, np.full(40_000, 42, np.uint32), 64, "int", graph=True)


@pytest.mark.parametrize("D", [3, 64, 2052])
def test_staged_scatter_global_layout_zero_rows(lm, D):
    """G = 3 emulated through the staged ABI: S4 writes M_g in the global slot
    layout (l2g), absent slots exactly +0, present rows bit-exact in
    INT mode."""
    V, K, G = 4000, 3001, 3
    J = [synth.zipf_ids(V, 1.0, K, rank=g) for g in range(G)]
    Dl = [synth.grad_values(K, D, "int", rank=g) for g in range(G)]
    ctx = lm.Context(V, K, D, world=G, flags=lm.FLAG_NO_COMM)
    I = torch.from_numpy(np.concatenate(J).view(np.int32)).to(dev())
    ref = oracle.sync_unique(J, [d.numpy() for d in Dl], np.zeros((V, D), np.float32), 1.0)
    for g in range(G):
        ctx.unique(torch.from_numpy(J[g].view(np.int32)).to(dev()), want_outputs=False)
        ctx.global_unique(I)
        ctx.scatter_expand(Dl[g].to(dev()))
        sg = ctx.sparse_grad()
        assert sg.counts is None   # the staged calls do not exchange counts
        np.testing.assert_array_equal(sg.rows.cpu().numpy(), ref["M"][g].astype(np.float32))
    ctx.close()


def test_id_range_error_leaves_everything_untouched(lm):
    ctx = lm.Context(1000, 5000, 64)
    J = synth.zipf_ids(1000, 1.0, 5000)
    J[1234] = 1000
    E = torch.ones(1000, 64, device=dev())
    g = torch.ones(5000, 64, device=dev())
    ctx.step(torch.from_numpy(J.view(np.int32)).to(dev()), g, E, 0.5)
    torch.cuda.synchronize()
    assert torch.equal(E, torch.ones(1000, 64, device=dev()))
    with pytest.raises(lm.LmscaleError) as e:
        ctx.sparse_grad()
    assert e.value.status == lm.ID_RANGE
    # the next good step is exact (wcount / bitmap invariants restored)
    J[1234] = 3
    ctx.step(torch.from_numpy(J.view(np.int32)).to(dev()), g, E, 0.5)
    torch.cuda.synchronize()
    Eo = np.ones((1000, 64), np.float32)
    oracle.sync_unique([J], [g.cpu().numpy()], Eo, 0.5)
    np.testing.assert_array_equal(E.cpu().numpy(), Eo)
    ctx.close()


def _random_w1(n=24, seed=18101005):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        out.append((i, int(rng.choice([1, 2, 31, 33, 1000, 40000, 300000])),
                    int(rng.choice([1, 2, 7, 300, 2049, 5000, 70000])),
                    int(rng.choice([1, 3, 4, 17, 64, 100, 512, 516, 2048])),
                    float(rng.choice([0.5, 1.0, 1.5])), bool(rng.integers(0, 2))))
    return out


@pytest.mark.parametrize("i,V,K,D,s,graph", _random_w1(),
                         ids=[f"case{c[0]}-V{c[1]}-K{c[2]}-D{c[3]}-s{c[4]}-{'graph' if c[5] else 'eager'}"
                              for c in _random_w1()])
def test_world1_step_random_shapes(lm, i, V, K, D, s, graph):
    """Seeded random shapes for the world-1 step (S1 + S4 with S6 folded;
    the scalar kernel for dim % 4 != 0; vocab from 1 id; K from 1 token;
    ranges cut inside runs of every length), eager or CUDA-graph replay,
    INT mode: the whole table bit-exact against the oracle's steps 1-7."""
    lr = synth.default_lr("int")
    J = synth.zipf_ids(V, s, K, step=i)
    g = synth.grad_values(K, D, "int", step=i)
    E0 = synth.table_values(V, D, "int", device=dev())
    E = E0.clone()
    ctx = lm.Context(V, K, D, flags=lm.FLAG_GRAPH if graph else 0)
    ids = torch.from_numpy(J.view(np.int32)).to(dev())
    gd = g.to(dev())
    for _ in range(2):
        ctx.step(ids, gd, E, lr)
    torch.cuda.synchronize()
    Eo = E0.cpu().numpy().copy()
    for _ in range(2):
        oracle.sync_unique([J], [g.numpy()], Eo, lr)
    np.testing.assert_array_equal(E.cpu().numpy(), Eo)
    ctx.close()
