"""GPU parity of the G > 1 kernels on ONE GPU (lmscale_emulate_step).

The world-G step of lmscale_step's P2P path -- S1 on every rank,
the J^-set exchange S3 (steps 3-4, as peer presence bitmaps,
DESIGN.md R17), S4 in the local-slot layout, the fused S5+S6
exchange + row update (steps 6-7: k_p2p_bulk; k_p2p_update for
dim % 4 != 0; compressed, Sec. 3.3 / R15: both phases of k_p2p_update_c) --
runs on G contexts of one device: the same kernels, with the NCCL window
replaced by the other contexts' buffers and the cross-rank barriers by launch
order.  Every replica of E is compared with the oracle (oracle.sync_unique,
steps 1-7) element by element: INT mode bit-exact, SIGNED within
tests/tolerances.py, and all replicas bit-identical.

The real multi-process runs of the same kernels over NVLink are
tests/test_multigpu.py (they need 2-4 GPUs); this file keeps the G > 1 rows
of SURVEY 8(a) under test on a one-GPU box.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.tolerances import check_compressed_rows, check_rows, compressed_tol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lm():
    from paper_1810_10045_b200 import lmscale
    return lmscale


def dev():
    return torch.device("cuda", 0)


def ids_dev(J):
    return torch.from_numpy(np.asarray(J, np.uint32).view(np.int32)).to(dev())


def make(lm, cfg, G, F=0.0, fmt="fp16"):
    ctxs = [lm.Context(cfg.V, cfg.K, cfg.D, world=G, rank=r, flags=lm.FLAG_NO_COMM)
            for r in range(G)]
    for c in ctxs:
        if F > 0:
            c.set_compression(F)
            c.set_codec(fmt)
    return ctxs


def close(ctxs):
    for c in ctxs:
        c.close()
    torch.cuda.empty_cache()


def check_replicas(tables, what):
    for r in range(1, len(tables)):
        assert torch.equal(tables[r], tables[0]), f"{what}: replica {r} differs from replica 0"


def oracle_mhat(J, Dl, want_A=True):
    """Steps 1-6 in fp64 without a table: I^, M^ and the
    summation-error scale A (the same steps over |Delta|; None if not wanted)."""
    ranks = []
    for Jg, Dg in zip(J, Dl):
        Jhat, _, inverse = oracle.unique_local(Jg)
        ranks.append((Jhat, inverse, oracle.reduce_local(Dg, inverse, Jhat.size)))
    Ihat, _ = oracle.unique_global(oracle.allgather_ids(J))
    Ms = []
    for Jhat, inverse, dhat in ranks:
        l2g, _ = oracle.remap(Jhat, Ihat, inverse)
        Ms.append(oracle.scatter_expand(dhat, l2g, Ihat.size))
    Mhat64 = oracle.allreduce_sum(Ms)
    del Ms
    A = oracle.abs_scale(J, Dl, Ihat) if want_A else None
    return Ihat, Mhat64, A


def run(lm, cfg, G, mode, F=0.0, fmt="fp16"):
    lr = synth.default_lr(mode)
    if F > 0:
        lr = float(np.float32(lr))  # fp32 lr on both sides (the fma rounds once)
    J = [synth.ids_for(cfg, g) for g in range(G)]
    Dl = [synth.grad_values(cfg.K, cfg.D, mode, rank=g) for g in range(G)]
    E0 = synth.table_values(cfg.V, cfg.D, mode, device=dev())
    tables = [E0.clone() for _ in range(G)]
    ctxs = make(lm, cfg, G, F, fmt)
    lm.emulate_step(ctxs, [ids_dev(j) for j in J], [d.to(dev()) for d in Dl], tables, lr)
    torch.cuda.synchronize()
    return ctxs, J, Dl, E0, tables, lr


SMALL = [(2, "int", 64), (2, "signed", 64), (3, "int", 64), (4, "int", 64), (4, "signed", 64),
         (8, "int", 64), (8, "signed", 64), (2, "int", 37), (3, "signed", 37), (2, "int", 2052),
         (4, "int", 2052)]


@pytest.mark.parametrize("G,mode,D", SMALL, ids=[f"G{g}-{m}-D{d}" for g, m, d in SMALL])
def test_emulated_step_whole_table(lm, G, mode, D):
    """tiny-shaped inputs (Zipf ids, several tiles, ragged tails); D = 37
    takes the unstaged k_p2p_update<float>, D = 2052 five column blocks of
    k_p2p_bulk (the last one 16 bytes wide)."""
    base = synth.CONFIGS["tiny"]
    cfg = synth.Config("emu", V=base.V, K=base.K if D <= 64 else 1500, D=D, G=G)
    ctxs, J, Dl, E0, tables, lr = run(lm, cfg, G, mode)
    Eo = E0.cpu().numpy().copy()
    ref = oracle.sync_unique(J, [d.numpy() for d in Dl], Eo, lr)
    got = tables[0].cpu().numpy()
    if mode == "int":
        np.testing.assert_array_equal(got, Eo)
    else:
        t = ref["Ihat"].astype(np.int64)
        A = oracle.abs_scale(J, [d.numpy() for d in Dl], ref["Ihat"])
        E0n = E0.cpu().numpy().astype(np.float64)
        check_rows(got[t], E0n[t] - lr * ref["Mhat64"], np.abs(E0n[t]) + lr * A, "signed",
                   f"G={G} D={D} E rows")
        untouched = np.setdiff1d(np.arange(cfg.V), t)
        np.testing.assert_array_equal(got[untouched], E0.cpu().numpy()[untouched])
    check_replicas(tables, f"G={G} {mode} D={D}")
    # I^, U_g and the global counts of every rank: the sparse-grad view after
    # the step (counts summed over the peers' S1 counts read from their windows)
    for c in ctxs:
        sg = c.sparse_grad()
        assert sg.num_unique == ref["Ug"]
        np.testing.assert_array_equal(sg.ids.cpu().numpy().view(np.uint32), ref["Ihat"])
        np.testing.assert_array_equal(sg.counts.cpu().numpy(), ref["gcounts"])
        assert sg.rows is None  # the fused exchange consumed M
    close(ctxs)


def test_emulated_second_step_and_all_equal(lm):
    """Two steps in a row on the same contexts (the presence bitmaps are
    rebuilt, the handshake-free S3 reads the new ones), then a batch where
    every rank holds only one word (one run cut by every S4 range edge, U_g = 1)."""
    cfg = synth.Config("emu", V=5000, K=3000, D=64, G=3)
    G, mode = 3, "int"
    ctxs, J, Dl, E0, tables, lr = run(lm, cfg, G, mode)
    lm.emulate_step(ctxs, [ids_dev(j) for j in J], [d.to(dev()) for d in Dl], tables, lr)
    torch.cuda.synchronize()
    Eo = E0.cpu().numpy().copy()
    for _ in range(2):
        oracle.sync_unique(J, [d.numpy() for d in Dl], Eo, lr)
    np.testing.assert_array_equal(tables[0].cpu().numpy(), Eo)
    check_replicas(tables, "two steps")
    J1 = [np.full(cfg.K, 4321, np.uint32) for _ in range(G)]
    lm.emulate_step(ctxs, [ids_dev(j) for j in J1], [d.to(dev()) for d in Dl], tables, lr)
    torch.cuda.synchronize()
    ref = oracle.sync_unique(J1, [d.numpy() for d in Dl], Eo, lr)
    assert ref["Ug"] == 1
    np.testing.assert_array_equal(tables[0].cpu().numpy(), Eo)
    check_replicas(tables, "all equal")
    close(ctxs)


def test_emulated_id_error_touches_nothing(lm):
    """An id >= vocab on one rank: ID_RANGE, and no replica is touched
    (every rank's fused kernel leaves before its first store)."""
    cfg = synth.Config("emu", V=5000, K=3000, D=64, G=2)
    G, mode = 2, "int"
    J = [synth.ids_for(cfg, g) for g in range(G)]
    J[1] = J[1].copy()
    J[1][1234] = cfg.V + 7
    Dl = [synth.grad_values(cfg.K, cfg.D, mode, rank=g) for g in range(G)]
    E0 = synth.table_values(cfg.V, cfg.D, mode, device=dev())
    tables = [E0.clone() for _ in range(G)]
    ctxs = make(lm, cfg, G)
    with pytest.raises(lm.LmscaleError) as ei:
        lm.emulate_step(ctxs, [ids_dev(j) for j in J], [d.to(dev()) for d in Dl], tables, 0.5)
    assert ei.value.status == lm.ID_RANGE
    for t in tables:
        assert torch.equal(t, E0)
    close(ctxs)


def test_emulated_rejects_mismatched_contexts(lm):
    cfg = synth.Config("emu", V=5000, K=300, D=8, G=2)
    a = lm.Context(cfg.V, cfg.K, cfg.D, world=2, rank=0, flags=lm.FLAG_NO_COMM)
    b = lm.Context(cfg.V, cfg.K, cfg.D, world=2, rank=0, flags=lm.FLAG_NO_COMM)  # rank 0 twice
    ids = ids_dev(synth.ids_for(cfg, 0))
    g = torch.zeros(cfg.K, cfg.D, device=dev())
    E = torch.zeros(cfg.V, cfg.D, device=dev())
    with pytest.raises(lm.LmscaleError) as ei:
        lm.emulate_step([a, b], [ids, ids], [g, g], [E, E.clone()], 1.0)
    assert ei.value.status == lm.INVALID_ARG
    a.close()
    b.close()


COMP = [(2, "int", 1.0, "fp16"), (2, "signed", 32.0, "fp16"), (4, "int", 1024.0, "fp16"),
        (4, "signed", 1.0, "fp16"), (3, "signed", 1.0, "bf16"), (8, "int", 1.0, "fp16")]


@pytest.mark.parametrize("G,mode,F,fmt", COMP, ids=[f"G{g}-{m}-F{f:g}-{c}" for g, m, f, c in COMP])
def test_emulated_compressed_exchange(lm, G, mode, F, fmt):
    """Sec. 3.3 (R15): the codec on each transfer, against
    oracle.sync_unique_compressed -- INT bit-exact over the whole table,
    float modes within compressed_tol; replicas bit-identical."""
    cfg = synth.CONFIGS["tiny"].with_(G=G)
    ctxs, J, Dl, E0, tables, lr = run(lm, cfg, G, mode, F, fmt)
    Eo = E0.cpu().numpy().copy()
    ref = oracle.sync_unique_compressed(J, [d.numpy() for d in Dl], Eo, lr, F, fmt)
    got = tables[0].cpu().numpy()
    if mode == "int":
        np.testing.assert_array_equal(got, Eo)
    else:
        t = ref["Ihat"].astype(np.int64)
        A = oracle.abs_scale(J, [d.numpy() for d in Dl], ref["Ihat"])
        E0n = E0.cpu().numpy()
        tol = lr * compressed_tol(A, F, G) * (8 if fmt == "bf16" else 1) + 2.0 ** -23 * np.abs(E0n[t])
        check_compressed_rows(got[t], Eo[t], tol, f"compressed G={G} {mode} F={F} {fmt}")
        untouched = np.setdiff1d(np.arange(cfg.V), t)
        np.testing.assert_array_equal(got[untouched], E0n[untouched])
    check_replicas(tables, f"compressed G={G} {mode}")
    close(ctxs)


def test_emulated_compressed_codec_on_each_transfer(lm):
    """R15's discriminating case on the device path: rank 0 sends 2049, rank 1
    sends 1, F = 1: the codec on each transfer gives 2048 (2049 -> 2048 at
    the sender, 2049 -> 2048 at the owner); one codec on the exact sum would
    give 2050."""
    cfg = synth.Config("emu", V=16, K=1, D=8, G=2)
    ctxs = make(lm, cfg, 2, F=1.0)
    tables = [torch.zeros(16, 8, device=dev()) for _ in range(2)]
    ids = [torch.tensor([3], dtype=torch.int32, device=dev())] * 2
    grads = [torch.full((1, 8), 2049.0, device=dev()), torch.full((1, 8), 1.0, device=dev())]
    lm.emulate_step(ctxs, ids, grads, tables, 1.0)
    torch.cuda.synchronize()
    for t in tables:
        assert torch.all(t[3] == -2048.0), t[3]
        assert torch.count_nonzero(t) == 8
    close(ctxs)


FULL = [("1b", 4, "int"), ("1b", 4, "signed"), ("1b", 8, "int")]


@pytest.mark.parametrize("name,G,mode", FULL, ids=[f"{n}-G{g}-{m}" for n, g, m in FULL])
def test_emulated_full_size_whole_matrix(lm, name, G, mode):
    """BASELINE.json's 1b config at G = 4 and 8 (the launch configuration
    bench.py times at world G, emulated): every row of I^ of every replica
    against the oracle's steps 1-7, every other row untouched."""
    cfg = synth.CONFIGS[name].with_(G=G)
    ctxs, J, Dl, E0, tables, lr = run(lm, cfg, G, mode)
    Ihat, Mhat64, A = oracle_mhat(J, [d.numpy() for d in Dl], want_A=mode != "int")
    rows = torch.from_numpy(Ihat.astype(np.int64)).to(dev())
    E0r = synth.table_rows(cfg.V, cfg.D, mode, Ihat).numpy().astype(np.float64)
    got = tables[0][rows].cpu().numpy()
    if mode == "int":
        check_rows(got, E0r - lr * Mhat64, None, "int", f"{name} G={G} E rows")
    else:
        check_rows(got, E0r - lr * Mhat64, np.abs(E0r) + lr * A, "signed", f"{name} G={G} E rows")
    mask = torch.ones(cfg.V, dtype=torch.bool, device=dev())
    mask[rows] = False
    assert torch.equal(tables[0][mask], E0[mask])
    check_replicas(tables, f"{name} G={G}")
    close(ctxs)
    del tables, E0


SAMPLED = [("tieba", 2, "int", 0.0), ("tieba", 2, "signed", 0.0), ("amazon", 2, "signed", 0.0),
           ("1b", 4, "signed", 1.0)]


@pytest.mark.parametrize("name,G,mode,F", SAMPLED, ids=[f"{n}-G{g}-{m}-F{f:g}" for n, g, m, f in SAMPLED])
def test_emulated_full_size_sampled(lm, name, G, mode, F):
    """The largest configs (tieba, amazon) at G = 2 and the compressed 1b G = 4:
    the 8 hottest words (runs cut by many S4 ranges, rows held by every rank)
    and 400 uniform words, each against the oracle's per-word steps
    (oracle.type_gradient: the definition of a row of M^); replicas
    bit-identical and untouched rows unchanged on the device."""
    cfg = synth.CONFIGS[name].with_(G=G)
    ctxs, J, Dl, E0, tables, lr = run(lm, cfg, G, mode, F)
    Ihat, gcounts = oracle.unique_global(np.concatenate(J))
    for c in ctxs:
        sg = c.sparse_grad()
        assert sg.num_unique == Ihat.size
    rows_t = torch.from_numpy(Ihat.astype(np.int64)).to(dev())
    mask = torch.ones(cfg.V, dtype=torch.bool, device=dev())
    mask[rows_t] = False
    assert torch.equal(tables[0][mask], E0[mask])
    check_replicas(tables, f"{name} G={G}")
    order = np.argsort(-gcounts, kind="stable")
    rng = np.random.default_rng(7)
    words = np.unique(np.concatenate([Ihat[order[:8]], rng.choice(Ihat, 400, replace=False)]))
    gotE = tables[0][torch.from_numpy(words.astype(np.int64)).to(dev())].cpu().numpy()
    E0w = synth.table_rows(cfg.V, cfg.D, mode, words).numpy().astype(np.float64)
    Dn = [d.numpy() for d in Dl]
    for i, w in enumerate(words):
        Js, Ds = [], []
        for g in range(G):
            pos = np.nonzero(J[g] == w)[0]
            Js.append(J[g][pos])
            Ds.append(Dn[g][pos])
        ref, Aw, _ = oracle.type_gradient(Js, Ds, int(w))
        if F > 0:
            parts = []
            for Jg, Dg in zip(Js, Ds):
                m, _, _ = oracle.type_gradient([Jg], [Dg], int(w))
                parts.append(oracle.decompress(oracle.compress(m.astype(np.float32), F), F))
            s = oracle.sum_f32(parts)
            mh = oracle.decompress(oracle.compress(s, F), F).astype(np.float64)
            tol = lr * compressed_tol(Aw, F, G) + 2.0 ** -23 * np.abs(E0w[i])
            check_compressed_rows(gotE[i], (E0w[i] - lr * mh).astype(np.float32), tol,
                                  f"{name} G={G} compressed word {w}", min_exact=0.9)
        elif mode == "int":
            check_rows(gotE[i:i + 1], (E0w[i] - lr * ref)[None], None, "int", f"{name} word {w}")
        else:
            check_rows(gotE[i:i + 1], (E0w[i] - lr * ref)[None], (np.abs(E0w[i]) + lr * Aw)[None],
                       "signed", f"{name} G={G} word {w}")
    close(ctxs)
    del tables, E0


@pytest.mark.parametrize("policy", ["power", "same", "distinct"])
def test_emulated_seeded_output_exchange(lm, policy):
    """Sec. 3.2 (R16) on the device path at G = 4: every rank draws
    S candidates with its group's seed (lmscale_plan_seeds +
    lmscale_draw_samples) into the tail of [K targets || S samples], then the
    world-G step; against the oracle's plan, draws and steps 1-7 over every
    rank's list (INT mode, bit-exact; replicas bit-identical)."""
    G, S, step, mode = 4, 1024, 3, "int"
    cfg = synth.CONFIGS["tiny"].with_(G=G)
    lr = synth.default_lr(mode)
    seeds, ngroups = lm.plan_seeds(G, policy, 0.64, master_seed=181010045)
    oseeds, on = oracle.plan_seeds(G, policy, alpha=0.64, master_seed=181010045)
    assert (seeds, ngroups) == (oseeds, on)
    ctxs = [lm.Context(cfg.V, cfg.K + S, cfg.D, world=G, rank=r, flags=lm.FLAG_NO_COMM)
            for r in range(G)]
    ids = []
    for r in range(G):
        t = torch.empty(cfg.K + S, dtype=torch.int32, device=dev())
        t[:cfg.K] = ids_dev(synth.ids_for(cfg, r))
        ctxs[r].draw_samples(seeds[r], step, S, out=t[cfg.K:])
        ids.append(t)
    Dl = [synth.grad_values(cfg.K + S, cfg.D, mode, rank=g) for g in range(G)]
    E0 = synth.table_values(cfg.V, cfg.D, mode, device=dev())
    tables = [E0.clone() for _ in range(G)]
    lm.emulate_step(ctxs, ids, [d.to(dev()) for d in Dl], tables, lr)
    torch.cuda.synchronize()
    Jall = [np.concatenate([synth.ids_for(cfg, g), oracle.draw_samples(oseeds[g], step, S, cfg.V)])
            for g in range(G)]
    for r in range(G):
        np.testing.assert_array_equal(ids[r].cpu().numpy().view(np.uint32), Jall[r])
    Eo = E0.cpu().numpy().copy()
    ref = oracle.sync_unique(Jall, [d.numpy() for d in Dl], Eo, lr)
    np.testing.assert_array_equal(tables[0].cpu().numpy(), Eo)
    check_replicas(tables, f"seeded {policy}")
    assert ctxs[0].sparse_grad().num_unique == ref["Ug"]
    close(ctxs)


def _random_cases(n=24, seed=18101004):
    rng = np.random.default_rng(seed)
    cases = []
    for i in range(n):
        G = int(rng.integers(2, 9))
        V = int(rng.choice([1, 2, 31, 33, 1000, 40000]))
        K = int(rng.choice([1, 2, 7, 300, 2049, 5000]))
        D = int(rng.choice([1, 3, 4, 17, 64, 100, 512, 516]))
        s = float(rng.choice([0.5, 1.0, 1.5]))
        cases.append((i, G, V, K, D, s))
    return cases


@pytest.mark.parametrize("i,G,V,K,D,s", _random_cases(),
                         ids=[f"case{c[0]}-G{c[1]}-V{c[2]}-K{c[3]}-D{c[4]}-s{c[5]}" for c in _random_cases()])
def test_emulated_random_shapes(lm, i, G, V, K, D, s):
    """Seeded random shapes for the world-G step (vocab 1..40000 incl. one
    bitmap word and its edge, K from 1 token, D from 1 float, the vector and
    the scalar kernels, flat to steep Zipf): INT mode, every replica's whole
    table bit-exact against oracle.sync_unique, I^ and the global counts too."""
    cfg = synth.Config("rand", V=V, K=K, D=D, G=G, s=s)
    lr = synth.default_lr("int")
    J = [synth.zipf_ids(V, s, K, rank=g, step=i) for g in range(G)]
    Dl = [synth.grad_values(K, D, "int", rank=g, step=i) for g in range(G)]
    E0 = synth.table_values(V, D, "int", device=dev())
    tables = [E0.clone() for _ in range(G)]
    ctxs = make(lm, cfg, G)
    lm.emulate_step(ctxs, [ids_dev(j) for j in J], [d.to(dev()) for d in Dl], tables, lr)
    torch.cuda.synchronize()
    Eo = E0.cpu().numpy().copy()
    ref = oracle.sync_unique(J, [d.numpy() for d in Dl], Eo, lr)
    np.testing.assert_array_equal(tables[0].cpu().numpy(), Eo)
    check_replicas(tables, f"random case {i}")
    for c in ctxs:
        sg = c.sparse_grad()
        assert sg.num_unique == ref["Ug"]
        np.testing.assert_array_equal(sg.ids.cpu().numpy().view(np.uint32), ref["Ihat"])
        np.testing.assert_array_equal(sg.counts.cpu().numpy(), ref["gcounts"])
    close(ctxs)
