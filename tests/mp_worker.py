"""Multi-GPU parity worker (one process per GPU, launched by torchrun).

Each rank runs the REAL collective path (lmscale_sync_embedding_grad with its
own NCCL communicator: ID all-gather + U_g x D all-reduce) and then checks, on
its own, against the CPU oracle: every rank can regenerate every other rank's
seeded inputs (synth), so no expected value travels through the GPU path.
Also checks that all replicas of the table are bit-identical afterwards
 and the dense all-gather baseline.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/mp_worker.py
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1810_10045_b200 import lmscale  # noqa: E402
from paper_1810_10045_b200.distributed import make_context  # noqa: E402
from tests.tolerances import check_compressed_rows, check_rows, compressed_tol  # noqa: E402


def u32(t):
    return t.view(torch.int32).cpu().numpy().view(np.uint32)


def table_digest(E):
    """Bitwise digest of the table (int64 sum of the raw bits, per row block)."""
    bits = E.view(torch.int32).to(torch.int64)
    return torch.stack([bits.sum(), (bits * 1315423911).sum(), bits[::7].sum()])


def check_replicas(E, what):
    d = table_digest(E)
    allds = [torch.empty_like(d) for _ in range(dist.get_world_size())]
    dist.all_gather(allds, d)
    for x in allds:
        assert torch.equal(x, allds[0]), f"{what}: replicas differ"


def run_small(ctx_full, cfg, mode, rank, G, dev):
    lr = synth.default_lr(mode)
    J = [synth.ids_for(cfg, g) for g in range(G)]
    Dh = [synth.grad_values(cfg.K, cfg.D, mode, rank=g) for g in range(G)]
    E0 = synth.table_values(cfg.V, cfg.D, mode)
    ctx = make_context(cfg.V, cfg.K, cfg.D)
    E = E0.to(dev)
    sg = ctx.sync(torch.from_numpy(J[rank].view(np.int32)).to(dev), Dh[rank].to(dev))
    ids, rows = u32(sg.ids), sg.rows.cpu().numpy()
    ctx.apply_update(E, sg, lr)
    torch.cuda.synchronize()
    Eo = E0.numpy().copy()
    ref = oracle.sync_unique(J, [d.numpy() for d in Dh], Eo, lr)
    np.testing.assert_array_equal(ids, ref["Ihat"])
    A = oracle.abs_scale(J, [d.numpy() for d in Dh], ref["Ihat"])
    check_rows(rows, ref["Mhat64"], A, mode, f"G={G} {cfg.name} {mode} Mhat")
    if mode == "int":
        np.testing.assert_array_equal(E.cpu().numpy(), Eo)
    maps = ctx.local_maps()
    np.testing.assert_array_equal(maps[3].cpu().numpy(), ref["ranks"][rank]["l2g"])
    check_replicas(E, f"{cfg.name} {mode}")
    # dense baseline on the same inputs
    Ed = E0.to(dev)
    ctx.sync_dense(torch.from_numpy(J[rank].view(np.int32)).to(dev), Dh[rank].to(dev), Ed, lr)
    torch.cuda.synchronize()
    Edo = oracle.sync_dense(J, [d.numpy() for d in Dh], E0.numpy().copy(), lr)
    if mode == "int":
        np.testing.assert_array_equal(Ed.cpu().numpy(), Edo)
        check_replicas(Ed, f"dense {cfg.name} {mode}")
    else:
        # fp32 atomics land in a different order on every GPU, so the dense
        # baseline's replicas agree only to rounding (the unique path above is
        # bit-identical by construction: P:433-435)
        np.testing.assert_allclose(Ed.cpu().numpy(), Edo, rtol=0, atol=2e-5)
    ctx.close()


def run_fused_small(cfg, mode, rank, G, dev, own_table=False):
    """lmscale_step (S1-S6 in one call; S5+S6 as the fused NVLS kernel when the
    box has multicast) against the oracle; replicas must be bit-identical."""
    lr = synth.default_lr(mode)
    J = [synth.ids_for(cfg, g) for g in range(G)]
    Dh = [synth.grad_values(cfg.K, cfg.D, mode, rank=g) for g in range(G)]
    E0 = synth.table_values(cfg.V, cfg.D, mode)
    ctx = make_context(cfg.V, cfg.K, cfg.D)
    if own_table:   # the context's symmetric-window table (direct multicast update)
        E = ctx.alloc_table()
        E.copy_(E0.to(dev))
        torch.cuda.synchronize()
    else:
        E = E0.to(dev)
    ug = ctx.step(torch.from_numpy(J[rank].view(np.int32)).to(dev), Dh[rank].to(dev), E, lr,
                  want_num_unique=True)
    torch.cuda.synchronize()
    st = ctx.stats()
    if os.environ.get("LMSCALE_REQUIRE_NVLS") == "1":
        assert st["fused_s5_s6"] == (2 if own_table else 1), f"fused NVLS path: {st['fused_s5_s6']}"
    Eo = E0.numpy().copy()
    ref = oracle.sync_unique(J, [d.numpy() for d in Dh], Eo, lr)
    assert ug == ref["Ug"]
    got = E.cpu().numpy()
    if mode == "int":
        np.testing.assert_array_equal(got, Eo)
    else:
        A = oracle.abs_scale(J, [d.numpy() for d in Dh], ref["Ihat"])
        t = ref["Ihat"].astype(np.int64)
        E0n = E0.numpy()
        check_rows(got[t], E0n[t].astype(np.float64) - lr * ref["Mhat64"], np.abs(E0n[t]) + lr * A,
                   "signed", f"fused G={G} {cfg.name}")
        untouched = np.setdiff1d(np.arange(cfg.V), t)
        np.testing.assert_array_equal(got[untouched], E0n[untouched])
    check_replicas(E, f"fused {cfg.name} {mode}")
    # a second step on the updated table: the fused kernel leaves M reusable
    ctx.step(torch.from_numpy(J[rank].view(np.int32)).to(dev), Dh[rank].to(dev), E, lr)
    torch.cuda.synchronize()
    check_replicas(E, f"fused step 2 {cfg.name} {mode}")
    if rank == 0:
        print(f"fused={st['fused_s5_s6']} nvls={st['nvls_available']} G={G} {cfg.name} {mode} "
              f"own_table={own_table}", flush=True)
    ctx.close()


def run_consistency_check(cfg, rank, G, dev):
    """LMSCALE_FLAG_CHECK: U_g and the I^ checksum agree on every rank,
    so the checked step and sync return OK and match an unchecked context."""
    lr = synth.default_lr("int")
    ids = torch.from_numpy(synth.ids_for(cfg, rank).view(np.int32)).to(dev)
    g = synth.grad_values(cfg.K, cfg.D, "int", rank=rank).to(dev)
    outs = []
    for flags in (0, lmscale.FLAG_CHECK):
        ctx = make_context(cfg.V, cfg.K, cfg.D, flags=flags)
        E = synth.table_values(cfg.V, cfg.D, "int").to(dev)
        ug = ctx.step(ids, g, E, lr, want_num_unique=True)
        sg = ctx.sync(ids, g)
        assert sg.num_unique == ug
        torch.cuda.synchronize()
        outs.append(E.cpu())
        ctx.close()
    assert torch.equal(outs[0], outs[1])
    if rank == 0:
        print(f"consistency check ok G={G} U_g={ug}", flush=True)


def run_graph_equals_eager(cfg, rank, G, dev, F=0.0):
    """World > 1 with LMSCALE_FLAG_GRAPH (peer-bitmap S3 + fused S5+S6, no NCCL
    host calls): three captured-and-replayed steps give the same table bits as
    three eager steps, new buffer contents included.  INT mode: sums are exact
    in any order (S1's grouping order is the tickets' arrival order, R18)."""
    mode = "int"
    lr = synth.default_lr(mode)
    ids = torch.from_numpy(synth.ids_for(cfg, rank).view(np.int32)).to(dev)
    g = synth.grad_values(cfg.K, cfg.D, mode, rank=rank).to(dev)
    outs = []
    for flags in (0, lmscale.FLAG_GRAPH):
        ctx = make_context(cfg.V, cfg.K, cfg.D, flags=flags)
        if F > 0:
            ctx.set_compression(F)
        E = ctx.alloc_table()
        E.copy_(synth.table_values(cfg.V, cfg.D, mode).to(dev))
        ids_b, g_b = ids.clone(), g.clone()
        for t in range(3):
            if t == 2:
                ids_b.copy_(torch.from_numpy(synth.ids_for(cfg, rank, step=1).view(np.int32)).to(dev))
            ctx.step(ids_b, g_b, E, lr)
        torch.cuda.synchronize()
        outs.append(E.clone())
        check_replicas(E, f"graph={flags} {cfg.name}")
        ctx.close()
    assert torch.equal(outs[0], outs[1]), "graph replay differs from eager"
    if rank == 0:
        print(f"graph==eager G={G} {cfg.name} F={F}", flush=True)


def run_graph_compression_toggle(cfg, rank, G, dev):
    """with LMSCALE_FLAG_GRAPH, switching compression on after a
    step was captured must not replay the old (fp32) graph -- the step after
    the switch runs the compressed exchange and matches the oracle's R15
    exchange bit for bit (INT mode, F = 1)."""
    lr = synth.default_lr("int")
    J = [synth.ids_for(cfg, g) for g in range(G)]
    Dh = [synth.grad_values(cfg.K, cfg.D, "int", rank=g) for g in range(G)]
    E0 = synth.table_values(cfg.V, cfg.D, "int")
    ctx = make_context(cfg.V, cfg.K, cfg.D, flags=lmscale.FLAG_GRAPH)
    E = ctx.alloc_table()
    E.copy_(E0.to(dev))
    ids = torch.from_numpy(J[rank].view(np.int32)).to(dev)
    g = Dh[rank].to(dev)
    ctx.step(ids, g, E, lr)                 # captured without compression
    torch.cuda.synchronize()
    assert ctx.stats()["fused_s5_s6"] == 2
    E.copy_(E0.to(dev))
    torch.cuda.synchronize()
    ctx.set_compression(1.0)
    ctx.step(ids, g, E, lr)                 # same arguments: must re-capture
    torch.cuda.synchronize()
    assert ctx.stats()["fused_s5_s6"] == 3
    Eo = E0.numpy().copy()
    oracle.sync_unique_compressed(J, [d.numpy() for d in Dh], Eo, lr, 1.0)
    np.testing.assert_array_equal(E.cpu().numpy(), Eo)
    check_replicas(E, "graph compression toggle")
    if rank == 0:
        print(f"graph compression toggle G={G}", flush=True)
    ctx.close()


def run_compressed_small(cfg, mode, rank, G, dev, F, own_table=False, fmt="fp16"):
    """lmscale_step with compression (Sec. 3.3, R15) against
    oracle.sync_unique_compressed: INT mode bit-exact over the whole table,
    float modes within compressed_tol; replicas bit-identical.  lr is taken
    at fp32 precision on both sides so that equal M^ rows give equal E rows
    (the GPU's fma rounds once, like the oracle's fp64 update)."""
    lr = float(np.float32(synth.default_lr(mode)))
    J = [synth.ids_for(cfg, g) for g in range(G)]
    Dh = [synth.grad_values(cfg.K, cfg.D, mode, rank=g) for g in range(G)]
    E0 = synth.table_values(cfg.V, cfg.D, mode)
    ctx = make_context(cfg.V, cfg.K, cfg.D)
    ctx.set_compression(F)
    ctx.set_codec(fmt)
    if own_table:
        E = ctx.alloc_table()
        E.copy_(E0.to(dev))
        torch.cuda.synchronize()
    else:
        E = E0.to(dev)
    ug = ctx.step(torch.from_numpy(J[rank].view(np.int32)).to(dev), Dh[rank].to(dev), E, lr,
                  want_num_unique=True)
    torch.cuda.synchronize()
    assert ctx.stats()["fused_s5_s6"] == 3
    Eo = E0.numpy().copy()
    ref = oracle.sync_unique_compressed(J, [d.numpy() for d in Dh], Eo, lr, F, fmt)
    assert ug == ref["Ug"]
    got = E.cpu().numpy()
    if mode == "int":
        np.testing.assert_array_equal(got, Eo)
    else:
        t = ref["Ihat"].astype(np.int64)
        A = oracle.abs_scale(J, [d.numpy() for d in Dh], ref["Ihat"])
        E0n = E0.numpy()
        tol = lr * compressed_tol(A, F, G) * (8 if fmt == "bf16" else 1) + 2.0 ** -23 * np.abs(E0n[t])
        check_compressed_rows(got[t], Eo[t], tol, f"compressed G={G} {cfg.name} {mode} F={F}")
        untouched = np.setdiff1d(np.arange(cfg.V), t)
        np.testing.assert_array_equal(got[untouched], E0n[untouched])
    check_replicas(E, f"compressed {cfg.name} {mode}")
    ctx.step(torch.from_numpy(J[rank].view(np.int32)).to(dev), Dh[rank].to(dev), E, lr)
    torch.cuda.synchronize()
    check_replicas(E, f"compressed step 2 {cfg.name} {mode}")
    # compression off again: the plain fused exchange on the same context
    ctx.set_compression(0.0)
    ctx.step(torch.from_numpy(J[rank].view(np.int32)).to(dev), Dh[rank].to(dev), E, lr)
    torch.cuda.synchronize()
    assert ctx.stats()["fused_s5_s6"] in (1, 2)
    check_replicas(E, f"uncompressed after compressed {cfg.name} {mode}")
    if rank == 0:
        print(f"compressed G={G} {cfg.name} {mode} F={F} {fmt} own_table={own_table}", flush=True)
    ctx.close()


def run_seeded(cfg, rank, G, dev, policy, S=1024, mode="int"):
    """Sec. 3.2 output-embedding exchange: every rank draws S candidates with
    its group's seed (lmscale_plan_seeds + lmscale_draw_samples, R16) into the
    tail of [K targets || S samples] and runs lmscale_step; checked against
    the oracle's plan, draws and seven-step exchange over every rank's list."""
    lr = synth.default_lr(mode)
    seeds, ngroups = lmscale.plan_seeds(G, policy, 0.64, master_seed=181010045)
    oseeds, on = oracle.plan_seeds(G, policy, alpha=0.64, master_seed=181010045)
    assert (seeds, ngroups) == (oseeds, on)
    step = 3
    ctx = make_context(cfg.V, cfg.K + S, cfg.D)
    J = torch.empty(cfg.K + S, dtype=torch.int32, device=dev)
    J[:cfg.K] = torch.from_numpy(synth.ids_for(cfg, rank).view(np.int32)).to(dev)
    ctx.draw_samples(seeds[rank], step, S, out=J[cfg.K:])
    Dh = [synth.grad_values(cfg.K + S, cfg.D, mode, rank=g) for g in range(G)]
    E0 = synth.table_values(cfg.V, cfg.D, mode)
    E = E0.to(dev)
    ug = ctx.step(J, Dh[rank].to(dev), E, lr, want_num_unique=True)
    torch.cuda.synchronize()
    Jall = [np.concatenate([synth.ids_for(cfg, g), oracle.draw_samples(oseeds[g], step, S, cfg.V)])
            for g in range(G)]
    np.testing.assert_array_equal(u32(J), Jall[rank])
    Eo = E0.numpy().copy()
    ref = oracle.sync_unique(Jall, [d.numpy() for d in Dh], Eo, lr)
    assert ug == ref["Ug"]
    if mode == "int":
        np.testing.assert_array_equal(E.cpu().numpy(), Eo)
    check_replicas(E, f"seeded {policy}")
    if rank == 0:
        print(f"seeded G={G} {cfg.name} policy={policy} groups={ngroups} U_g={ug}", flush=True)
    ctx.close()
    return ug


def compressed_row(Js, Ds, w, F):
    """Oracle M^ row of one word under compression, from the definition: each
    rank's M_g row is the fp64 sum of its Delta rows of that word, rounded to
    fp32 (absent: zeros), then the R15 codec around the fp32 rank-order sum."""
    a = []
    for Jg, Dg in zip(Js, Ds):
        m, _, _ = oracle.type_gradient([Jg], [Dg], int(w))   # zeros when absent
        a.append(oracle.decompress(oracle.compress(m.astype(np.float32), F), F))
    s = oracle.sum_f32(a)
    return oracle.decompress(oracle.compress(s, F), F)


def run_full(cfg, rank, G, dev, n_rand=24, fused=False, F=0.0, own_table=False):
    """BASELINE full size on G real GPUs: integers in full, sampled float rows.
    own_table: the table in the context's symmetric window (lmscale_alloc_table),
    i.e. the launch configuration bench.py times (P2P fused S5+S6, local-slot M,
    S4 beside the peer-bitmap S3)."""
    mode = "signed"
    lr = synth.default_lr(mode)
    if F > 0:
        lr = float(np.float32(lr))   # fp32 lr on both sides (see run_compressed_small)
    J = [synth.ids_for(cfg, g) for g in range(G)]
    ctx = make_context(cfg.V, cfg.K, cfg.D)
    grad = synth.grad_values(cfg.K, cfg.D, mode, rank=rank, device=dev)
    if own_table:
        E = ctx.alloc_table()
        E.copy_(synth.table_values(cfg.V, cfg.D, mode, device=dev))
        torch.cuda.synchronize()
    else:
        E = synth.table_values(cfg.V, cfg.D, mode, device=dev)
    Ihat, gcounts = oracle.unique_global(np.concatenate(J))
    if F > 0:
        ctx.set_compression(F)
    if fused:
        ctx.step(torch.from_numpy(J[rank].view(np.int32)).to(dev), grad, E, lr)
        torch.cuda.synchronize()
        st = ctx.stats()
        if own_table:   # the P2P kernels (compressed or not), as bench.py runs them
            assert st["fused_s5_s6"] == (3 if F > 0 else 2), st["fused_s5_s6"]
        ids = u32(ctx.sparse_grad().ids)
        rows = None
    else:
        sg = ctx.sync(torch.from_numpy(J[rank].view(np.int32)).to(dev), grad)
        rows = sg.rows.clone()
        ids = u32(sg.ids)
        ctx.apply_update(E, sg, lr)
        torch.cuda.synchronize()
    np.testing.assert_array_equal(ids, Ihat)
    order = np.argsort(-gcounts, kind="stable")
    rng = np.random.default_rng(rank)
    words = np.unique(np.concatenate([Ihat[order[:6]], rng.choice(Ihat, n_rand, replace=False)]))
    slots = np.searchsorted(Ihat, words)
    got = rows[torch.from_numpy(slots).to(dev)].cpu().numpy() if rows is not None else None
    gotE = E[torch.from_numpy(words.astype(np.int64)).to(dev)].cpu().numpy()
    E0 = synth.table_rows(cfg.V, cfg.D, mode, words).numpy().astype(np.float64)
    for i, w in enumerate(words):
        Js, Ds = [], []
        for g in range(G):
            pos = np.nonzero(J[g] == w)[0]
            Js.append(J[g][pos])
            Ds.append(synth.grad_rows(cfg.D, mode, pos, rank=g).numpy().reshape(len(pos), cfg.D))
        ref, A, n = oracle.type_gradient(Js, Ds, w)
        if F > 0:
            mh = compressed_row(Js, Ds, w, F).astype(np.float64)
            tol = lr * compressed_tol(A, F, G) + 2.0 ** -23 * np.abs(E0[i])
            expE = (E0[i] - lr * mh).astype(np.float32)       # one rounding (R5)
            check_compressed_rows(gotE[i], expE, tol, f"{cfg.name} G={G} comp word {w}",
                                  min_exact=0.9)
            continue
        if got is not None:
            check_rows(got[i:i + 1], ref[None], A[None], mode, f"{cfg.name} G={G} word {w}")
        check_rows(gotE[i:i + 1], (E0[i] - lr * ref)[None], (np.abs(E0[i]) + lr * A)[None],
                   "signed", f"{cfg.name} G={G} E row {w}")
    check_replicas(E, f"full {cfg.name}")
    if rank == 0:
        print(f"full {cfg.name} G={G} fused={fused} F={F} own_table={own_table} "
              f"words={len(words)}", flush=True)
    ctx.close()


def run_compressed_discriminating(rank, G, dev):
    """R15 on real GPUs: one word, rank 0 contributes 2049, rank 1 contributes
    1, the others 0 (F = 1): the codec on each transfer gives 2049 -> 2048
    (sender), 2049 -> 2048 (owner's sum), so every replica holds -2048; a codec
    applied once to the exact sum would give -2050."""
    D = 8
    ctx = make_context(16, 4, D)
    ctx.set_compression(1.0)
    E = ctx.alloc_table()
    E.zero_()
    val = {0: 2049.0, 1: 1.0}.get(rank, 0.0)
    g = torch.full((1, D), val, dtype=torch.float32, device=dev)
    ids = torch.tensor([3], dtype=torch.int32, device=dev)
    ctx.step(ids, g, E, 1.0)
    torch.cuda.synchronize()
    assert torch.all(E[3] == -2048.0), E[3]
    assert torch.count_nonzero(E) == D
    check_replicas(E, "compressed 2049+1")
    if rank == 0:
        print(f"compressed 2049+1 -> 2048 G={G}", flush=True)
    ctx.close()


def run_long(cfg, rank, G, dev, steps=200, comp=False):
    """Many CUDA-graph replays of the benched path (table window, P2P fused
    S5+S6, S4 beside the peer-bitmap S3 -- or the compressed exchange) with a
    new batch every step (ids and gradients copied into the captured
    buffers): the flag handshake epochs, the LSA barriers and the presence
    bitmaps are exercised `steps` times; INT mode, the final table bit-exact
    against the oracle applying the same `steps` exchanges in order."""
    mode = "int"
    lr = synth.default_lr(mode)
    ctx = make_context(cfg.V, cfg.K, cfg.D, flags=lmscale.FLAG_GRAPH)
    if comp:
        ctx.set_compression(1.0)
    E = ctx.alloc_table()
    E0 = synth.table_values(cfg.V, cfg.D, mode)
    E.copy_(E0.to(dev))
    ids = torch.empty(cfg.K, dtype=torch.int32, device=dev)
    grad = torch.empty(cfg.K, cfg.D, dtype=torch.float32, device=dev)
    Eo = E0.numpy().copy()
    for s in range(steps):
        J = [synth.ids_for(cfg, g, step=s) for g in range(G)]
        Dl = [synth.grad_values(cfg.K, cfg.D, mode, rank=g, step=s) for g in range(G)]
        ids.copy_(torch.from_numpy(J[rank].view(np.int32)))
        grad.copy_(Dl[rank])
        ctx.step(ids, grad, E, lr)
        if comp:
            oracle.sync_unique_compressed(J, [d.numpy() for d in Dl], Eo, lr, 1.0)
        else:
            oracle.sync_unique(J, [d.numpy() for d in Dl], Eo, lr)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(E.cpu().numpy(), Eo)
    check_replicas(E, f"long {cfg.name} comp={comp}")
    if rank == 0:
        print(f"long G={G} {cfg.name} {steps} graph-replayed steps comp={comp}: bit-exact", flush=True)
    ctx.close()


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, G = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", local)
    which = sys.argv[1:] or ["small", "1b", "char"]
    if "small" in which:
        for mode in ("int", "signed"):
            run_small(None, synth.CONFIGS["tiny"].with_(G=G), mode, rank, G, dev)
        run_small(None, synth.Config("odd", V=3000, K=2500, D=37, G=G), "int", rank, G, dev)
        for mode in ("int", "signed"):
            run_fused_small(synth.CONFIGS["tiny"].with_(G=G), mode, rank, G, dev)
        run_fused_small(synth.Config("odd", V=3000, K=2500, D=37, G=G), "int", rank, G, dev)
        for mode in ("int", "signed"):
            run_fused_small(synth.CONFIGS["tiny"].with_(G=G), mode, rank, G, dev, own_table=True)
    if "small" in which:
        run_consistency_check(synth.CONFIGS["tiny"].with_(G=G), rank, G, dev)
    if "small" in which or "graph" in which:
        run_graph_equals_eager(synth.CONFIGS["tiny"].with_(G=G), rank, G, dev)
        run_graph_equals_eager(synth.CONFIGS["tiny"].with_(G=G), rank, G, dev, F=1.0)
        run_graph_compression_toggle(synth.CONFIGS["tiny"].with_(G=G), rank, G, dev)
    if "seed" in which:
        ugs = {p: run_seeded(synth.CONFIGS["tiny"].with_(G=G), rank, G, dev, p, S=512)
               for p in ("distinct", "power", "same")}
        assert ugs["same"] <= ugs["power"] <= ugs["distinct"]
    if "comp" in which:
        for F in (1.0, 1024.0):
            run_compressed_small(synth.CONFIGS["tiny"].with_(G=G), "int", rank, G, dev, F)
        run_compressed_small(synth.CONFIGS["tiny"].with_(G=G), "signed", rank, G, dev, 1.0)
        run_compressed_small(synth.CONFIGS["tiny"].with_(G=G), "pos", rank, G, dev, 32.0,
                             own_table=True)
        run_compressed_small(synth.Config("odd", V=3000, K=2500, D=37, G=G), "int", rank, G, dev,
                             1.0)
        run_full(synth.CONFIGS["1b"], rank, G, dev, fused=True, F=1.0)
        run_compressed_small(synth.CONFIGS["tiny"].with_(G=G), "int", rank, G, dev, 1.0, fmt="bf16")
        run_compressed_small(synth.CONFIGS["tiny"].with_(G=G), "signed", rank, G, dev, 1.0,
                             own_table=True, fmt="bf16")
    if "long" in which:
        cfg = synth.Config("long", V=50000, K=8192, D=128, G=G)
        run_long(cfg, rank, G, dev, steps=200)
        run_long(cfg, rank, G, dev, steps=100, comp=True)
    if "p2p" in which:
        # the launch configuration bench.py times (table window, P2P fused
        # S5+S6), fp32 and compressed, at 1b and tieba full size
        run_compressed_discriminating(rank, G, dev)
        for name in ("1b", "tieba"):
            run_full(synth.CONFIGS[name], rank, G, dev, n_rand=400, fused=True, own_table=True)
            run_full(synth.CONFIGS[name], rank, G, dev, n_rand=200, fused=True, own_table=True,
                     F=1.0)
    for name in ("1b", "char", "amazon", "tieba"):
        if name in which:
            run_full(synth.CONFIGS[name], rank, G, dev)
            run_full(synth.CONFIGS[name], rank, G, dev, fused=True)
    dist.barrier()
    if rank == 0:
        print(f"MP_OK G={G} {which}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
