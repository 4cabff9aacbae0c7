"""Small single-GPU driver for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel of the world-1 step (S1 grouping, S4 with S6 folded
in, eager and CUDA-graph replay), the staged G = 2 emulation (S1, S3, S4 in
the global-slot layout with zero rows, S6), the dense baseline, the codec,
lookup and seeding draws -- on small seeded inputs, checked against the
oracle so a silent corruption also fails.

    compute-sanitizer --tool memcheck python tools/sanitize_step.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1810_10045_b200 import lmscale  # noqa: E402

dev = torch.device("cuda", 0)


def ids_dev(J):
    return torch.from_numpy(np.asarray(J, np.uint32).view(np.int32)).to(dev)


def world1(V, K, D, flags=0, steps=2):
    J = synth.zipf_ids(V, 1.0, K)
    g = synth.grad_values(K, D, "int", device=dev)
    E0 = synth.table_values(V, D, "int", device=dev)
    E = E0.clone()
    ctx = lmscale.Context(V, K, D, flags=flags)
    for _ in range(steps):
        ctx.step(ids_dev(J), g, E, 2.0 ** -4)
    torch.cuda.synchronize()
    Eo = E0.cpu().numpy()
    for _ in range(steps):
        oracle.sync_unique([J], [g.cpu().numpy()], Eo, 2.0 ** -4)
    assert np.array_equal(E.cpu().numpy(), Eo), (V, K, D, flags)
    ctx.close()


def staged(V, K, D, G=2):
    J = [synth.zipf_ids(V, 1.0, K, rank=r) for r in range(G)]
    Dl = [synth.grad_values(K, D, "int", rank=r) for r in range(G)]
    ctx = lmscale.Context(V, K, D, world=G, flags=lmscale.FLAG_NO_COMM)
    I = ids_dev(np.concatenate(J))
    ref = oracle.sync_unique(J, [d.numpy() for d in Dl], np.zeros((V, D), np.float32), 1.0)
    for r in range(G):
        ctx.unique(ids_dev(J[r]), want_outputs=True)
        ctx.global_unique(I)
        ctx.scatter_expand(Dl[r].to(dev))
        sg = ctx.sparse_grad()
        assert np.array_equal(sg.rows.cpu().numpy(), ref["M"][r].astype(np.float32))
    ctx.close()


def extras():
    ctx = lmscale.Context(5000, 3000, 32)
    J = synth.zipf_ids(5000, 1.0, 3000)
    E = synth.table_values(5000, 32, "int", device=dev)
    ctx.sync_dense(ids_dev(J), synth.grad_values(3000, 32, "int", device=dev), E, 0.5)
    out = ctx.lookup(ids_dev(J), E)
    q = ctx.compress(out.flatten(), 4.0)
    ctx.decompress(q, 4.0)
    ctx.draw_samples(7, 1, 1024)
    sg = ctx.sync(ids_dev(J), synth.grad_values(3000, 32, "signed", device=dev))
    ctx.apply_update(E, sg, 0.1)
    torch.cuda.synchronize()
    ctx.close()


if __name__ == "__main__":
    world1(10_000, 4096, 64)                       # tiny
    world1(20_000, 20_000, 128, lmscale.FLAG_GRAPH, steps=3)
    world1(300, 9000, 2052)                        # two column blocks, long runs
    world1(3000, 2500, 37)                         # unstaged scalar path
    staged(10_000, 4096, 64)
    staged(4000, 3001, 3)
    extras()
    print("sanitize driver ok", flush=True)
