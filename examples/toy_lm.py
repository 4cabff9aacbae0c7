"""Toy end-to-end use of the library: a pooled-embedding
language model trained with the uniqueness exchange, or with the dense
all-gather baseline, on seeded synthetic Zipf text.

Per step: the K tokens of a GPU form K/c contexts of c tokens;
`lmscale_lookup` gathers their input-embedding rows (the forward projection),
the mean of each context's rows predicts the next token through an output
matrix (dense torch SGD) and a full softmax, autograd gives the K x D gradient rows of
the gathered embeddings, and the library exchanges and applies them --
`lmscale_step` (S1-S6) or `lmscale_sync_dense_baseline` (S0).  The model
math is plain PyTorch (plumbing, not the product); the gather, exchange and
update run in the library's kernels.

    python examples/toy_lm.py [steps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1810_10045_b200 import lmscale  # noqa: E402


def run(steps=8, path="unique", V=10_000, D=64, K=4096, c=8, lr=20.0, lr_out=20.0, seed=7,
        device=0):
    dev = torch.device("cuda", device)
    g = torch.Generator().manual_seed(seed)
    E = (torch.randn(V, D, generator=g) * 0.1).to(dev)          # input embedding (trained)
    W = (torch.randn(V, D, generator=g) * 0.1).to(dev).requires_grad_(True)  # output embedding
    ctx = lmscale.Context(V, K, D)
    losses = []
    for t in range(steps):
        toks = synth.zipf_ids(V, 1.0, K + K // c, seed=seed, step=t)
        ids = torch.from_numpy(toks[:K].view(np.int32)).to(dev)
        nxt = torch.from_numpy(toks[K:].astype(np.int64)).to(dev)   # next token per context
        X = ctx.lookup(ids, E).requires_grad_(True)                # K x D (forward lookup)
        pooled = X.view(K // c, c, D).mean(dim=1)
        loss = torch.nn.functional.cross_entropy(pooled @ W.t(), nxt)
        loss.backward()
        grad = X.grad.contiguous()
        with torch.no_grad():   # output layer: plain dense SGD in torch (not the exchanged layer)
            W -= lr_out * W.grad
            W.grad = None
        if path == "unique":
            ctx.step(ids, grad, E, lr)
        else:
            ctx.sync_dense(ids, grad, E, lr)
        torch.cuda.synchronize()
        losses.append(float(loss.item()))
    ctx.close()
    return losses


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    u = run(n, "unique")
    d = run(n, "dense")
    for t, (a, b) in enumerate(zip(u, d)):
        print(f"step {t}: loss unique {a:.6f}  dense {b:.6f}  rel diff {abs(a - b) / b:.2e}")
