"""Emulated world-G step (lmscale_emulate_step) of one BASELINE config on ONE
GPU, for ncu captures of the fused S5+S6 kernel (k_p2p_bulk<EMU>) with every
'peer' access in local HBM: how fast the kernel body runs when the link is
not the limit.

    ncu -k regex:k_p2p_bulk python tools/emu_profile.py tieba 2
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1810_10045_b200 import lmscale  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tieba"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = synth.CONFIGS[name].with_(G=G)
dev = torch.device("cuda", 0)
ids = [torch.from_numpy(synth.ids_for(cfg, r).view(np.int32)).to(dev) for r in range(G)]
grads = [synth.grad_values(cfg.K, cfg.D, "signed", rank=r, device=dev) for r in range(G)]
tables = [synth.table_values(cfg.V, cfg.D, "signed", device=dev) for _ in range(G)]
ctxs = [lmscale.Context(cfg.V, cfg.K, cfg.D, world=G, rank=r, flags=lmscale.FLAG_NO_COMM)
        for r in range(G)]
F = float(os.environ.get("EMU_COMPRESS", "0"))   # Sec. 3.3 compressed exchange (binary16 M rows)
if F > 0:
    for c in ctxs:
        c.set_compression(F)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for s in range(steps):
    torch.cuda.synchronize()
    ev[0].record()
    lmscale.emulate_step(ctxs, ids, grads, tables, 0.1)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"{name} G={G} emulated step {s}: {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us "
          f"(all G ranks' kernels, one GPU)", flush=True)
for c in ctxs:
    c.close()
