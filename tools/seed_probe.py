"""Time lmscale_draw_samples and the seeded step separately (one GPU)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1810_10045_b200 import lmscale

cfg = synth.CONFIGS["1b"]
S = 1024
dev = torch.device("cuda", 0)
ctx = lmscale.Context(cfg.V, cfg.K + S, cfg.D, flags=lmscale.FLAG_GRAPH)
ids = torch.empty(cfg.K + S, dtype=torch.int32, device=dev)
ids[:cfg.K] = torch.from_numpy(synth.ids_for(cfg, 0).view(np.int32)).to(dev)
grad = synth.grad_values(cfg.K + S, cfg.D, "signed", device=dev)
E = synth.table_values(cfg.V, cfg.D, "signed", device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for t in range(12):
    ev[0].record()
    ctx.draw_samples(5, t, S, out=ids[cfg.K:])
    ev[1].record()
    ctx.step(ids, grad, E, 0.1)
    ev[2].record()
    torch.cuda.synchronize()
    print(f"step {t}: draw {ev[0].elapsed_time(ev[1])*1e3:.1f} us  step {ev[1].elapsed_time(ev[2])*1e3:.1f} us", flush=True)
