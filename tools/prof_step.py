"""Short single-GPU driver for ncu: W warm-up + N steps of lmscale_step on a
BASELINE config (world 1), L2 flushed between steps like bench.py.

    python tools/prof_step.py --config 1b --steps 3 --warmup 2
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1810_10045_b200 import lmscale  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="1b")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--no-graph", action="store_true")
args = ap.parse_args()
cfg = synth.CONFIGS[args.config]
dev = torch.device("cuda", 0)
ids = torch.from_numpy(synth.ids_for(cfg, 0).view(np.int32)).to(dev)
grad = synth.grad_values(cfg.K, cfg.D, "signed", device=dev)
E = synth.table_values(cfg.V, cfg.D, "signed", device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
ctx = lmscale.Context(cfg.V, cfg.K, cfg.D, flags=0 if args.no_graph else lmscale.FLAG_GRAPH)
for i in range(args.warmup + args.steps):
    flush.zero_()
    ctx.step(ids, grad, E, 0.1)
torch.cuda.synchronize()
print("ok", cfg.name, ctx.stats()["kernels_last_call"], flush=True)
ctx.close()
