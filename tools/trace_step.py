"""Run a few exchange steps of one config with the in-kernel phase trace on.

    LMSCALE_PHASE_TRACE=1 python tools/trace_step.py 1b [steps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1810_10045_b200 import lmscale  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "1b"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = synth.CONFIGS[name]
if os.environ.get("TRACE_S"):   # Zipf exponent override
    cfg = cfg.with_(s=float(os.environ["TRACE_S"]))
dev = torch.device("cuda", 0)
ids = torch.from_numpy(synth.ids_for(cfg, 0).view(np.int32)).to(dev)
grad = synth.grad_values(cfg.K, cfg.D, "signed", device=dev)
table = synth.table_values(cfg.V, cfg.D, "signed", device=dev)
world = int(os.environ.get("WORLD_SIZE", "1"))
if world > 1:
    import torch.distributed as dist
    from paper_1810_10045_b200.distributed import make_context
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    dev = torch.device("cuda", local)
    ids = torch.from_numpy(synth.ids_for(cfg, rank).view(np.int32)).to(dev)
    grad = synth.grad_values(cfg.K, cfg.D, "signed", rank=rank, device=dev)
    ctx = make_context(cfg.V, cfg.K, cfg.D,
                       flags=0 if os.environ.get("TRACE_NO_EVENTS") else lmscale.FLAG_TIMING)
    table = ctx.alloc_table()   # the symmetric-window table: the P2P fused path bench.py runs
    table.copy_(synth.table_values(cfg.V, cfg.D, "signed", device=dev))
else:
    flags = (0 if os.environ.get("TRACE_NO_EVENTS") else lmscale.FLAG_TIMING) | \
        (lmscale.FLAG_GRAPH if os.environ.get("TRACE_GRAPH") else 0)
    ctx = lmscale.Context(cfg.V, cfg.K, cfg.D, flags=flags)
for i in range(steps):
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()   # ranks enter the step together (eager launches skew them otherwise)
    ctx.step(ids, grad, table, 0.1)
    torch.cuda.synchronize()
    st = ctx.stats()
    print({k: round(v, 2) for k, v in st.items() if k.startswith("us_")}, file=sys.stderr)
