"""Probe: step time of lmscale_step at G>1 under timing modes 0/1/2, in both orders."""
import os, sys, time
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1810_10045_b200 import lmscale
from paper_1810_10045_b200.distributed import make_context
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "1b"]
dev = torch.device("cuda", local)
ids = torch.from_numpy(synth.ids_for(cfg, rank).view(np.int32)).to(dev)
grad = synth.grad_values(cfg.K, cfg.D, "signed", rank=rank, device=dev)
ctx = make_context(cfg.V, cfg.K, cfg.D)
table = ctx.alloc_table() if os.environ.get("OWN_TABLE", "1") == "1" else synth.table_values(cfg.V, cfg.D, "signed", device=dev)
torch.cuda.synchronize()
def run(mode, n=10, sync="cuda"):
    ctx.set_timing(mode)
    ts = []
    for i in range(n):
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); ctx.step(ids, grad, table, 0.1); b.record()
        if sync == "cuda": torch.cuda.synchronize()
        else: ctx.stats()
        ts.append(a.elapsed_time(b) * 1e3) if sync == "cuda" else ts.append(None)
        if sync != "cuda":
            torch.cuda.synchronize(); ts[-1] = a.elapsed_time(b) * 1e3
    return np.median(ts)
for i in range(3): ctx.step(ids, grad, table, 0.1)
torch.cuda.synchronize()
res = []
for mode, sync in [(0, "cuda"), (1, "stats"), (0, "cuda"), (1, "cuda"), (2, "stats"), (0, "stats"), (0, "cuda")]:
    res.append((mode, sync, round(run(mode, sync=sync), 1)))
if rank == 0:
    print("PROBE", cfg.name, world, res, flush=True)
dist.barrier(); dist.destroy_process_group()
