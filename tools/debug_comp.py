"""Debug the compressed exchange at G ranks (torchrun): dump mismatches."""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, synth
from paper_1810_10045_b200 import lmscale
from paper_1810_10045_b200.distributed import make_context

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, G = dist.get_rank(), dist.get_world_size()
dev = torch.device("cuda", local)
F = float(os.environ.get("F", "1"))
mode = os.environ.get("MODE", "int")
cfg = synth.CONFIGS["tiny"].with_(G=G)
lr = synth.default_lr(mode)
J = [synth.ids_for(cfg, g) for g in range(G)]
Dh = [synth.grad_values(cfg.K, cfg.D, mode, rank=g) for g in range(G)]
E0 = synth.table_values(cfg.V, cfg.D, mode)
ctx = make_context(cfg.V, cfg.K, cfg.D)
ctx.set_compression(F)
E = E0.to(dev)
ug = ctx.step(torch.from_numpy(J[rank].view(np.int32)).to(dev), Dh[rank].to(dev), E, lr, want_num_unique=True)
torch.cuda.synchronize()
sg = ctx.sparse_grad()
Eo = E0.numpy().copy()
ref = oracle.sync_unique_compressed(J, [d.numpy() for d in Dh], Eo, lr, F)
print(rank, "ug", ug, ref["Ug"], "stats", ctx.stats()["fused_s5_s6"], flush=True)
ucap = min(G * cfg.K, cfg.V)
base = sg.rows.data_ptr()
n16 = ucap * cfg.D
raw = torch.empty(0)
import ctypes
# local M16 and Mhat16 via a cudaMemcpy of the raw bytes
buf = torch.empty(2 * n16 + 4096, dtype=torch.uint8, device=dev)
cudart = ctypes.CDLL("libcudart.so.12") if False else None
m_all = torch.cuda.ByteStorage if False else None
# use torch.from_blob-like: wrap with lmscale's _view helper
from paper_1810_10045_b200.lmscale import _view
m16 = _view(base, (ucap, cfg.D), torch.int16, dev)
off = ((2 * ucap * cfg.D + 255) // 256) * 256
mh16 = _view(base + off, (ucap, cfg.D), torch.int16, dev)
Ug = ref["Ug"]
got_m = m16[:Ug].cpu().numpy().view(np.uint16)
l2g = ref["ranks"][rank]["l2g"]
exp_m = ref["Q"][rank]
bad = np.argwhere(got_m[l2g] != exp_m[l2g])
print(rank, "M16 present rows mismatches", len(bad), bad[:5].tolist(), flush=True)
got_h = mh16[:Ug].cpu().numpy().view(np.uint16)
bad = np.argwhere(got_h != ref["Qhat"])
print(rank, "Mhat16 mismatches", len(bad), bad[:5].tolist(), flush=True)
if len(bad):
    r, c = bad[0]
    print(rank, "r", r, "got", got_h[r, c], "exp", ref["Qhat"][r, c], "S", ref["S"][r, c],
          "Q", [q[r, c] for q in ref["Q"]], flush=True)
got = E.cpu().numpy()
bad = np.argwhere(got != Eo)
print(rank, "E mismatches", len(bad), bad[:5].tolist(), flush=True)
dist.barrier()
dist.destroy_process_group()
