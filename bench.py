#!/usr/bin/env python
"""Benchmark of the uniqueness embedding-gradient exchange (arXiv 1810.10045 Sec. 3.1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1b] [--impl lmscale|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

One step = the whole hot path (S1 dedup, S2 ID all-gather, S3 global unique,
S4 scatter-add, S5 all-reduce, S6 row update) over one synthetic batch of K
tokens per GPU, inputs resident in HBM.  Weak scaling: every rank owns its own
K tokens.  Prints ONE JSON line on rank 0 (metric/unit from BASELINE.json):
value = whole-job tokens/s = N*K / (max over ranks of the device-timed step).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "emb-grad sync µs/step & tokens/s at 1/2/4/8 B200; HBM GB/s vs peak"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="1b")
    ap.add_argument("--mode", default="signed", choices=["int", "pos", "signed"])
    ap.add_argument("--s", type=float, default=None, help="Zipf exponent override")
    ap.add_argument("--impl", default="lmscale", choices=["lmscale", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches (no CUDA graph)")
    ap.add_argument("--seeding", default=None,
                    choices=["distinct", "same", "log2", "loge", "log10", "power"],
                    help="Sec. 3.2 output-embedding exchange: each step draws --samples "
                         "candidates per GPU with its seed group's seed, then exchanges "
                         "[K targets || samples]")
    ap.add_argument("--samples", type=int, default=1024, help="sampled-softmax S per GPU (P:605)")
    ap.add_argument("--codec", default="fp16", choices=["fp16", "bf16"],
                    help="16-bit payload format of --compress")
    ap.add_argument("--compress", type=float, default=0.0,
                    help="Sec. 3.3 compressed exchange with scale F (0 = off, fp32 rows)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--out", default=None, help="also append the JSON line to this file")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# ------------------------------------------------------------- clocks sampler

class Clocks:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_indices):
        self.idx = ",".join(str(i) for i in device_indices)
        self.proc = None
        self.lines = []

    def start(self):
        try:
            interval = os.environ.get("BENCH_CLOCK_MS", "200")
            nice = ["nice", "-n", "19"] if os.environ.get("BENCH_CLOCK_NICE") else []
            self.proc = subprocess.Popen(
                nice + ["nvidia-smi", "-i", str(self.idx),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", interval],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for l in self.lines:
            parts = [x.strip() for x in l.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                mask = int(parts[2], 16)
            except ValueError:
                continue
            for bit, name in self.REASONS.items():
                if mask & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------- CPU oracle legs

def oracle_sample(cfg, G, mode, seconds):
    """Time the CPU oracle (as it stands, single-threaded C) on a bounded sample
    of the workload: whole G-rank steps over the config's shapes, repeated until
    ~`seconds` of CPU work.  Returns (tokens/s, sample description, steps)."""
    import oracle
    import synth
    J = [synth.ids_for(cfg, g) for g in range(G)]
    Dl = [synth.grad_values(cfg.K, cfg.D, mode, rank=g).numpy() for g in range(G)]
    E = np.zeros((cfg.V, cfg.D), np.float32)   # values do not change the oracle's work
    lr = synth.default_lr(mode)
    oracle.sync_unique(J, Dl, E, lr)           # build + warm
    t0 = time.perf_counter()
    n = 0
    while True:
        oracle.sync_unique(J, Dl, E, lr)
        n += 1
        dt = time.perf_counter() - t0
        if dt >= seconds or n >= 1000:
            break
    tps = n * G * cfg.K / dt
    desc = (f"{n} full oracle steps of workload {cfg.name} (G={G} simulated ranks x K={cfg.K} "
            f"tokens, D={cfg.D}) in {dt:.1f}s; single-threaded C, fp64 accumulation")
    return tps, desc, n, dt


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    import synth  # noqa: F401
    per_step = max(1.0, min(20.0, 90.0 / max(1, args.steps + args.warmup)))
    times = []
    for i in range(args.warmup + args.steps):
        tps, desc, n, dt = oracle_sample(cfg, world, args.mode, per_step)
        if i >= args.warmup:
            times.append(tps)
    v = statistics.median(times)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * world * cfg.K / v, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(cfg, args, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line, args)


def config_dict(cfg, args, world):
    return {"workload": cfg.name, "V": cfg.V, "K_per_gpu": cfg.K, "D": cfg.D, "zipf_s": cfg.s,
            "G": world, "value_mode": args.mode, "global_tokens": world * cfg.K,
            "parallelism": f"dp{world}",
            "l2": "flushed between timed steps (256 MiB write, then a 256 MiB read sweep), "
                  "outside the timed region",
            "cuda_graph": not getattr(args, "no_graph", True),
            "compression": (f"{getattr(args, 'codec', 'fp16')}:F={args.compress:g}"
                            if args.compress > 0 else "off"),
            "seeding": (f"{args.seeding} (alpha 0.64), S={args.samples} samples/GPU; ids per "
                        f"GPU = K targets + S samples" if getattr(args, "seeding", None)
                        else "off (input-embedding exchange)")}


def emit(line, args):
    s = json.dumps(line)
    print(s, flush=True)
    if args.out:
        with open(args.out, "a") as f:
            f.write(s + "\n")


# ---------------------------------------------------------------- GPU arm

def main():
    args = parse()
    import torch
    import torch.distributed as dist
    import synth

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = synth.CONFIGS[args.config]
    if args.s is not None:
        cfg = cfg.with_(s=args.s)
    cfg = cfg.with_(G=world)

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    from paper_1810_10045_b200 import lmscale
    from paper_1810_10045_b200.distributed import make_context, max_over_ranks

    # ---- inputs resident in HBM (seeded, per rank)
    J = synth.ids_for(cfg, rank)
    S_smp = args.samples if args.seeding else 0
    Kt = cfg.K + S_smp            # ids per GPU in the exchange
    ids = torch.empty(Kt, dtype=torch.int32, device=dev)
    ids[:cfg.K] = torch.from_numpy(J.view(np.int32)).to(dev)
    grad = synth.grad_values(Kt, cfg.D, args.mode, rank=rank, device=dev)
    lr = synth.default_lr(args.mode)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > L2
    sweep = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    sweep.zero_()
    sink = torch.empty(1, dtype=torch.float32, device=dev)
    torch.sum(sweep, dim=(0,), out=sink.view(()))   # load the reduction kernel before timing

    def flush_l2():
        # write a buffer larger than L2, then read another one: L2 ends up
        # holding clean, unrelated lines (the flush's own write-backs are not
        # charged to the timed step)
        flush.zero_()
        torch.sum(sweep, dim=(0,), out=sink.view(()))

    flags = 0 if args.no_graph else lmscale.FLAG_GRAPH
    if world > 1:
        ctx = make_context(cfg.V, Kt, cfg.D, flags=flags)
    else:
        ctx = lmscale.Context(cfg.V, Kt, cfg.D, device=local, flags=flags)
    seed_plan = None
    if args.seeding:
        seeds, ngroups = lmscale.plan_seeds(world, args.seeding, 0.64, master_seed=synth.MASTER_SEED)
        seed_plan = {"policy": args.seeding, "groups": ngroups, "samples_per_gpu": S_smp}
        ctx.draw_samples(seeds[rank], 0, S_smp, out=ids[cfg.K:])
    # the table: with G > 1 the context allocates it in a symmetric window so
    # the fused S5+S6 kernel multicasts updated rows into every replica
    if world > 1:
        table = ctx.alloc_table()
        table.copy_(synth.table_values(cfg.V, cfg.D, args.mode, device=dev))
    else:
        table = synth.table_values(cfg.V, cfg.D, args.mode, device=dev)
    if args.compress > 0:
        ctx.set_compression(args.compress)
        ctx.set_codec(args.codec)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps, warmup, collect=None):
        for _ in range(warmup):
            flush_l2()
            fn()
        barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        if world > 1:          # one untimed step absorbs the ranks' start skew
            flush_l2()
            fn()
        # steps are enqueued back to back (no host round trip between them);
        # each is bracketed by its own events, the L2 flush between steps is
        # outside them, and the step's own collectives keep ranks in lock-step
        for i in range(steps):
            flush_l2()
            ev[i][0].record(stream)
            fn()
            ev[i][1].record(stream)
            if collect:
                collect()
        barrier()
        ms = [a.elapsed_time(b) for a, b in ev]
        return ms

    # ---- the unique exchange (S1-S6)
    phase = {k: [] for k in ("us_dedup", "us_gather", "us_merge", "us_scatter", "us_allreduce",
                             "us_update", "us_total")}
    info = {}
    launches = [0]

    step_no = [0]

    def step():
        if seed_plan:   # this step's candidates (same words within a seed group)
            step_no[0] += 1
            ctx.draw_samples(seeds[rank], step_no[0], S_smp, out=ids[cfg.K:])
        ctx.step(ids, grad, table, lr)

    def collect():
        st = ctx.stats()
        for k in phase:
            phase[k].append(st[k])
        info["u_local"] = st["u_local"]

    # One nvidia-smi sampler, on rank 0, for every rank's GPU (one sampler per
    # rank was measured to perturb multi-GPU steps).  It runs through a
    # ~0.3 s untimed load window, the timed region and a short tail, so the
    # samples cover the timed region even when it lasts under a millisecond.
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    phys = [int(x) for x in vis.split(",")][:world] if vis else list(range(world))
    clk = Clocks(phys) if rank == 0 and not os.environ.get("BENCH_NO_CLOCKS") else None

    def load_window(seconds):
        # a fixed number of steps, the same on every rank (collectives must
        # match): sized from rank 0's timing of one batch of 8 steps
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(8):
            step()
        torch.cuda.synchronize()
        per = max(time.perf_counter() - t0, 1e-6) / 8
        n = torch.tensor([int(seconds / per) // 8 + 1], dtype=torch.int64, device=dev)
        if world > 1:
            dist.broadcast(n, 0)
        for _ in range(int(n.item())):
            for _ in range(8):
                step()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # Timed region (value): no events inside the step (each event node is a
    # GPU-side serialisation point worth several microseconds).
    ctx.set_timing(0)
    for _ in range(args.warmup):
        step()
    if clk:
        clk.start()
    load_window(0.3)
    k_before = ctx.stats()["kernels_total_lo"]
    ms = timed(step, args.steps, 0)
    launches[0] = ctx.stats()["kernels_total_lo"] - k_before
    load_window(0.1)
    clocks = clk.stop() if clk else None
    info["ug"] = ctx.sparse_grad().num_unique
    # Second timed pass, same steps, with the two events that bracket the S4
    # kernel: its live per-launch duration for the roofline.
    ctx.set_timing(1)
    scat = []

    def collect_s4():
        v = ctx.stats()["us_scatter"]
        if v > 0:
            scat.append(v)
    ms_s4 = timed(step, args.steps, 1, collect_s4)
    # Diagnostic pass (not timed for `value`): every phase bracketed by events.
    ctx.set_timing(2)
    timed(step, 3, 1, collect)
    ctx.set_timing(0)
    all_ms = [ms]
    if world > 1:
        all_ms = [None] * world
        dist.all_gather_object(all_ms, [round(1e3 * x, 1) for x in ms])
    total_ms = max_over_ranks(sum(ms), dev)
    ms_step = total_ms / args.steps
    tokens = world * cfg.K
    value = tokens / (ms_step * 1e-3)
    ug = info["ug"]
    sync_launches = launches[0]

    # per-phase device times (median over timed steps), max over ranks
    ph = {k: max_over_ranks(statistics.median(v), dev) for k, v in phase.items() if v}
    ph["note"] = "diagnostic pass with an event around every phase (~3 us each); not the timed region"
    s4_us = max_over_ranks(statistics.median(scat) if scat else ph["us_scatter"], dev)
    hbm_peak, peak_kind = peaks()
    st_last = ctx.stats()
    D = cfg.D
    inline_s6 = world == 1 and not os.environ.get("LMSCALE_NO_INLINE_S6")
    if inline_s6:
        # world 1: S6 folded into S4 -- grad read once, each E row of I^ read
        # and written once; M is never materialised
        kname = "k_scatter (S4 segmented scatter-add + folded S6 row update, one launch)"
        scatter_bytes = 4 * Kt * D + 8 * ug * D
    elif st_last.get("fused_s5_s6") in (2, 3):
        # fused P2P exchange: only the present rows of M_g are written
        # (fp32, or binary16 with compression)
        esz = 2 if st_last.get("fused_s5_s6") == 3 else 4
        kname = ("k_scatter (S4 segmented scatter-add, present rows only"
                 + (", binary16 output)" if esz == 2 else ")"))
        scatter_bytes = 4 * Kt * D + esz * int(info.get("u_local") or 0) * D
    else:
        kname = "k_scatter (S4 segmented scatter-add + cut-run fixup, one launch)"
        scatter_bytes = 4 * Kt * D + 4 * ug * D   # grad read + M written once
    scatter_us = s4_us
    roof = {"kernel": kname, "bound": "hbm",
            "achieved": scatter_bytes / (scatter_us * 1e-6) / 1e9, "peak": hbm_peak,
            "unit": "GB/s", "peak_kind": peak_kind,
            "bytes_per_launch": scatter_bytes, "us_per_launch": scatter_us}
    roof["frac"] = roof["achieved"] / hbm_peak
    roof["measured_in"] = ("second timed pass of the same steps with two CUDA events bracketing "
                           "the kernel on its launch stream; that pass's step time: "
                           f"{max_over_ranks(sum(ms_s4), dev) / args.steps * 1e3:.1f} us")
    roof["traffic"] = ncu_traffic(cfg.name, world)
    fused = st_last.get("fused_s5_s6", 0)
    if fused:
        # NVLink ingress per GPU (the busier direction), averaged over ranks:
        #   P2P kernels: owners load the remote present copies of their rows
        #   (sum_i U_i (G-1)/G^2 rows) and receive the other owners' rows
        #   ((G-1)/G U_g rows); 4 B/elem fp32, 2 B/elem compressed (R15);
        #   NVLS multicast: (1 + 1/G) U_g rows (reduce + broadcast).
        if dist.is_initialized():
            t = torch.tensor([float(info.get("u_local") or 0)], dtype=torch.float64, device=dev)
            dist.all_reduce(t)
            ui_sum = float(t.item())
        else:
            ui_sum = float(info.get("u_local") or 0)
        p2p = fused == 3 or (fused == 2 and world <= 8)
        esz = 2 if fused == 3 else 4
        if p2p:
            rows_in = ui_sum * (world - 1) / world ** 2 + ug * (world - 1) / world
            kname2 = ("k_p2p_update_c (compressed S5+S6: binary16 reduce-scatter + all-gather "
                      "over NVLink P2P, local S6)" if fused == 3 else
                      "k_p2p_update (S5+S6 fused over NVLink P2P: present rows only)")
        else:
            rows_in = (1 + 1 / world) * ug
            kname2 = "k_nvls_update (S5+S6 fused, NVLS multimem)"
        nvl = rows_in * esz * D
        upd = {"kernel": kname2, "bound": "nvlink",
               "bytes_per_direction": nvl, "us_per_launch": ph["us_allreduce"],
               "achieved": nvl / (ph["us_allreduce"] * 1e-6) / 1e9, "peak": 770.0,
               "peak_kind": "guide: measured peer copy per direction (900 nominal)"}
        upd["frac"] = upd["achieved"] / upd["peak"]
    elif inline_s6:
        upd = {"kernel": "folded into k_scatter (world 1)", "achieved": None,
               "bytes_per_launch": 0, "us_per_launch": 0.0, "frac": None}
    else:
        update_bytes = 12 * ug * D
        upd = {"kernel": "k_update (S6 row update)", "achieved": update_bytes /
               (ph["us_update"] * 1e-6) / 1e9, "bytes_per_launch": update_bytes,
               "us_per_launch": ph["us_update"]}
        upd["frac"] = upd["achieved"] / hbm_peak

    # ---- dense comparison path (S0), same inputs, separate table copy
    dense = None
    if not args.no_dense:
        try:
            table_d = table.clone()
            dms = timed(lambda: ctx.sync_dense(ids, grad, table_d, lr), args.steps,
                        min(args.warmup, 3))
            dense_ms = max_over_ranks(sum(dms), dev) / args.steps
            del table_d
            ratio_model = (world * Kt * cfg.D) / (world * Kt + ug * cfg.D)
            dense = {"ms_per_step": dense_ms, "tokens_per_s": tokens / (dense_ms * 1e-3),
                     "speedup_unique_vs_dense": dense_ms / ms_step,
                     "paper_ratio_GKD_over_GK_plus_UD": ratio_model,
                     "gate_0.8x": 0.8 * ratio_model}
        except Exception as e:  # pragma: no cover
            dense = {"error": str(e)[:200]}

    # ---- e2e: host (pinned) buffers through the C ABI, copies inside the timed region
    e2e = None
    if args.seeding:
        e2e = {"skipped": "seeding mode draws the candidates on the device"}
    elif not args.no_e2e:
        ids_h = torch.from_numpy(J.view(np.int32)).pin_memory()
        grad_h = grad.cpu().pin_memory()
        out_h = torch.empty(world * cfg.K, dtype=torch.int32).pin_memory()
        ug_box = [0]

        def hstep():
            ug_box[0] = ctx.train_step_host(ids_h, grad_h, table, lr, out_h)

        ems = timed(hstep, max(3, args.steps // 2), min(args.warmup, 3))
        e_ms = max_over_ranks(sum(ems), dev) / len(ems)
        e2e = {"value": tokens / (e_ms * 1e-3), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": 4 * cfg.K + 4 * cfg.K * cfg.D,
               "d2h_bytes_per_step": 4 * ug_box[0],
               "api": "lmscale_train_step_host (pinned host ids+grad -> S1..S6 -> I^ to host)"}

    # ---- CPU oracle baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.seeding:
        tps, desc, n, dt = oracle_sample(cfg, 1, args.mode, args.cpu_seconds)
        cpu = {"value": tps, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc,
               "host_cores_available": host_cores()}

    if rank == 0:
        eu = synth.expected_unique(cfg.V, cfg.s, world * cfg.K)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "us_per_step": 1e3 * ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded Zipf ids, "
                "counter-hash fp32 gradients/table; no datasets)",
                "config": config_dict(cfg, args, world),
                "U_local": info.get("u_local"), "U_global": ug, "E_U_global_closed_form": eu,
                "phases_us_diagnostic": ph, "roofline": roof, "roofline_s5_s6": upd,
                "dense_baseline": dense, "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks,
                "seed_plan": seed_plan,
                "gpu_launches": sync_launches, "gpu_launches_per_step": sync_launches / args.steps,
                "step_us_per_rank": all_ms if world > 1 else [[round(1e3 * x, 1) for x in ms]],
                "library": lmscale.version()}
        emit(line, args)
    ctx.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def ncu_traffic(workload, world):
    """dram read+write bytes per launch of k_scatter from the committed ncu
    --set full summary (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"{workload}/G{world}", {}).get("k_scatter")
    except Exception:
        return None


if __name__ == "__main__":
    main()
