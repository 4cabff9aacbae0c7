#!/usr/bin/env python
"""Benchmark of the uniqueness embedding-gradient exchange (arXiv 1810.10045 Sec. 3.1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config tieba] [--impl lmscale|reference]

``--gpus N`` (N > 1) without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks on 127.0.0.1 (one process per GPU);
under torchrun the environment's WORLD_SIZE is used.

One step = the whole hot path (S1 dedup, S2 id exchange, S3 global unique,
S4 scatter-add, S5 all-reduce, S6 row update) over one synthetic batch of K
tokens per GPU, inputs resident in HBM.  Weak scaling: every rank owns its own
K tokens.  Prints ONE JSON line on rank 0 (metric/unit from BASELINE.json):
value = whole-job tokens/s = N*K / (max over ranks of the device-timed step)
on the headline workload (the largest single-GPU BASELINE config, tieba);
``supporting`` holds the same measurement, in brief, for the other configs.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
NVLINK_NOMINAL = 900.0   # GB/s per direction per GPU (north_star's roofline)
NVLINK_MEASURED = 770.0  # GB/s peer copy per direction (B200_PROFILING.md)
# GB/s per direction of SM-initiated traffic mixing bulk-copy pulls and SM
# stores into the peer, both GPUs active (tools/p2p_probe.cu,
# profiles/r02/g2_nvlink_ceiling_probe.txt): the fused kernel's own pattern
NVLINK_SM_MIX = 699.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="tieba",
                    help="headline workload (default: tieba, the largest single-GPU config)")
    ap.add_argument("--supporting", default="1b",
                    help="comma-separated extra configs reported in brief under 'supporting' "
                         "('none' to skip)")
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
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy test)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def pct(xs, q):
    xs = sorted(xs)
    if not xs:
        return None
    i = min(len(xs) - 1, max(0, int(round(q / 100.0 * (len(xs) - 1)))))
    return xs[i]


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


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
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx),
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

def oracle_sample(cfg, G, mode, seconds, threads=1, inputs=None):
    """Time the CPU oracle (as it stands: plain C loops, fp64) on a bounded
    sample of the workload: whole G-rank steps over the config's shapes,
    repeated until ~`seconds` of CPU work (at least one step).  threads > 1:
    the all-cores variant (step 2 split over column blocks, bit-identical).
    Returns (tokens/s, sample description, steps, seconds)."""
    import oracle
    import synth
    if inputs is None:
        J = [synth.ids_for(cfg, g) for g in range(G)]
        Dl = [synth.grad_values(cfg.K, cfg.D, mode, rank=g).numpy() for g in range(G)]
    else:
        J, Dl = inputs
    E = np.zeros((cfg.V, cfg.D), np.float32)   # values do not change the oracle's work
    lr = synth.default_lr(mode)
    run = (lambda: oracle.sync_unique(J, Dl, E, lr)) if threads <= 1 else \
        (lambda: oracle.sync_unique_threads(J, Dl, E, lr, threads))
    t0 = time.perf_counter()
    n = 0
    while True:
        run()
        n += 1
        dt = time.perf_counter() - t0
        if dt >= seconds or n >= 1000:
            break
    tps = n * G * cfg.K / dt
    kind = "single-threaded C" if threads <= 1 else f"{threads} threads (step 2 split by columns)"
    desc = (f"{n} full oracle steps of workload {cfg.name} (G={G} simulated ranks x K={cfg.K} "
            f"tokens, D={cfg.D}) in {dt:.1f}s; {kind}, fp64 accumulation; CPU {cpu_model()}")
    return tps, desc, n, dt


ORACLE_MEM_BUDGET = 12 << 30   # host bytes one whole-width oracle step may hold


def oracle_step_bytes(cfg, G, Dc):
    """Host bytes of one oracle step (sync_unique) over Dc columns: the G
    inputs, the G fp64 M_g (U_g x Dc), M^, the G fp64 local sums and E."""
    import synth
    ug = min(synth.expected_unique(cfg.V, cfg.s, G * cfg.K) * 1.05, cfg.V)
    ui = min(synth.expected_unique(cfg.V, cfg.s, cfg.K) * 1.05, cfg.V)
    return int(Dc * (G * cfg.K * 4 + (G + 1) * ug * 8 + G * ui * 8 + cfg.V * 4))


def oracle_inputs_cols(cfg, G, mode, Dc):
    """Ids of the G ranks and Dc-column gradient blocks (the same seeded
    value distribution; the oracle's work does not depend on the values)."""
    import synth
    return ([synth.ids_for(cfg, g) for g in range(G)],
            [synth.grad_values(cfg.K, Dc, mode, rank=g).numpy() for g in range(G)])


def oracle_sample_cols(cfg, G, mode, seconds, Dc, inputs):
    """The oracle on a workload too large for host memory in whole-width
    steps: the same functions in sync_unique's order, with the
    id steps (1, 3, 4 and the remap) on the full streams and the value steps
    (2, 5, 6, 7 -- column-separable, the same work per column) on a Dc-column
    block; a step's time = t_ids + (D / Dc) t_values."""
    import oracle
    import synth
    J, Dl = inputs
    E = np.zeros((cfg.V, Dc), np.float32)
    lr = synth.default_lr(mode)
    t_ids = t_val = 0.0
    n = 0
    while True:
        t0 = time.perf_counter()
        ranks = [oracle.unique_local(J[g]) for g in range(G)]            # step 1
        I = oracle.allgather_ids(J)                                      # step 3
        Ihat, _ = oracle.unique_global(I)                                # step 4
        l2g = [oracle.remap(Jh, Ihat, inv)[0] for Jh, _, inv in ranks]
        t1 = time.perf_counter()
        Ms = []
        for g, (Jh, _, inv) in enumerate(ranks):
            dhat = oracle.reduce_local(Dl[g], inv, Jh.size)               # step 2
            Ms.append(oracle.scatter_expand(dhat, l2g[g], Ihat.size))    # step 5
        Mhat64 = oracle.allreduce_sum(Ms)                                # step 6
        oracle.update_rows(E, Ihat, Mhat64, lr)                          # step 7
        t2 = time.perf_counter()
        del Ms, Mhat64
        t_ids += t1 - t0
        t_val += t2 - t1
        n += 1
        if t_ids + t_val >= seconds or n >= 1000:
            break
    step = (t_ids + (cfg.D / Dc) * t_val) / n
    desc = (f"{n} oracle steps of workload {cfg.name} (G={G} simulated ranks x K={cfg.K} tokens, "
            f"D={cfg.D}): id steps on the full streams, value steps on a {Dc}-column block "
            f"scaled by D/{Dc} (a whole-width step needs "
            f"{oracle_step_bytes(cfg, G, cfg.D) / 2**30:.0f} GiB of host memory); "
            f"single-threaded C, fp64 accumulation; CPU {cpu_model()}")
    return G * cfg.K / step, desc, n, t_ids + t_val


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


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU oracle as it stands, on this arm's workload
    (G = world simulated ranks), timed on the host cores; rank 0 only."""
    if rank != 0:
        return
    per_step = max(1.0, min(20.0, 90.0 / max(1, args.steps + args.warmup)))
    import synth
    Dc = cfg.D
    while Dc > 8 and oracle_step_bytes(cfg, world, Dc) > ORACLE_MEM_BUDGET:
        Dc //= 2
    if Dc == cfg.D:
        inputs = ([synth.ids_for(cfg, g) for g in range(world)],
                  [synth.grad_values(cfg.K, cfg.D, args.mode, rank=g).numpy() for g in range(world)])
    else:
        inputs = oracle_inputs_cols(cfg, world, args.mode, Dc)
    times, descs = [], []
    for i in range(args.warmup + args.steps):
        if Dc != cfg.D:
            tps, desc, n, dt = oracle_sample_cols(cfg, world, args.mode, per_step, Dc, inputs)
        else:
            tps, desc, n, dt = oracle_sample(cfg, world, args.mode, per_step, inputs=inputs)
        if i >= args.warmup:
            times.append(tps)
            descs.append(desc)
    v = statistics.median(times)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * world * cfg.K / v, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(cfg, args, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": descs[-1], "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line, args)


def emit(line, args):
    s = json.dumps(line)
    print(s, flush=True)
    if args.out:
        with open(args.out, "a") as f:
            f.write(s + "\n")


def heaps(cfg, world_max=8):
    """Measured U of the synthetic streams at G = 1, 2, 4, 8 ranks (rank-g
    streams concatenated, the oracle's global unique) and the least-squares
    Heaps fit U = c (GK)^alpha, next to the paper's alpha = 0.64."""
    import oracle
    import synth
    pts = []
    J = []
    for G in (1, 2, 4, 8):
        while len(J) < G:
            J.append(synth.ids_for(cfg, len(J)))
        ug = int(oracle.unique_global(np.concatenate(J[:G]))[0].size)
        pts.append({"G": G, "GK": G * cfg.K, "U_g": ug,
                    "E_U_closed_form": synth.expected_unique(cfg.V, cfg.s, G * cfg.K)})
    alpha, c = synth.heaps_fit([p["GK"] for p in pts], [p["U_g"] for p in pts])
    return {"points": pts, "alpha": alpha, "c": c, "paper_alpha": 0.64,
            "source": "oracle.unique_global over the seeded per-rank streams (CPU)"}


# ---------------------------------------------------------------- GPU arm

def launch_self(args):
    """--gpus N without a torchrun environment: re-exec under torchrun."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    in_torchrun = "WORLD_SIZE" in os.environ
    if args.impl == "lmscale" and args.gpus > 1 and not in_torchrun:
        launch_self(args)
    import synth

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1")) if in_torchrun else args.gpus
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = synth.CONFIGS[args.config]
    if args.s is not None:
        cfg = cfg.with_(s=args.s)
    cfg = cfg.with_(G=world)

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    bench = Bench(args, rank, world, local, dev)
    line = bench.run(cfg, headline=True)
    sup = {}
    for name in [x for x in args.supporting.split(",") if x and x != "none"]:
        if name == cfg.name or name not in synth.CONFIGS:
            continue
        c2 = synth.CONFIGS[name].with_(G=world)
        if args.s is not None:
            c2 = c2.with_(s=args.s)
        sup[name] = bench.run(c2, headline=False)
    if rank == 0:
        line["supporting"] = sup
        emit(line, args)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


class Bench:
    def __init__(self, args, rank, world, local, dev):
        import torch
        self.args, self.rank, self.world, self.local, self.dev = args, rank, world, local, dev
        self.flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB
        self.sweep = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
        self.sink = torch.empty(1, dtype=torch.float32, device=dev)
        torch.sum(self.sweep, dim=(0,), out=self.sink.view(()))

    def flush_l2(self):
        import torch
        # write a buffer larger than L2, then read another one: L2 ends up
        # holding clean, unrelated lines (the flush's own write-backs are not
        # charged to the timed step)
        self.flush.zero_()
        torch.sum(self.sweep, dim=(0,), out=self.sink.view(()))

    def barrier(self):
        import torch
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(self, x):
        from paper_1810_10045_b200.distributed import max_over_ranks
        return max_over_ranks(x, self.dev)

    def timed(self, fn, steps, warmup, collect=None, on_start=None):
        import torch
        for _ in range(warmup):
            self.flush_l2()
            fn()
        self.barrier()
        stream = torch.cuda.current_stream()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        if self.world > 1:          # one untimed step absorbs the ranks' start skew
            self.flush_l2()
            fn()
        if on_start:
            on_start()
        # steps are enqueued back to back (no host round trip between them);
        # each is bracketed by its own events, the L2 flush between steps is
        # outside them, and the step's own exchange keeps ranks in lock-step
        for i in range(steps):
            self.flush_l2()
            ev[i][0].record(stream)
            fn()
            ev[i][1].record(stream)
            if collect:
                collect()
        self.barrier()
        return [a.elapsed_time(b) for a, b in ev]

    def run(self, cfg, headline):
        import torch
        import torch.distributed as dist
        import synth
        from paper_1810_10045_b200 import lmscale
        from paper_1810_10045_b200.distributed import make_context
        args, rank, world, dev = self.args, self.rank, self.world, self.dev

        # ---- inputs resident in HBM (seeded, per rank)
        J = synth.ids_for(cfg, rank)
        S_smp = args.samples if args.seeding else 0
        Kt = cfg.K + S_smp            # ids per GPU in the exchange
        ids = torch.empty(Kt, dtype=torch.int32, device=dev)
        ids[:cfg.K] = torch.from_numpy(J.view(np.int32)).to(dev)
        grad = synth.grad_values(Kt, cfg.D, args.mode, rank=rank, device=dev)
        lr = synth.default_lr(args.mode)
        flags = 0 if args.no_graph else lmscale.FLAG_GRAPH
        if world > 1:
            ctx = make_context(cfg.V, Kt, cfg.D, flags=flags)
        else:
            ctx = lmscale.Context(cfg.V, Kt, cfg.D, device=self.local, flags=flags)
        seed_plan, seeds = None, None
        if args.seeding:
            seeds, ngroups = lmscale.plan_seeds(world, args.seeding, 0.64,
                                                master_seed=synth.MASTER_SEED)
            seed_plan = {"policy": args.seeding, "groups": ngroups, "samples_per_gpu": S_smp}
            ctx.draw_samples(seeds[rank], 0, S_smp, out=ids[cfg.K:])
        # the table: with G > 1 the context allocates it in a symmetric window
        # so the fused S5+S6 kernel stores updated rows into every replica
        if world > 1:
            table = ctx.alloc_table()
            table.copy_(synth.table_values(cfg.V, cfg.D, args.mode, device=dev))
        else:
            table = synth.table_values(cfg.V, cfg.D, args.mode, device=dev)
        if args.compress > 0:
            ctx.set_compression(args.compress)
            ctx.set_codec(args.codec)
        torch.cuda.synchronize()

        step_no = [0]

        def step():
            if seed_plan:   # this step's candidates (same words within a seed group)
                step_no[0] += 1
                ctx.draw_samples(seeds[rank], step_no[0], S_smp, out=ids[cfg.K:])
            ctx.step(ids, grad, table, lr)

        # One nvidia-smi sampler, on rank 0, for every rank's GPU, through a
        # short untimed load window, the timed region and a short tail.
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        phys = [int(x) for x in vis.split(",")][:world] if vis else list(range(world))
        clk = Clocks(phys) if (headline and rank == 0 and
                               not os.environ.get("BENCH_NO_CLOCKS")) else None

        def load_window(seconds):
            # a fixed number of steps, the same on every rank (collectives
            # must match): sized from rank 0's timing of one batch of 8 steps
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

        # ---- timed region (value): no events inside the step
        ctx.set_timing(0)
        for _ in range(args.warmup):
            step()
        if clk:
            clk.start()
        load_window(0.3 if headline else 0.05)
        k_before = [0]

        def mark():
            k_before[0] = ctx.stats()["kernels_total_lo"]
        ms = self.timed(step, args.steps, 0, on_start=mark)
        launches = ctx.stats()["kernels_total_lo"] - k_before[0]   # the timed steps' kernels
        if headline:
            load_window(0.1)
        clocks = clk.stop() if clk else None
        st_last = ctx.stats()     # U_g / U_i and the byte accounting of the last step
        ug, ui = st_last["u_global"], st_last["u_local"]

        # ---- second pass: two events bracketing the S4 kernel (its live duration)
        ctx.set_timing(1)
        scat = []

        def collect_s4():
            v = ctx.stats()["us_scatter"]
            if v > 0:
                scat.append(v)
        ms_s4 = self.timed(step, args.steps, 1, collect_s4)
        # ---- third pass (G > 1): two events bracketing the fused S5+S6 kernel
        s56 = []
        if world > 1:
            ctx.set_timing(3)

            def collect_s56():
                v = ctx.stats()["us_allreduce"]
                if v > 0:
                    s56.append(v)
            self.timed(step, args.steps, 1, collect_s56)
        # ---- diagnostic pass (not timed for value): every phase bracketed
        phase = {k: [] for k in ("us_dedup", "us_gather", "us_merge", "us_scatter",
                                 "us_allreduce", "us_update", "us_total")}

        def collect():
            s = ctx.stats()
            for k in phase:
                phase[k].append(s[k])
        ctx.set_timing(2)
        self.timed(step, 3, 1, collect)
        ctx.set_timing(0)

        all_ms = [[round(1e3 * x, 1) for x in ms]]
        if world > 1:
            all_ms = [None] * world
            dist.all_gather_object(all_ms, [round(1e3 * x, 1) for x in ms])
        total_ms = self.max_over_ranks(sum(ms))
        ms_step = total_ms / args.steps
        # per-step percentiles (us) of the slowest rank at each step
        per_step = [max(r[i] for r in all_ms) for i in range(args.steps)]
        tokens = world * cfg.K
        value = tokens / (ms_step * 1e-3)

        ph = {k: self.max_over_ranks(statistics.median(v)) for k, v in phase.items() if v}
        ph["note"] = ("diagnostic pass with an event around every phase (~3 us each); "
                      "not the timed region")
        s4_us = self.max_over_ranks(statistics.median(scat) if scat else ph["us_scatter"])
        hbm_peak, peak_kind = peaks()
        D = cfg.D
        fused = st_last.get("fused_s5_s6", 0)
        if world == 1:
            kname = "k_seg (S4 segmented sum + folded S6 row update, one launch)"
            scatter_bytes = 4 * Kt * D + 8 * ug * D   # grad once; each E row of I^ read + written
        elif fused in (2, 3):
            esz = 2 if fused == 3 else 4
            kname = ("k_seg (S4 segmented sum, present rows only"
                     + (", binary16 output)" if esz == 2 else ")"))
            scatter_bytes = 4 * Kt * D + esz * ui * D
        else:
            kname = "k_seg (S4 segmented sum, all U_g rows incl. zero rows)"
            scatter_bytes = 4 * Kt * D + 4 * ug * D
        roof = {"kernel": kname, "bound": "hbm",
                "achieved": scatter_bytes / (s4_us * 1e-6) / 1e9, "peak": hbm_peak,
                "unit": "GB/s", "peak_kind": peak_kind,
                "bytes_per_launch": scatter_bytes, "us_per_launch": s4_us,
                "bytes_formula": ("4KD + 8U_gD (world 1: S6 folded)" if world == 1 else
                                  "4KD + e U_i D (present rows, e = 4 fp32 / 2 binary16)"
                                  if fused in (2, 3) else "4KD + 4U_gD")}
        roof["frac"] = roof["achieved"] / hbm_peak
        roof["measured_in"] = ("second timed pass of the same steps with two CUDA events "
                               "bracketing the kernel on its launch stream; that pass's step "
                               f"time: {self.max_over_ranks(sum(ms_s4)) / args.steps * 1e3:.1f} us")
        roof["traffic"] = ncu_traffic(cfg.name, world)

        upd = None
        if fused:
            # NVLink ingress per GPU (the busier direction), averaged over ranks:
            #   P2P kernels: owners load the remote present copies of their rows
            #   (sum_i U_i (G-1)/G^2 rows) and receive the other owners' rows
            #   ((G-1)/G U_g rows); 4 B/elem fp32, 2 B/elem compressed (R15);
            #   NVLS multicast: (1 + 1/G) U_g rows (reduce + broadcast).
            t = torch.tensor([float(ui)], dtype=torch.float64, device=dev)
            dist.all_reduce(t)
            ui_sum = float(t.item())
            p2p = fused == 3 or (fused == 2 and world <= 8)
            esz = 2 if fused == 3 else 4
            if p2p:
                rows_in = ui_sum * (world - 1) / world ** 2 + ug * (world - 1) / world
                kname2 = ("k_p2p_update_c (compressed S5+S6: binary16 reduce-scatter + "
                          "all-gather over NVLink P2P, local S6)" if fused == 3 else
                          "k_p2p_update (S5+S6 fused over NVLink P2P: present rows only)")
            else:
                rows_in = (1 + 1 / world) * ug
                kname2 = "k_nvls_update (S5+S6 fused, NVLS multimem)"
            nvl = rows_in * esz * D
            us56 = self.max_over_ranks(statistics.median(s56)) if s56 else ph["us_allreduce"]
            upd = {"kernel": kname2, "bound": "nvlink", "bytes_per_direction": nvl,
                   "us_per_launch": us56, "achieved": nvl / (us56 * 1e-6) / 1e9,
                   "peak": NVLINK_NOMINAL, "unit": "GB/s",
                   "peak_kind": "nominal NVLink 5 per direction per GPU (north_star)",
                   "measured_in": "third timed pass, two events bracketing the fused kernel"}
            upd["frac"] = upd["achieved"] / NVLINK_NOMINAL
            upd["frac_of_measured_peer_copy"] = upd["achieved"] / NVLINK_MEASURED
            upd["frac_of_sm_pattern_ceiling"] = upd["achieved"] / NVLINK_SM_MIX

        # ---- dense comparison path (S0), same inputs, separate table copy
        dense = None
        if not args.no_dense:
            try:
                table_d = table.clone()
                dms = self.timed(lambda: ctx.sync_dense(ids, grad, table_d, lr), args.steps,
                                 min(args.warmup, 3))
                dense_ms = self.max_over_ranks(sum(dms)) / args.steps
                del table_d
                ratio_model = (world * Kt * cfg.D) / (world * Kt + ug * cfg.D)
                dense = {"ms_per_step": dense_ms, "tokens_per_s": tokens / (dense_ms * 1e-3),
                         "speedup_unique_vs_dense": dense_ms / ms_step,
                         "paper_ratio_GKD_over_GK_plus_UD": ratio_model,
                         "gate_0.8x": 0.8 * ratio_model,
                         "path": ("all-gather of (ids, Delta) in chunks, each scattered with "
                                  "128-bit vector atomics as soon as it has arrived"
                                  if world > 1 else "one atomic scatter of the local rows")}
            except Exception as e:  # pragma: no cover
                dense = {"error": str(e)[:200]}

        brief = {"us_per_step": 1e3 * ms_step, "tokens_per_s": value,
                 "us_per_step_p10_p50_p90": [pct(per_step, 10), pct(per_step, 50),
                                             pct(per_step, 90)],
                 "U_local": ui, "U_global": ug, "S4_us": s4_us,
                 "S4_roofline_frac": roof["frac"], "S1_us_diagnostic": ph.get("us_dedup"),
                 "dense_us_per_step": dense["ms_per_step"] * 1e3 if dense and "ms_per_step" in
                 dense else None,
                 "speedup_unique_vs_dense": dense.get("speedup_unique_vs_dense") if dense
                 else None,
                 "gate_0.8x": dense.get("gate_0.8x") if dense else None,
                 "S5_S6": upd, "gpu_launches_per_step": launches / args.steps}
        if not headline:
            ctx.close()
            del table, grad, ids
            torch.cuda.empty_cache()
            return brief

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

            ems = self.timed(hstep, max(3, args.steps // 2), min(args.warmup, 3))
            e_ms = self.max_over_ranks(sum(ems)) / len(ems)
            e2e = {"value": tokens / (e_ms * 1e-3), "unit": UNIT, "ms_per_step": e_ms,
                   "h2d_bytes_per_step": 4 * cfg.K + 4 * cfg.K * cfg.D,
                   "d2h_bytes_per_step": 4 * ug_box[0],
                   "api": "lmscale_train_step_host (pinned host ids+grad -> S1..S6 -> I^ to host)"}
            del grad_h

        # ---- CPU oracle baselines (rank 0, N=1 only): single thread and all cores
        cpu = cpu_all = None
        if rank == 0 and world == 1 and not args.no_cpu and not args.seeding:
            inputs = ([J], [grad[:cfg.K].cpu().numpy()])
            tps, desc, n, dt = oracle_sample(cfg, 1, args.mode, args.cpu_seconds, inputs=inputs)
            cpu = {"value": tps, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc,
                   "cpu_model": cpu_model(), "host_cores_available": host_cores()}
            nt = host_cores()
            tps2, desc2, n2, dt2 = oracle_sample(cfg, 1, args.mode, args.cpu_seconds / 2,
                                                 threads=nt, inputs=inputs)
            cpu_all = {"value": tps2, "unit": UNIT, "cores": nt, "kind": "oracle (all cores)",
                       "sample": desc2, "cpu_model": cpu_model()}

        heaps_fit = heaps(cfg) if rank == 0 else None
        line = None
        if rank == 0:
            eu = synth.expected_unique(cfg.V, cfg.s, world * cfg.K)
            line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                    "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                    "us_per_step": 1e3 * ms_step,
                    "us_per_step_p10_p50_p90": brief["us_per_step_p10_p50_p90"],
                    "higher_is_better": True, "scaling": "weak",
                    "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded Zipf ids, "
                    "counter-hash fp32 gradients/table; no datasets)",
                    "config": config_dict(cfg, args, world),
                    "U_local": ui, "U_global": ug, "E_U_global_closed_form": eu,
                    "heaps": heaps_fit,
                    "phases_us_diagnostic": ph, "roofline": roof, "roofline_s5_s6": upd,
                    "bytes_per_step": {k: st_last[k] for k in
                                       ("bytes_ids_gathered", "bytes_grad_allreduce",
                                        "bytes_scatter", "bytes_update")},
                    "dense_baseline": dense, "e2e": e2e, "cpu_baseline": cpu,
                    "cpu_baseline_all_cores": cpu_all, "clocks": clocks,
                    "seed_plan": seed_plan,
                    "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
                    "step_us_per_rank": all_ms,
                    "library": lmscale.version()}
        ctx.close()
        del table, grad, ids
        torch.cuda.empty_cache()
        return line


def ncu_traffic(workload, world):
    """dram read+write bytes per launch of the S4 kernel from the committed ncu
    --set full summary (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"{workload}/G{world}", {}).get("k_seg")
    except Exception:
        return None


if __name__ == "__main__":
    main()
