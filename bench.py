#!/usr/bin/env python
"""Benchmark of SPION's hot path on B200: one step = pattern generation from a
synthetic head-averaged score matrix (Alg. 3/4) + block-sparse attention
forward + backward over every (batch, head) of the LRA-shaped workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config image|listops|text|retrieval]
    torchrun --nproc-per-node N bench.py --gpus N ...          (one rank per GPU, NCCL)
    python bench.py --impl reference ...                       (the CPU oracle, bounded sample)

Prints ONE JSON line on rank 0 (contract in DESIGN.md §6).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2309_12578_b200 import accounting  # noqa: E402

METRIC = "sparse-attn fwd+bwd tokens/s at LRA shapes; % bf16 tensor peak on useful blocks"
UNIT = "tokens/s"

# BASELINE.json configs (d = 64, bf16); towers = 2 for Retrieval (two documents)
CONFIGS = {
    "image": dict(workload="lra_image", L=1024, block=32, heads=4, d=64, batch=64, towers=1),
    "listops": dict(workload="lra_listops", L=2048, block=64, heads=8, d=64, batch=32, towers=1),
    "text": dict(workload="lra_text", L=4096, block=64, heads=8, d=64, batch=16, towers=1),
    "retrieval": dict(workload="lra_retrieval", L=4096, block=64, heads=8, d=64, batch=16, towers=2),
}
FILTER = 31


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# DRAM bytes per launch of each call from one `ncu --set full` capture (tools/ncu_traffic.py)
TRAFFIC_FILE = "profiles/r1/ncu_traffic.json"


def ncu_traffic(config, call):
    try:
        with open(os.path.join(ROOT, TRAFFIC_FILE)) as f:
            v = json.load(f).get(config, {}).get(call)
        return float(v) if v is not None else None
    except (OSError, ValueError):
        return None


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML while the timed region runs."""
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML missing
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ distributed
def dist_setup(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        return dist, rank, world, local
    return None, 0, 1, 0


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ------------------------------------------------------------------ oracle leg
def oracle_sample(cfg, mask_fl, alpha, budget_s=20.0, seed=99):
    """Time the CPU oracle (as it stands) on a bounded sample of the step: the pattern once
    plus fwd+bwd of k (batch, head) slices run concurrently on all host cores; the step time
    is extrapolated linearly to every (batch, head).  Returns (tokens/s, cores, description)."""
    import concurrent.futures as cf

    import oracle

    L, B, d = cfg["L"], cfg["block"], cfg["d"]
    bh = cfg["batch"] * cfg["towers"] * cfg["heads"]
    tokens = cfg["batch"] * cfg["towers"] * L
    cores = os.cpu_count() or 1
    A = synth.lra_scores(L, B, seed=1).numpy()
    t0 = time.perf_counter()
    fl, _, _ = oracle.pattern(A, B, FILTER, alpha)
    t_pat = time.perf_counter() - t0
    scale = 1.0 / math.sqrt(d)

    def one(b):
        q, k, v, do = (x[0].double().numpy() for x in synth.qkvdo(1, L, d, seed=seed, dtype=torch.bfloat16,
                                                                  start_bh=b))
        t = time.perf_counter()
        oracle.attn_fwd(q, k, v, fl, B, scale, "paper")
        oracle.attn_bwd(q, k, v, do, fl, B, scale, "paper")
        return time.perf_counter() - t

    # calibrate with one slice, then size the sample to the budget
    t1 = one(0)
    k = int(max(1, min(bh - 1, budget_s / max(t1, 1e-6) * cores * 0.8)))
    k = max(cores, (k // cores) * cores) if k >= cores else k
    k = min(k, bh - 1) if bh > 1 else 0
    t0 = time.perf_counter()
    if k > 0:
        with cf.ThreadPoolExecutor(max_workers=cores) as ex:
            list(ex.map(one, range(1, 1 + k)))
    wall = time.perf_counter() - t0
    per_slice_parallel = (wall / k) if k > 0 else t1
    t_step = t_pat + per_slice_parallel * bh
    desc = (f"pattern once ({t_pat:.2f}s) + fwd+bwd of {k + 1} of {bh} (batch,head) slices "
            f"({k} concurrently on {cores} threads in {wall:.2f}s); extrapolated linearly to all {bh}")
    return tokens / t_step, cores, desc, t_step


def run_reference(args, cfg):
    dist, rank, world, _ = dist_setup(args.gpus)
    if rank != 0:
        return
    per_rank_cfg = dict(cfg)
    value, cores, desc, t_step = oracle_sample(per_rank_cfg, None, args.alpha, budget_s=args.cpu_budget)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "L": cfg["L"], "block": cfg["block"], "heads": cfg["heads"],
                   "d": cfg["d"], "batch": cfg["batch"], "towers": cfg["towers"], "alpha": args.alpha,
                   "filter": FILTER},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="spion", choices=["spion", "reference"])
    ap.add_argument("--config", default="image", choices=sorted(CONFIGS))
    ap.add_argument("--alpha", type=float, default=75.0,
                    help="flood-fill quantile (75 gives ~9-12%% block density on the synthetic LRA scores)")
    ap.add_argument("--mode", default="paper", choices=["paper", "masked"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--phase-detail", action="store_true", help="also print per-phase timings to stderr")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args, cfg)

    from paper_2309_12578_b200 import spion
    from paper_2309_12578_b200 import _native as N
    from paper_2309_12578_b200.dist import broadcast_pattern

    dist, rank, world, local = dist_setup(args.gpus)
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    hbm_peak, tc_peak, tc_sust, peak_src = load_peaks()

    L, B, H, d = cfg["L"], cfg["block"], cfg["heads"], cfg["d"]
    bh = cfg["batch"] * cfg["towers"] * H          # per rank (weak scaling over ranks)
    tokens_rank = cfg["batch"] * cfg["towers"] * L
    scale = 1.0 / math.sqrt(d)

    # inputs resident in HBM; two rotating sets so a step never finds its inputs in L2
    NSETS = 2
    sets = []
    for s in range(NSETS):
        A = synth.lra_scores(L, B, seed=1 + 1000 * s, device=dev)
        q, k, v, do = synth.qkvdo(bh, L, d, seed=7 + 100003 * s, dtype=torch.bfloat16, device=dev,
                                  start_bh=rank * bh)
        sets.append((A, q, k, v, do))
    outs = [dict(o=torch.empty_like(q), lse=torch.empty((bh, L), dtype=torch.float32, device=dev),
                 dq=torch.empty_like(q), dk=torch.empty_like(q), dv=torch.empty_like(q)) for _ in range(NSETS)]
    ws = spion.attn_workspace(bh, L, d, torch.bfloat16, dev)
    bps = [spion.empty_pattern(L, B, dev) for _ in range(NSETS)]
    # (pattern workspace is attached to each BlockPattern on first use)

    def step(i, ev=None):
        A, q, k, v, do = sets[i % NSETS]
        o = outs[i % NSETS]
        bp = bps[i % NSETS]
        if ev is not None:
            ev[0].record()
        if rank == 0 or world == 1:
            spion.pattern(A, B, filter=FILTER, alpha=args.alpha, out=bp)
        if world > 1:
            broadcast_pattern(bp.flat, src=0)  # the per-layer pattern: one NCCL collective
        if ev is not None:
            ev[1].record()
        spion.attn_fwd(q, k, v, bp, args.mode, scale, out=o["o"], lse=o["lse"])
        if ev is not None:
            ev[2].record()
        spion.attn_bwd(q, k, v, o["o"], do, o["lse"], bp, args.mode, scale, workspace=ws,
                       dq=o["dq"], dk=o["dk"], dv=o["dv"])
        if ev is not None:
            ev[3].record()

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    nnzb_sets = [bp_.nnzb for bp_ in bps]  # steps alternate between the sets' patterns
    nnzb = sum(nnzb_sets) / len(nnzb_sets)
    density = nnzb / (L // B) ** 2

    # ---- timed region: K steps, events on the launching stream at phase boundaries
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = spion.launch_count()
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        barrier(dist)
        torch.cuda.synchronize()
        start.record()
        for i in range(args.steps):
            step(i, evs[i])
        end.record()
        torch.cuda.synchronize()
        barrier(dist)
    launches = spion.launch_count() - launches0
    ms = start.elapsed_time(end) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ph = {"pattern": [], "fwd": [], "bwd": []}
    for e in evs:
        ph["pattern"].append(e[0].elapsed_time(e[1]))
        ph["fwd"].append(e[1].elapsed_time(e[2]))
        ph["bwd"].append(e[2].elapsed_time(e[3]))
    ph_ms = {k_: statistics.mean(v_) for k_, v_ in ph.items()}

    # ---- roofline of the dominant call (algorithmic bytes / measured duration)
    n = L // B
    alg = {
        "pattern": accounting.pattern_bytes(L, n),
        "fwd": (8 * d + 4) * L * bh,         # read Q,K,V; write O (bf16) + lse (fp32)
        "bwd": (16 * d + 4) * L * bh,        # read Q,K,V,O,dO + lse; write dQ,dK,dV
    }
    flops = {"pattern": 0, "fwd": accounting.useful_flops(B, d, nnzb, bh, True, False),
             "bwd": accounting.useful_flops(B, d, nnzb, bh, False, True)}
    dom = max(ph_ms, key=ph_ms.get)
    t_dom = ph_ms[dom] * 1e-3
    gbs = alg[dom] / t_dom / 1e9
    traffic = ncu_traffic(args.config, dom)
    roofline = {"kernel": f"spion_attn_{dom}" if dom != "pattern" else "spion_pattern", "bound": "hbm",
                "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak, "traffic": traffic,
                "traffic_source": TRAFFIC_FILE if traffic is not None else None,
                "peak_source": peak_src, "alg_bytes_per_launch": alg[dom], "ms_per_launch": ph_ms[dom],
                "useful_tflops": flops[dom] / t_dom / 1e12 if flops[dom] else 0.0}
    step_flops = accounting.useful_flops(B, d, nnzb, bh)
    value = tokens_rank * world / (ms * 1e-3)

    # ---- end to end through the C ABI from pinned host buffers (H2D + D2H inside)
    e2e = None
    if args.e2e_steps > 0:
        lib = N.lib()
        A, q, k, v, do = sets[0]
        hA = A.cpu().pin_memory()
        hq, hk, hv, hdo = (x.cpu().pin_memory() for x in (q, k, v, do))
        ho, hdq, hdk, hdv = (torch.empty_like(hq).pin_memory() for _ in range(4))
        hlse = torch.empty((bh, L), dtype=torch.float32).pin_memory()
        arena_bytes = lib.spion_step_arena_bytes(bh, L, d, B, N.BF16)
        arena = torch.empty(arena_bytes, dtype=torch.uint8, device=dev)
        import ctypes
        P = lambda t: ctypes.c_void_p(t.data_ptr())
        nnz = ctypes.c_int32(0)
        strm = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)

        def host_step():
            st = lib.spion_step_host(P(hA), P(hq), P(hk), P(hv), P(hdo), P(ho), P(hlse), P(hdq), P(hdk), P(hdv),
                                     bh, L, d, B, FILTER, args.alpha, N.THRESH["linear"], N.BF16,
                                     N.SOFTMAX[args.mode], scale, P(arena), arena_bytes, ctypes.byref(nnz), strm)
            N.check(st, "spion_step_host")

        host_step()
        barrier(dist)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.e2e_steps):
            host_step()
        e1.record()
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / args.e2e_steps
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        tb = bh * L * d * 2
        e2e = {"value": tokens_rank * world / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": L * L * 4 + 4 * tb,
               "d2h_bytes_per_step": 4 * tb + bh * L * 4, "ms_per_step": ems}
        del arena

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v_, cores, desc, _ = oracle_sample(cfg, None, args.alpha, budget_s=args.cpu_budget)
        cpu = {"value": v_, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {
                "workload": cfg["workload"], "L": L, "block": B, "heads": H, "d": d, "batch_per_rank": cfg["batch"],
                "towers": cfg["towers"], "bh_per_rank": bh, "filter": FILTER, "alpha": args.alpha,
                "softmax": args.mode, "nnzb": nnzb, "nnzb_sets": nnzb_sets, "block_density": round(density, 4),
                "step": "pattern(scores)+attn_fwd+attn_bwd", "parallelism": f"dp{world} over batch*head",
                "l2": f"{NSETS} rotating input sets (> L2 per step)",
            },
            "phases_ms": ph_ms,
            "useful_tflops": step_flops / (ms * 1e-3) / 1e12 * world,
            "pct_bf16_peak_useful": 100.0 * step_flops * world / (ms * 1e-3) / (tc_peak * 1e12 * world),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
