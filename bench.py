#!/usr/bin/env python
"""Benchmark of SPION's hot path on B200: one step = pattern generation from a
synthetic head-averaged score matrix (Alg. 3/4) + block-sparse attention
forward + backward over every (batch, head) of the LRA-shaped workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config text|image|listops|retrieval]
    python bench.py --gpus 8 ...          (re-launches itself under torch.distributed.run, one rank per GPU)
    torchrun --nproc-per-node N bench.py --gpus N ...
    python bench.py --impl reference ...  (the CPU oracle, bounded sample per step)

Default workload: LRA Text (BASELINE configs[3], the largest single-GPU config).
Multi-GPU: strong scaling by default — the config's global (batch x head) slices are
split into N contiguous shards; `--scaling weak` gives every rank the
whole config.  Prints ONE JSON line on rank 0 (contract in DESIGN.md section 7).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2309_12578_b200 import accounting  # noqa: E402
from paper_2309_12578_b200.dist import shard  # noqa: E402

METRIC = "sparse-attn fwd+bwd tokens/s at LRA shapes; % bf16 tensor peak on useful blocks"
UNIT = "tokens/s"

# BASELINE.json configs (d = 64, bf16); towers = 2 for Retrieval (two documents).  alpha: the
# flood-fill quantile that puts the block density of the synthetic LRA scores near the north
# star's ~10 % (~90 % block sparsity): measured with the oracle on synth.lra_scores seeds 1 / 1001
# (DESIGN.md section 5): Image 11.8 / 10.7 %, ListOps 12.6 / 9.9 %, Text 10.1 / 10.0 %.
CONFIGS = {
    "image": dict(workload="lra_image", L=1024, block=32, heads=4, d=64, batch=64, towers=1, alpha=75.0),
    "listops": dict(workload="lra_listops", L=2048, block=64, heads=8, d=64, batch=32, towers=1, alpha=75.0),
    "text": dict(workload="lra_text", L=4096, block=64, heads=8, d=64, batch=16, towers=1, alpha=55.0),
    "retrieval": dict(workload="lra_retrieval", L=4096, block=64, heads=8, d=64, batch=16, towers=2, alpha=55.0),
}
FILTER = 31
SCORE_SEEDS = (1, 1001)  # the score matrices of the rotating input sets (set s uses SCORE_SEEDS[s % 2])


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# DRAM bytes per launch of each call from one `ncu --set full` capture (tools/ncu_traffic.py)
TRAFFIC_FILE = "profiles/r2/ncu_traffic.json"


def ncu_traffic(config, call):
    try:
        with open(os.path.join(ROOT, TRAFFIC_FILE)) as f:
            v = json.load(f).get(config, {}).get(call)
        return float(v) if v is not None else None
    except (OSError, ValueError):
        return None


def config_dict(cfg, args, world):
    """The workload description both arms print (identical for the same flags)."""
    bh = cfg["batch"] * cfg["towers"] * cfg["heads"]
    return {
        "workload": cfg["workload"], "L": cfg["L"], "block": cfg["block"], "heads": cfg["heads"], "d": cfg["d"],
        "batch": cfg["batch"], "towers": cfg["towers"], "bh": bh, "filter": FILTER, "alpha": args.alpha,
        "softmax": args.mode, "step": "pattern(scores)+attn_fwd+attn_bwd",
        "pipeline": "sequential" if args.no_pipeline else
        f"pattern of step i+{args.pipeline_depth} on a second stream during step i's attention",
        "parallelism": (f"emulated: rank 0's share of dp{args.emulate_world} over batch*head ({args.scaling} "
                        "scaling) on one GPU; the all-reduced pool arrives by a device copy"
                        if world == 1 and args.emulate_world > 1 else
                        f"dp{world} over batch*head ({args.scaling} scaling)"
                        + (f", pattern by {args.pattern_exchange}" if world > 1 else "")),
        "l2": "rotating input sets, >= 2x L2 of other data between two uses of a set",
    }


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
            self.sample()
            time.sleep(0.01)

    def sample(self):
        if not self.nv:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit and bit != 0x1:
                    self.reasons.add(name)
        except Exception:
            pass

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()
            self.sample()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ distributed
def maybe_self_launch(args):
    """`--gpus N` (N > 1) without a torch.distributed environment: re-launch this script under
    torch.distributed.run with one rank per GPU (rendezvous on 127.0.0.1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    r = subprocess.run(cmd)
    sys.exit(r.returncode)


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = os.environ.get("SPION_BENCH_BACKEND", "nccl")  # "gloo": host-logic check of the N-rank path
        if torch.cuda.is_available() and backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            # gloo (CPU tests, or every rank time-sharing the visible GPUs to exercise the N-rank path)
            if torch.cuda.is_available():
                local = local % torch.cuda.device_count()
                torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        return dist, rank, world, local
    return None, 0, 1, 0


def barrier(dist):
    if dist is not None:
        dist.barrier()


def rank_slices(cfg, scaling, rank, world):
    """(start, stop) of this rank's global (batch x head) slices."""
    bh_total = cfg["batch"] * cfg["towers"] * cfg["heads"]
    if scaling == "weak":
        return rank * bh_total, (rank + 1) * bh_total
    return shard(bh_total, rank, world)


# ------------------------------------------------------------------ oracle leg
def oracle_scores(cfg):
    return synth.lra_scores(cfg["L"], cfg["block"], seed=SCORE_SEEDS[0]).numpy()


def oracle_step(cfg, alpha, mode, slices, A, cores, seed=99):
    """One bounded oracle step: the pattern (Alg. 3/4) once, then fwd+bwd of the given (batch, head)
    slices, one slice per host thread (the oracle's C calls release the GIL).  Returns
    (seconds, pattern seconds, blocks)."""
    import concurrent.futures as cf

    import oracle

    L, B, d = cfg["L"], cfg["block"], cfg["d"]
    scale = 1.0 / math.sqrt(d)
    t0 = time.perf_counter()
    fl, _, _ = oracle.pattern(A, B, FILTER, alpha)
    t_pat = time.perf_counter() - t0

    def one(b):
        q, k, v, do = (x[0].double().numpy() for x in synth.qkvdo(1, L, d, seed=seed, dtype=torch.bfloat16,
                                                                  start_bh=b))
        oracle.attn_fwd(q, k, v, fl, B, scale, mode)
        oracle.attn_bwd(q, k, v, do, fl, B, scale, mode)

    if slices:
        with cf.ThreadPoolExecutor(max_workers=cores) as ex:
            list(ex.map(one, slices))
    return time.perf_counter() - t0, t_pat, int(fl.sum())


def oracle_single_slice_seconds(cfg, alpha, mode, A):
    """Single-thread seconds of fwd+bwd for one (batch, head) slice."""
    import oracle

    L, B, d = cfg["L"], cfg["block"], cfg["d"]
    fl, _, _ = oracle.pattern(A, B, FILTER, alpha)
    q, k, v, do = (x[0].double().numpy() for x in synth.qkvdo(1, L, d, seed=99, dtype=torch.bfloat16))
    t = time.perf_counter()
    oracle.attn_fwd(q, k, v, fl, B, 1.0 / math.sqrt(d), mode)
    oracle.attn_bwd(q, k, v, do, fl, B, 1.0 / math.sqrt(d), mode)
    return time.perf_counter() - t


def oracle_sample(cfg, alpha, mode, budget_s, bh_total):
    """cpu_baseline leg (N=1, rank 0): the oracle as it stands on all host cores, on a bounded
    sample (~budget_s of CPU work): pattern once + fwd+bwd of k slices."""
    cores = os.cpu_count() or 1
    A = oracle_scores(cfg)
    t1 = oracle_single_slice_seconds(cfg, alpha, mode, A)
    k = int(max(1, min(bh_total, budget_s / max(t1, 1e-6) * cores * 0.8)))
    if k >= cores:
        k = (k // cores) * cores
    secs, t_pat, _ = oracle_step(cfg, alpha, mode, list(range(k)), A, cores)
    tokens = k * cfg["L"] / cfg["heads"]  # a (batch, head) slice is 1/heads of L tokens' attention work
    desc = (f"pattern once ({t_pat:.2f}s) + fwd+bwd of {k} of {bh_total} (batch,head) slices on {cores} threads "
            f"in {secs - t_pat:.2f}s; value = the sample's tokens ({k} slices x L / heads) / its measured time")
    return {"value": tokens / secs, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
            "single_thread_slice_s": t1, "cpu_model": cpu_model()}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, cfg):
    """--impl reference: the oracle (this tier's reference arm) timed on the host cores, K steps
    after W warm-up steps; each step = the pattern + fwd+bwd of a bounded sample of (batch, head)
    slices (sized so the whole run takes ~--cpu-budget-total seconds); value = the sample's tokens
    over the measured step time.  Under torchrun only rank 0 runs."""
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:  # the oracle runs once, on rank 0's host cores; the other ranks exit without work
        return
    cores = os.cpu_count() or 1
    A = oracle_scores(cfg)
    a, b = rank_slices(cfg, args.scaling, 0, 1)
    bh_total = (b - a) * (world if args.scaling == "weak" else 1)
    t1 = oracle_single_slice_seconds(cfg, args.alpha, args.mode, A)
    per_step_budget = args.cpu_budget_total / (args.steps + args.warmup)
    k = int(max(1, min(bh_total, per_step_budget / max(t1, 1e-6) * cores * 0.8)))
    if k >= cores:
        k = (k // cores) * cores
    slices = list(range(k))
    for _ in range(args.warmup):
        oracle_step(cfg, args.alpha, args.mode, slices, A, cores)
    times = []
    for _ in range(args.steps):
        secs, t_pat, nnzb = oracle_step(cfg, args.alpha, args.mode, slices, A, cores)
        times.append(secs)
    t_step = statistics.mean(times)  # measured seconds per (sampled) step, pattern included
    tokens = k * cfg["L"] / cfg["heads"]  # a (batch, head) slice is 1/heads of L tokens' attention work
    value = tokens / t_step
    desc = (f"{args.steps} timed steps after {args.warmup} warm-up; each step = the pattern (Alg. 3/4) once + "
            f"fwd+bwd of {k} of the config's {bh_total} (batch,head) slices on {cores} threads; value = the "
            f"sample's tokens ({k} slices x L / heads) / measured step time (no extrapolation)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_dict(cfg, args, world),
        "pattern": {"nnzb": nnzb, "score_seed": SCORE_SEEDS[0]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                         "single_thread_slice_s": t1, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
class Phases:
    """One step's calls, eager or as three CUDA graphs (pattern / fwd / bwd) with timing events
    recorded between the graph launches on the launching stream."""

    def __init__(self, fns, use_graphs, stream):
        self.fns, self.graphs, self.stream = fns, None, stream
        if use_graphs:
            self.graphs = []
            for fn in fns:
                if fn is None:
                    self.graphs.append(None)
                    continue
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    fn()
                self.graphs.append(g)

    def run(self, k):
        if self.graphs is not None:
            g = self.graphs[k]
            if g is not None:
                g.replay()
        elif self.fns[k] is not None:
            self.fns[k]()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="spion", choices=["spion", "reference"])
    ap.add_argument("--config", default="text", choices=sorted(CONFIGS))
    ap.add_argument("--alpha", type=float, default=None,
                    help="flood-fill quantile (default per config: ~10%% block density on the synthetic scores)")
    ap.add_argument("--mode", default="paper", choices=["paper", "masked"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-graphs", action="store_true", help="launch eagerly instead of CUDA-graph replays")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="run each step's pattern on the attention stream (default: the next step's pattern "
                         "runs on a second stream, concurrent with this step's attention)")
    ap.add_argument("--pattern-exchange", default="allreduce", choices=["allreduce", "broadcast"],
                    help="N ranks: sum per-rank partial pools (each rank pools L/N score rows) or broadcast "
                         "rank 0's pattern")
    ap.add_argument("--pipeline-depth", type=int, default=None,
                    help="pipelined steps: step i launches the pattern of step i+D (default 1 on one GPU; 3 with "
                         "N ranks, where a rank's attention share is shorter than the pattern's latency: "
                         "K2 + the collective)")
    ap.add_argument("--emulate-world", type=int, default=1,
                    help="one GPU: run rank 0's share of an E-rank job (its (batch, head) shard, its slab of the "
                         "pattern's score rows; the all-reduced pool delivered by a device copy) to project "
                         "strong scaling without the collective's latency; the line adds emulated_world")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="cpu_baseline leg: seconds of oracle work")
    ap.add_argument("--cpu-budget-total", type=float, default=120.0, help="--impl reference: seconds for the run")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.alpha is None:
        args.alpha = cfg["alpha"]
    if args.warmup < 3:
        args.warmup = 3
    if args.pipeline_depth is None:
        args.pipeline_depth = 1 if max(int(os.environ.get("WORLD_SIZE", args.gpus)), args.emulate_world) <= 1 else 3
    if maybe_self_launch(args):
        return
    if args.impl == "reference":
        return run_reference(args, cfg)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (nRanks) for the record ...
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # ... on stderr: stdout keeps the one JSON line

    from paper_2309_12578_b200 import spion
    from paper_2309_12578_b200 import _native as N
    from paper_2309_12578_b200.dist import allreduce_pool, broadcast_pattern, pattern_rows

    dist, rank, world, local = dist_setup()
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    hbm_peak, tc_peak, tc_sust, peak_src = load_peaks()

    L, B, H, d = cfg["L"], cfg["block"], cfg["heads"], cfg["d"]
    emu = args.emulate_world if world == 1 else 1     # --emulate-world E: rank 0's share of E ranks
    s0, s1 = rank_slices(cfg, args.scaling, rank, max(world, emu))
    bh = s1 - s0                                         # this rank's (batch, head) slices
    bh_total = cfg["batch"] * cfg["towers"] * H * (max(world, emu) if args.scaling == "weak" else 1)
    tokens_job = bh_total // H * L                       # tokens of the whole job per step
    scale = 1.0 / math.sqrt(d)

    # inputs resident in HBM; rotating sets so that between two uses of a set at least 2x the L2
    # of other data is touched (a step never finds its inputs in L2)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    set_bytes = 4 * L * L + 9 * bh * L * d * 2 + 2 * bh * L * 4
    # input sets in rotation (each with its own pattern buffer): >= 2, and one more than the pattern
    # look-ahead so pattern i+D never overwrites a buffer an unfinished step still reads
    NSETS = max(2, 1 + (0 if args.no_pipeline else args.pipeline_depth), min(16, math.ceil(2 * l2 / set_bytes) + 1))
    scores_cpu = [synth.lra_scores(L, B, seed=sd) for sd in SCORE_SEEDS]
    sets, outs = [], []
    for s in range(NSETS):
        A = scores_cpu[s % 2].to(dev)
        q, k, v, do = synth.qkvdo(bh, L, d, seed=7 + 100003 * s, dtype=torch.bfloat16, device=dev, start_bh=s0)
        sets.append((A, q, k, v, do))
        outs.append(dict(o=torch.empty_like(q), lse=torch.empty((bh, L), dtype=torch.float32, device=dev),
                         dq=torch.empty_like(q), dk=torch.empty_like(q), dv=torch.empty_like(q),
                         ws=spion.attn_workspace(bh, L, d, torch.bfloat16, dev)))
    bps = [spion.empty_pattern(L, B, dev) for _ in range(NSETS)]
    stream = torch.cuda.Stream(dev)

    # the per-layer pattern with N ranks: each rank pools its slab of score rows, ONE all-reduce sums
    # the pools, every rank finalises (default); or rank 0 generates it and broadcasts it
    exchange = "emulated" if emu > 1 else (None if world == 1 else args.pattern_exchange)
    p0, p1 = pattern_rows(L, B, rank, max(world, emu))
    if exchange == "emulated":
        # what the all-reduce would deliver: the pool region of the whole matrix (computed once)
        full_regions = [spion.pool_region(spion.pattern_pool(sets[i][0], L, B, filter=FILTER)).clone()
                        for i in range(NSETS)]
        torch.cuda.synchronize()

    def make_phases(i):
        A, q, k, v, do = sets[i]
        o, bp = outs[i], bps[i]
        fin = None
        if exchange in ("allreduce", "emulated"):
            pat = lambda: spion.pattern_pool(A[p0:p1], L, B, filter=FILTER, row_begin=p0, out=bp)
            fin = lambda: spion.pattern_finalize(bp, alpha=args.alpha)
        elif exchange == "broadcast" and rank != 0:
            pat = None
        else:
            pat = lambda: spion.pattern(A, B, filter=FILTER, alpha=args.alpha, out=bp)
        fwd = lambda: spion.attn_fwd(q, k, v, bp, args.mode, scale, out=o["o"], lse=o["lse"], workspace=o["ws"])
        bwd = lambda: spion.attn_bwd(q, k, v, o["o"], do, o["lse"], bp, args.mode, scale, workspace=o["ws"],
                                     dq=o["dq"], dk=o["dk"], dv=o["dv"])
        return [pat, fwd, bwd, fin]

    def exchange_pattern(j):
        """The one collective of the step (NCCL over NVLink; outside the CUDA graphs)."""
        if exchange == "allreduce":
            allreduce_pool(spion.pool_region(bps[j]))
        elif exchange == "emulated":  # one device: the summed pool arrives as a 32 KB device copy
            spion.pool_region(bps[j]).copy_(full_regions[j])
        elif exchange == "broadcast":
            broadcast_pattern(bps[j].flat, src=0)

    with torch.cuda.stream(stream):
        # eager pass first: allocates every pattern workspace, fills the descriptor caches, and
        # counts this library's kernel launches per step
        l0 = spion.launch_count()
        for i in range(NSETS):
            pat, fwd, bwd, fin = make_phases(i)
            if pat is not None:
                pat()
            exchange_pattern(i)
            for fn in (fin, fwd, bwd):
                if fn is not None:
                    fn()
        if exchange in ("allreduce", "emulated"):  # every rank holds exactly the one-device pattern (checked once)
            for i in range(NSETS):
                ref = spion.pattern(sets[i][0], B, filter=FILTER, alpha=args.alpha)
                if not torch.equal(ref.flat, bps[i].flat):
                    raise RuntimeError(f"rank {rank}: all-reduced pattern differs from the one-device pattern")
        launches_per_step = (spion.launch_count() - l0) / NSETS
        torch.cuda.synchronize()
        phases = [Phases(make_phases(i), not args.no_graphs, stream) for i in range(NSETS)]

        # Pipelined steps (default): step i runs fwd + bwd of input set i on `stream` once pattern i is
        # ready, and launches pattern i+1 (an independent input) on `pstream`, so the pattern kernels
        # (the single-CTA finalize in particular) overlap this step's attention.  Every step still does
        # the whole hot path: K timed steps contain exactly K patterns, K forwards and K backwards.
        pstream = torch.cuda.Stream(dev)
        pat_done = [torch.cuda.Event() for _ in range(NSETS)]
        att_done = [torch.cuda.Event() for _ in range(NSETS)]
        for e in att_done:
            e.record(stream)

        def pattern_on_pstream(j, ev=None):
            pstream.wait_event(att_done[j])  # the last attention that read pattern buffer j is done
            with torch.cuda.stream(pstream):
                if ev is not None:
                    ev[0].record(pstream)
                phases[j].run(0)
                exchange_pattern(j)  # the per-layer pattern: one NCCL collective
                phases[j].run(3)
                if ev is not None:
                    ev[1].record(pstream)
                pat_done[j].record(pstream)

        def step(i, ev=None):
            j = i % NSETS
            ph = phases[j]
            if args.no_pipeline:
                if ev is not None:
                    ev[0].record(stream)
                ph.run(0)
                exchange_pattern(j)  # the per-layer pattern: one NCCL collective
                ph.run(3)
                if ev is not None:
                    ev[1].record(stream)
            else:
                stream.wait_event(pat_done[j])
            if ev is not None:
                ev[2].record(stream)
            ph.run(1)
            if ev is not None:
                ev[3].record(stream)
            ph.run(2)
            if ev is not None:
                ev[4].record(stream)
            if not args.no_pipeline:
                att_done[j].record(stream)
                pattern_on_pstream((i + args.pipeline_depth) % NSETS, ev[5:] if ev is not None else None)

        if not args.no_pipeline:
            for j in range(args.pipeline_depth):
                pattern_on_pstream(j % NSETS)
        for i in range(args.warmup):
            step(i)
        torch.cuda.synchronize()
    nnzb_sets = [bp_.nnzb for bp_ in bps[:2]]
    nnzb = sum(nnzb_sets) / len(nnzb_sets)
    density = nnzb / (L // B) ** 2

    # ---- timed region: K steps; events on the launching stream at the phase boundaries
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(7)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream), ClockSampler(dev.index if dev.index is not None else 0) as clk:
        barrier(dist)
        torch.cuda.synchronize()
        start.record(stream)
        for i in range(args.warmup, args.warmup + args.steps):
            step(i, evs[i - args.warmup])
        if not args.no_pipeline:
            # the K-th pattern launched in the region
            stream.wait_event(pat_done[(args.warmup + args.steps + args.pipeline_depth - 1) % NSETS])
        end.record(stream)
        torch.cuda.synchronize()
        barrier(dist)
    launches = int(round(launches_per_step * args.steps))
    ms = start.elapsed_time(end) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ph = {"pattern": [], "fwd": [], "bwd": []}
    for e in evs:
        ph["pattern"].append(e[0].elapsed_time(e[1]) if args.no_pipeline else e[5].elapsed_time(e[6]))
        ph["fwd"].append(e[2].elapsed_time(e[3]))
        ph["bwd"].append(e[3].elapsed_time(e[4]))
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
    dom = max(("fwd", "bwd"), key=ph_ms.get)
    t_dom = ph_ms[dom] * 1e-3
    gbs = alg[dom] / t_dom / 1e9
    traffic = ncu_traffic(args.config, dom) if world == 1 else None
    roofline = {"kernel": f"spion_attn_{dom}", "bound": "hbm",
                "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak, "traffic": traffic,
                "traffic_source": TRAFFIC_FILE if traffic is not None else None,
                "peak_source": peak_src + " (MEASURED_PEAKS.json hbm_gbs: copy bandwidth)",
                "alg_bytes_per_launch": alg[dom], "alg_bytes_per_row": (16 * d + 4) if dom == "bwd" else (8 * d + 4),
                "ms_per_launch": ph_ms[dom], "useful_tflops": flops[dom] / t_dom / 1e12 if flops[dom] else 0.0}
    step_flops = accounting.useful_flops(B, d, nnzb, bh)
    value = tokens_job / (ms * 1e-3)

    # ---- end to end through the C ABI from pinned host buffers (H2D + D2H inside the timed region)
    e2e = None
    if args.e2e_steps > 0:
        import ctypes
        lib = N.lib()
        A, q, k, v, do = sets[0]
        hA = scores_cpu[0].pin_memory()
        hq, hk, hv, hdo = (x.cpu().pin_memory() for x in (q, k, v, do))
        ho, hdq, hdk, hdv = (torch.empty_like(hq).pin_memory() for _ in range(4))
        hlse = torch.empty((bh, L), dtype=torch.float32).pin_memory()
        arena_bytes = lib.spion_step_arena_bytes(bh, L, d, B, N.BF16)
        arena = torch.empty(arena_bytes, dtype=torch.uint8, device=dev)
        P = lambda t: ctypes.c_void_p(t.data_ptr())
        nnz = ctypes.c_int32(0)
        strm = ctypes.c_void_p(stream.cuda_stream)

        def host_step():
            st = lib.spion_step_host(P(hA), P(hq), P(hk), P(hv), P(hdo), P(ho), P(hlse), P(hdq), P(hdk), P(hdv),
                                     bh, L, d, B, FILTER, args.alpha, N.THRESH["linear"], N.BF16,
                                     N.SOFTMAX[args.mode], scale, P(arena), arena_bytes, ctypes.byref(nnz), strm)
            N.check(st, "spion_step_host")

        host_step()
        barrier(dist)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            host_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / args.e2e_steps
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        tb = bh * L * d * 2
        e2e = {"value": tokens_job / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": L * L * 4 + 4 * tb,
               "d2h_bytes_per_step": 4 * tb + bh * L * 4, "ms_per_step": ems,
               "path": "spion_step_host (pinned host buffers, per rank)"}
        del arena

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(cfg, args.alpha, args.mode, args.cpu_budget, bh)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": config_dict(cfg, args, world),
            "pattern": {"nnzb": nnzb, "nnzb_sets": nnzb_sets, "block_density": round(density, 4),
                        "score_seeds": list(SCORE_SEEDS)},
            "bh_per_rank": bh, "input_sets": NSETS, "cuda_graphs": not args.no_graphs,
            "phases_ms": ph_ms,
            "useful_tflops": step_flops * max(world, emu) / (ms * 1e-3) / 1e12,
            "pct_bf16_peak_useful": 100.0 * step_flops / (ms * 1e-3) / (tc_peak * 1e12),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if emu > 1:
            line["emulated_world"] = emu
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
