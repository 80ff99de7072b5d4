"""Copy a gpu_snapshot.sh run (gpurun_out/<tag>) into profiles/<round>/: bench lines, ncu launch
lists, --set full summaries (ncu_summary.md) and per-call DRAM traffic (ncu_traffic.json).
    python tools/snapshot_to_profiles.py gpurun_out/s2 profiles/r1"""
import os, shutil, subprocess, sys

src, dst = sys.argv[1], sys.argv[2]
os.makedirs(dst, exist_ok=True)
for f in sorted(os.listdir(src)):
    if f.startswith("bench_") and f.endswith(".json") or f.startswith("ncu_launches_"):
        shutil.copy(os.path.join(src, f), os.path.join(dst, f))
reps = {f[len("ncu_full_"):-len(".ncu-rep")]: os.path.join(src, f) for f in os.listdir(src) if f.startswith("ncu_full_")}
args = [f"{k}={v}" for k, v in sorted(reps.items())]
subprocess.run([sys.executable, "tools/ncu_traffic.py", os.path.join(dst, "ncu_traffic.json"), *args], check=True,
               capture_output=True)


def run(*a):
    return subprocess.run([sys.executable, "tools/ncu_summary.py", *a], capture_output=True, text=True).stdout


old = open(os.path.join(dst, "ncu_summary.md")).read() if os.path.exists(os.path.join(dst, "ncu_summary.md")) else ""
micro = old[old.index("## Microbenchmarks"):] if "## Microbenchmarks" in old else ""
nv = open(os.path.join(src, "nvsmi.txt")).read().strip() if os.path.exists(os.path.join(src, "nvsmi.txt")) else ""
out = [f"# ncu summaries, {os.path.basename(os.path.normpath(dst))} (snapshot `{os.path.basename(src)}`)\n",
       "`tools/gpu_r2.sh` (or `gpu_snapshot.sh`) on one B200; `ncu --set full --clock-control none` (cold-cache, serialised",
       "replays: compare shares, not absolutes). Bench lines of the same build: `bench_*.json`; DRAM traffic",
       "per call: `ncu_traffic.json` (the backward reads more than its algorithmic bytes because the dQ and",
       "dK/dV kernels both read Q, K, V and dO).", "", "```", nv, "```", ""]
for c in sorted(f[len("ncu_launches_"):-4] for f in os.listdir(src) if f.startswith("ncu_launches_")):
    out += [f"## Launch list, {c}", "```", run("list", os.path.join(src, f"ncu_launches_{c}.csv")), "```", ""]
for c, rep in sorted(reps.items()):
    out += [f"## --set full, {c}", "```", run("rep", rep), "```", ""]
open(os.path.join(dst, "ncu_summary.md"), "w").write("\n".join(out) + "\n" + micro)
print("wrote", dst)
