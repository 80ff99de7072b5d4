#!/usr/bin/env python
"""Summarise ncu output for profiles/.

  python tools/ncu_summary.py rep  <file.ncu-rep> [alg_bytes_per_launch ...]
  python tools/ncu_summary.py list <launches.csv>

`rep`: key metrics per profiled kernel (time, DRAM bytes, throughput %, tensor-pipe %,
occupancy, registers) and the top warp-stall reasons.  `list`: per-kernel launch counts,
total device time and share of the listed launches (cold-cache, serialised replays:
compare shares, not absolutes).
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("time_us", "gpu__time_duration.sum", 1e-3),
    ("dram_read_MB", "dram__bytes_read.sum", None),
    ("dram_write_MB", "dram__bytes_write.sum", None),
    ("dram_pct_peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed", None),
    ("tensor_utchmma_bf16_pct", "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", None),
    ("tensor_pipe_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", None),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", None),
    ("registers", "launch__registers_per_thread", None),
    ("grid", "launch__grid_size", None),
    ("block", "launch__block_size", None),
    ("smem_dyn_B", "launch__shared_mem_per_block_dynamic", None),
]


def _to_bytes(v, unit):
    v = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    return v * scale


def rep(path, alg=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for k, vals in enumerate(rows[2:]):
        m = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print(f"== {m.get('Kernel Name', '?')[:110]}")
        for label, key, _ in KEYS:
            if key not in m:
                continue
            v = m[key]
            if key.startswith("dram__bytes"):
                v = f"{_to_bytes(v, u[key]) / 1e6:.2f}"
            elif key == "gpu__time_duration.sum":
                t = float(v.replace(",", ""))
                v = f"{t * {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1, 'us': 1, 'msecond': 1e3, 'ms': 1e3}.get(u[key], 1):.2f}"
            print(f"   {label:26s} {v}")
        if alg and k < len(alg):
            rd = _to_bytes(m["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
            wr = _to_bytes(m["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
            print(f"   {'traffic/alg_bytes':26s} {(rd + wr) / float(alg[k]):.3f}  (alg {float(alg[k]) / 1e6:.2f} MB)")
        stalls = []
        for key, v in m.items():
            if key.startswith("smsp__average_warps_issue_stalled_") and key.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v.replace(",", "")), key[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        if stalls:
            print("   top stalls (warps per issue): " + ", ".join(f"{n}={v:.2f}" for v, n in stalls[:6]))


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0][:80]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r["Metric Unit"], 1.0)
        tot[name] += float(r["Metric Value"].replace(",", "")) * scale
        cnt[name] += 1
    allt = sum(tot.values())
    print(f"{'kernel':82s} {'launches':>8s} {'total_us':>10s} {'share':>6s}")
    for name, t in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{name:82s} {cnt[name]:8d} {t:10.1f} {100 * t / allt:5.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "rep":
        rep(sys.argv[2], sys.argv[3:] or None)
    else:
        launches(sys.argv[2])
