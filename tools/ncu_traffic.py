"""DRAM traffic per launch of each SPION call from `ncu --set full` reports -> profiles/<round>/ncu_traffic.json.

    python tools/ncu_traffic.py profiles/r1/ncu_traffic.json image=<rep> text=<rep> ...

call -> kernels: pattern = pattern_pool + pattern_finalize, fwd = attn_fwd_tc, bwd = attn_bwd_dq_tc + attn_bwd_dkdv_tc.
bench.py reports the dominant call's bytes as roofline.traffic (null for configs not captured)."""
import csv, io, json, subprocess, sys

CALLS = {"pattern": ["pattern_pool", "pattern_finalize"], "fwd": ["attn_fwd_tc"], "bwd": ["attn_bwd_dq_tc", "attn_bwd_dkdv_tc"]}


def traffic(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ik, ir, iw = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = {}
    for r in rows[2:]:
        b = float(r[ir]) * scale[units[ir]] + float(r[iw]) * scale[units[iw]]
        per.setdefault(r[ik], []).append(b)
    res = {}
    for call, ks in CALLS.items():
        tot = 0.0
        for k in ks:
            v = [x for name, xs in per.items() if k in name for x in xs]
            if not v:
                tot = None
                break
            tot += sum(v) / len(v)
        res[call] = tot
    return res


if __name__ == "__main__":
    dst = sys.argv[1]
    try:
        data = json.load(open(dst))
    except FileNotFoundError:
        data = {}
    for a in sys.argv[2:]:
        cfg, rep = a.split("=", 1)
        data[cfg] = traffic(rep)
        data[cfg]["source"] = rep.split("/")[-1]
    json.dump(data, open(dst, "w"), indent=1)
    print(json.dumps(data, indent=1))
