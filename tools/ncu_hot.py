"""Hottest SASS instructions (warp-stall samples) of one kernel in an ncu report."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Address" in r)
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
seen, data = set(), []
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= iss or r[ia] in seen:
        continue
    try:
        data.append((int(r[iss]), r[ia], r[isrc])); seen.add(r[ia])
    except ValueError:
        pass
tot = sum(d[0] for d in data)
print("samples", tot)
for d in sorted(data, reverse=True)[:n]:
    print(f"{d[0]:6d} {100 * d[0] / tot:5.1f}% {d[1][-5:]} {d[2][:100]}")
