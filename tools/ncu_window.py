"""SASS window (with stall samples) around an address of one kernel in an ncu report.
   python tools/ncu_window.py rep kernel_regex addr_suffix [before] [after]"""
import csv, subprocess, sys
rep, kern, addr = sys.argv[1], sys.argv[2], sys.argv[3].lower()
bef = int(sys.argv[4]) if len(sys.argv) > 4 else 30
aft = int(sys.argv[5]) if len(sys.argv) > 5 else 10
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Address" in r)
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
body, seen = [], set()
for r in rows[rows.index(hdr) + 1:]:
    if len(r) > iss and r[ia] not in seen:
        seen.add(r[ia]); body.append(r)
idx = next(i for i, r in enumerate(body) if r[ia].lower().endswith(addr))
for r in body[max(0, idx - bef): idx + aft]:
    print(f"{r[iss]:>6} {r[ia][-5:]} {r[isrc][:110]}")
