"""Summarise an ncu --csv metrics log: mean per kernel of DRAM read/write MB and duration (us)."""
import collections, csv, sys
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
acc = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    acc[r[ik].split("(")[0]][r[im]].append(float(r[iv].replace(",", "")))
for k, m in acc.items():
    rd = sum(m["dram__bytes_read.sum"]) / len(m["dram__bytes_read.sum"]) / 1e6
    wr = sum(m["dram__bytes_write.sum"]) / len(m["dram__bytes_write.sum"]) / 1e6
    t = m["gpu__time_duration.sum"]
    print(f"{sys.argv[2] if len(sys.argv) > 2 else ''} {k[:40]:40s} read {rd:8.1f} MB write {wr:7.1f} MB  {sum(t) / len(t) / 1e3:8.1f} us")
