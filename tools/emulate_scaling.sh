# Strong-scaling projection on one GPU: rank 0's share of an E-rank job (bench.py --emulate-world E)
#   bash tools/emulate_scaling.sh <tag> "<configs>"     -> gpurun_out/<tag>/emu_<cfg>_<E>.json + summary
tag=$1; cfgs=${2:-"text image"}
o=gpurun_out/$tag; mkdir -p $o
for c in $cfgs; do
  for e in 1 2 4 8; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --emulate-world $e \
      > $o/emu_${c}_$e.json 2> $o/emu_${c}_$e.err
  done
done
python - <<PY
import json, os
for c in "$cfgs".split():
    base = None
    for e in (1, 2, 4, 8):
        f = "$o/emu_%s_%d.json" % (c, e)
        try:
            d = json.load(open(f))
        except Exception as ex:
            print(c, e, "FAILED", ex); continue
        if e == 1: base = d["ms_per_step"]
        eff = base / (e * d["ms_per_step"]) if base else float("nan")
        print("%-8s E=%d  rank-0 ms/step %.4f  phases %s  job tokens/s %.3e  projected efficiency %.2f" %
              (c, e, d["ms_per_step"], {k: round(v, 4) for k, v in d["phases_ms"].items()}, d["value"], eff))
PY
