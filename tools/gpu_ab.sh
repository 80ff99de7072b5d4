# A/B timing of library variants: bash tools/gpu_ab.sh <tag> "<configs>" variant1 variant2 ...   ("base" = in-tree lib)
tag=$1; cfgs=$2; shift 2
o=gpurun_out/$tag; mkdir -p $o
for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib=build_variants/$v/libspion.so; fi
  for c in $cfgs; do
    SPION_LIB=$lib timeout 120 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 > $o/bench_${v}_$c.json 2> $o/bench_${v}_$c.err
    python - <<PY
import json
try:
    d=json.load(open("$o/bench_${v}_$c.json")); print("%-10s %-8s"%("$v","$c"), round(d["ms_per_step"],4), {k:round(x,4) for k,x in d["phases_ms"].items()})
except Exception as e: print("$v $c FAILED", e)
PY
  done
done
