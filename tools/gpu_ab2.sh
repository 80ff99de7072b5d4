# A/B timing of library variants and env settings on the text config:
#   bash tools/gpu_ab2.sh <tag> "<configs>" "name:VAR=val,VAR2=val:variantdir" ...   (variantdir "" = in-tree lib)
tag=$1; cfgs=$2; shift 2
o=gpurun_out/$tag; mkdir -p $o
for spec in "$@"; do
  name=${spec%%:*}; rest=${spec#*:}; envs=${rest%%:*}; v=${rest#*:}
  lib=""; [ -n "$v" ] && lib=build_variants/$v/libspion.so
  for c in $cfgs; do
    env SPION_LIB=$lib $(echo $envs | tr ',' ' ') timeout 180 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $o/bench_${name}_$c.json 2> $o/bench_${name}_$c.err
    python - <<PY
import json
try:
    d=json.load(open("$o/bench_${name}_$c.json")); print("%-10s %-9s"%("$name","$c"), round(d["ms_per_step"],4), {k:round(x,4) for k,x in d["phases_ms"].items()})
except Exception as e: print("$name $c FAILED", e, open("$o/bench_${name}_$c.err").read()[-500:])
PY
  done
done
