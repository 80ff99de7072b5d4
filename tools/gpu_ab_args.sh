# A/B timing of bench.py argument sets on one config:  bash tools/gpu_ab_args.sh <tag> <config> "<name>|<args>" ...
tag=$1; cfg=$2; shift 2
o=gpurun_out/$tag; mkdir -p $o
for spec in "$@"; do
  name=${spec%%|*}; a=${spec#*|}
  timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 $a > $o/bench_${name}_$cfg.json 2> $o/bench_${name}_$cfg.err
  python - <<PY
import json
try:
    d=json.load(open("$o/bench_${name}_$cfg.json")); print("%-12s %-9s"%("$name","$cfg"), round(d["ms_per_step"],4), {k:round(x,4) for k,x in d["phases_ms"].items()})
except Exception as e: print("$name $cfg FAILED", e, open("$o/bench_${name}_$cfg.err").read()[-800:])
PY
done
