# quick iteration: attention parity + benches (+ optional trace).  usage: bash tools/gpu_quick.sh <tag> [configs...]
tag=${1:-q}; shift; cfgs=${@:-"text image"}
o=gpurun_out/$tag; mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q > $o/pytest.log 2>&1; tail -3 $o/pytest.log
for c in $cfgs; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 > $o/bench_$c.json 2> $o/bench_$c.err
  python - <<PY
import json; d=json.load(open("$o/bench_$c.json")); print("$c", round(d["ms_per_step"],4), {k:round(v,4) for k,v in d["phases_ms"].items()}, d["config"]["nnzb_sets"], "roof", round(d["roofline"]["frac"],3))
PY
done
