# usage: bash tools/gpu_profile.sh <tag> [config]   (run under gpurun; outputs in gpurun_out/<tag>/)
tag=${1:-p}; cfg=${2:-text}
o=gpurun_out/$tag; mkdir -p $o
for c in image listops text retrieval; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 2 > $o/bench_$c.json 2> $o/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_$cfg.csv \
  python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"attn_|pattern_" -s 15 -c 5 \
  -o $o/full_$cfg python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $o/ncu_full.log 2>&1
ls -la $o
