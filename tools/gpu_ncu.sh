# ncu captures: bash tools/gpu_ncu.sh <tag> <config> [kernel-regex]
tag=$1; cfg=${2:-text}; kre=${3:-"attn_|pattern_"}
o=gpurun_out/$tag; mkdir -p $o
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$kre" -c 60 --csv --log-file $o/launches_$cfg.csv \
  python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$kre" -s 15 -c 5 \
  -o $o/full_$cfg python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $o/ncu_full.log 2>&1
ls -la $o
