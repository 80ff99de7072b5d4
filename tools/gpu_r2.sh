# round-2 measurement snapshot: smoke, GPU tests, benches (all configs; Text = the default headline),
# reference arm, ncu launch lists + --set full captures.  usage: bash tools/gpu_r2.sh <tag> [quick]
tag=${1:-snap}; o=gpurun_out/$tag; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $o/nvsmi.txt
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $o/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $o/pytest_gpu.log 2>&1; tail -3 $o/pytest_gpu.log
timeout 400 python bench.py --steps 20 --warmup 5 > $o/bench_text.json 2> $o/bench_text.err; tail -c 600 $o/bench_text.err
for c in image listops retrieval; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 --cpu-budget 5 > $o/bench_$c.json 2> $o/bench_$c.err
done
[ "$2" = quick ] && exit 0
timeout 400 python bench.py --impl reference --steps 20 --warmup 5 > $o/bench_reference_text.json 2> $o/bench_ref.err
for c in image listops text retrieval; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_|pattern_|transition" -c 60 --csv \
    --log-file $o/ncu_launches_$c.csv python bench.py --config $c --steps 5 --warmup 3 --no-graphs --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"attn_|pattern_" -s 12 -c 4 \
    -o $o/ncu_full_$c python bench.py --config $c --steps 2 --warmup 3 --no-graphs --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
ls -la $o
