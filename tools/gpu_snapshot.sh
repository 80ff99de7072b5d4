# full measurement snapshot: tests, benches (all configs, with CPU baseline), reference arm, ncu launch
# lists + --set full captures.  usage: bash tools/gpu_snapshot.sh <tag>
tag=${1:-snap}; o=gpurun_out/$tag; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $o/nvsmi.txt
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest_gpu.log 2>&1; tail -2 $o/pytest_gpu.log
for c in image listops text retrieval; do
  timeout 300 python bench.py --config $c > $o/bench_$c.json 2> $o/bench_$c.err
done
timeout 300 python bench.py --impl reference > $o/bench_reference_image.json 2> $o/bench_ref.err
for c in image text; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_|pattern_" -c 80 --csv \
    --log-file $o/ncu_launches_$c.csv python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"attn_|pattern_" -s 15 -c 5 \
    -o $o/ncu_full_$c python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
ls -la $o
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $o/smoke.log 2>&1; tail -1 $o/smoke.log
