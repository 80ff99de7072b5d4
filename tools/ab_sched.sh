# scheduler A/B: bench + bwd DRAM bytes per variant.  usage: bash tools/ab_sched.sh "<variants>"
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q --tb=short 2>&1 | tail -2
bash tools/gpu_ab.sh absched "text image" $1
for v in $1; do
  if [ $v = base ]; then lib=""; else lib=build_variants/$v/libspion.so; fi
  SPION_LIB=$lib timeout 300 ncu --metrics dram__bytes_read.sum -k regex:"attn_bwd" -s 6 -c 2 --csv python bench.py --config text --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | grep -E "dram__bytes" | awk -F'","' '{print "'$v'", substr($5,1,30), $NF}'
done
