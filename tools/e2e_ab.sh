# e2e A/B: bash tools/e2e_ab.sh "<configs>" variants...
cfgs=$1; shift
for v in "$@"; do
  if [ $v = base ]; then lib=""; else lib=build_variants/$v/libspion.so; fi
  for c in $cfgs; do
    SPION_LIB=$lib timeout 200 python bench.py --config $c --steps 5 --no-cpu-baseline --e2e-steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$c', round(d['e2e']['ms_per_step'],3), '%.3g' % d['e2e']['value'])"
  done
done
