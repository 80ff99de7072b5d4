# pattern-call A/B across builds: bash tools/k1_ab.sh variants...
for v in "$@"; do
  if [ $v = base ]; then lib=""; else lib=build_variants/$v/libspion.so; fi
  echo "== $v"; SPION_LIB=$lib python tools/trace_k2.py 2>&1 | grep "pattern call"
done
