for v in base k2t512 k2t256; do
  if [ $v = base ]; then lib=""; else lib=build_variants/$v/libspion.so; fi
  echo "== $v"; SPION_LIB=$lib python tools/trace_k2.py 2>&1 | grep -v "bsr+plan:\|thresh:"
done
SPION_LIB=build_variants/k2t256/libspion.so python -m pytest tests/test_gpu_pattern.py -q -x 2>&1 | tail -1
