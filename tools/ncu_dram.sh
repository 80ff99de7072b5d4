# per-launch DRAM bytes and duration of the attention kernels (ncu, cold L2 per replay) for library variants:
#   bash tools/ncu_dram.sh <tag> "<configs>" name:variantdir ...   (variantdir "" = in-tree lib)
tag=$1; cfgs=$2; shift 2
o=gpurun_out/$tag; mkdir -p $o
for spec in "$@"; do
  name=${spec%%:*}; v=${spec#*:}
  lib=""; [ -n "$v" ] && lib=build_variants/$v/libspion.so
  for c in $cfgs; do
    SPION_LIB=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:"attn_" -s 6 -c 6 --csv --log-file $o/${name}_${c}.csv \
      python bench.py --config $c --steps 2 --warmup 2 --no-graphs --no-cpu-baseline --e2e-steps 0 > $o/${name}_${c}.log 2>&1
    python tools/ncu_dram_summary.py $o/${name}_${c}.csv "$name $c"
  done
done
