# A/B of library variants (tools/build_variant.py NAME -D...): bench_variants.sh NAME...
for r in 1 2; do for v in default "$@"; do
  if [ $v = default ]; then L=""; else L=paper_2403_06348_b200/libalto_b200_$v.so; fi
  ALTO_B200_LIB=$L python bench.py --steps 30 --warmup 5 --no-apr --mttkrp-configs '' --no-cpu-baseline --no-drivers > gpurun_out/bv_${v}_$r.json 2>/dev/null
done; done
