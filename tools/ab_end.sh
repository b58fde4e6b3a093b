# A/B: piece-end accumulation (default build) vs the per-nonzero A_j product (variant end0)
timeout 900 python -m pytest tests/test_gpu_memo_fused.py tests/test_gpu_mttkrp.py tests/test_gpu_call_memo.py tests/test_gpu_drivers.py -x -q > gpurun_out/ab_end_tests.log 2>&1
echo rc=$? >> gpurun_out/ab_end_tests.log
for r in 1 2; do for v in default end0; do
  if [ $v = default ]; then L=""; else L=paper_2403_06348_b200/libalto_b200_$v.so; fi
  ALTO_B200_LIB=$L timeout 400 python bench.py --steps 30 --warmup 5 --no-apr --mttkrp-configs c3 --no-cpu-baseline --no-drivers > gpurun_out/abe_${v}_$r.json 2>gpurun_out/abe_${v}_$r.err
done; done
