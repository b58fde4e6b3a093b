python -m pytest tests/test_gpu_drivers.py tests/test_gpu_scale.py -q -x -k "memo" > gpurun_out/t_memo.log 2>&1; tail -2 gpurun_out/t_memo.log
python -m pytest tests/test_gpu_multirank.py tests/test_gpu_mttkrp.py -q -x -k "two_ranks or choice" > gpurun_out/t_mr2.log 2>&1; tail -2 gpurun_out/t_mr2.log
for v in 0 1; do ALTO_B200_MEMO_FUSED=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-apr --mttkrp-configs '' --no-cpu-baseline --no-drivers --no-e2e > gpurun_out/bm_fused$v.json 2> gpurun_out/bm_fused$v.err; done
