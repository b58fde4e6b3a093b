ALTO_B200_MEMO_SPLIT=0 python -m pytest tests/test_gpu_drivers.py tests/test_gpu_scale.py tests/test_gpu_deterministic.py -q -x -k "memo or det" > gpurun_out/t_fj.log 2>&1; tail -1 gpurun_out/t_fj.log
python tools/memo_split_prof.py > gpurun_out/msp_fj.log 2>&1
for r in 1 2; do for v in 0 1; do ALTO_B200_MEMO_SPLIT=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-apr --mttkrp-configs '' --no-cpu-baseline --no-drivers --no-e2e > gpurun_out/bm7_${v}_$r.json 2>/dev/null; done; done
