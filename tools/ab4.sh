python -m pytest tests/test_gpu_mttkrp.py tests/test_gpu_phi.py tests/test_gpu_drivers.py -q -x > gpurun_out/t_v4.log 2>&1; tail -2 gpurun_out/t_v4.log
ALTO_B200_MEMO_SPLIT=1 python -m pytest tests/test_gpu_drivers.py -q -x -k memo > gpurun_out/t_split.log 2>&1; tail -2 gpurun_out/t_split.log
python tools/memo_split_prof.py > gpurun_out/msp2.log 2>&1
for v in 0 1; do ALTO_B200_MEMO_SPLIT=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-apr --mttkrp-configs '' --no-cpu-baseline --no-drivers --no-e2e > gpurun_out/bm_split$v.json 2>/dev/null; done
