for v in 0 1; do ALTO_B200_DV_FIBER=$v timeout 600 python tools/kbench.py c2 dview > gpurun_out/kb8_c2_$v.log 2>&1; ALTO_B200_DV_FIBER=$v timeout 600 python tools/kbench.py c4 dview > gpurun_out/kb8_c4_$v.log 2>&1; done
ALTO_B200_DV_FIBER=1 python -m pytest tests/test_gpu_mttkrp.py tests/test_gpu_drivers.py -q -x > gpurun_out/t_dvf.log 2>&1; tail -1 gpurun_out/t_dvf.log
ALTO_B200_DV_FIBER=1 ALTO_B200_DETERMINISTIC=1 python -m pytest tests/test_gpu_deterministic.py -q -x > gpurun_out/t_dvf_det.log 2>&1; tail -1 gpurun_out/t_dvf_det.log
