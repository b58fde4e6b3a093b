python -m pytest tests/test_gpu_mttkrp.py -q -x -k "segment" > gpurun_out/t_seg2.log 2>&1; tail -2 gpurun_out/t_seg2.log
timeout 900 python tools/kbench.py c3 segment,dview > gpurun_out/kb2_c3.log 2>&1
ALTO_B200_SEG_NT512=1 timeout 900 python tools/kbench.py c3 segment > gpurun_out/kb2_c3_512.log 2>&1
timeout 900 python tools/kbench.py c5 segment > gpurun_out/kb2_c5.log 2>&1
timeout 900 python tools/kbench.py c4 segment > gpurun_out/kb2_c4.log 2>&1
python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/t_mr.log 2>&1; tail -2 gpurun_out/t_mr.log
