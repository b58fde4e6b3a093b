set -x
python -m pytest tests/test_gpu_mttkrp.py -q -x -k "segment" > gpurun_out/t_seg.log 2>&1; tail -3 gpurun_out/t_seg.log
for c in c3 c5; do timeout 900 python tools/kbench.py $c dview,segment,segment-atomic,oriented,atomic > gpurun_out/kb_$c.log 2>&1; done
timeout 600 python tools/kbench.py c2 dview,segment,segment-atomic > gpurun_out/kb_c2.log 2>&1
timeout 600 python tools/kbench.py c4 dview,segment > gpurun_out/kb_c4.log 2>&1
ALTO_B200_SEG_WAVES=1 timeout 600 python tools/kbench.py c3 segment > gpurun_out/kb_c3_w1.log 2>&1
ALTO_B200_SEG_WAVES=4 timeout 600 python tools/kbench.py c3 segment > gpurun_out/kb_c3_w4.log 2>&1
