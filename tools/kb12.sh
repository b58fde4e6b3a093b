python -m pytest tests -x -q -m gpu -k "dview or scale or phi or drivers" > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for v in 2 3; do
  ALTO_B200_DV=$v python tools/kbench.py c2 dview mttkrp
  ALTO_B200_DV=$v python tools/kbench.py c4 dview phi,mttkrp
done > gpurun_out/kb12.log 2>&1
grep sum_ms gpurun_out/kb12.log
