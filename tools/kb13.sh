python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python tools/kbench.py c2 dview mttkrp > gpurun_out/kb13.log 2>&1
python tools/kbench.py c4 dview phi,mttkrp >> gpurun_out/kb13.log 2>&1
grep sum_ms gpurun_out/kb13.log
