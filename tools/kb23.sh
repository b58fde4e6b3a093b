python -m pytest tests -x -q -m gpu > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log; grep -E "^E |FAILED" gpurun_out/t.log | head -3
python tools/kbench.py c2 dview mttkrp 2>&1 | grep sum_ms
python tools/kbench.py c4 dview phi,mttkrp 2>&1 | grep sum_ms
python tools/kbench.py c3 dview mttkrp 2>&1 | grep sum_ms
