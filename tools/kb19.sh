python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python tools/kbench.py c2 dview mttkrp 2>&1 | grep sum_ms
python tools/kbench.py c4 dview phi,mttkrp 2>&1 | grep sum_ms
python tools/kbench.py c3 dview mttkrp 2>&1 | grep sum_ms
