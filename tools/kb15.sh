python tools/kbench.py c2 dview mttkrp > gpurun_out/kb15.log 2>&1
ALTO_B200_BLOCK=0 python tools/kbench.py c2 dview mttkrp >> gpurun_out/kb15.log 2>&1
python tools/kbench.py c4 dview phi >> gpurun_out/kb15.log 2>&1
ALTO_B200_BLOCK_MIN_RUN=4 python tools/kbench.py c4 dview phi >> gpurun_out/kb15.log 2>&1
ALTO_B200_BLOCK_MIN_RUN=16 python tools/kbench.py c3 dview mttkrp >> gpurun_out/kb15.log 2>&1
python tools/kbench.py c3 dview mttkrp >> gpurun_out/kb15.log 2>&1
grep '"mode"\|sum_ms' gpurun_out/kb15.log
