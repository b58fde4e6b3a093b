for b in 16384 32768 65536 131072; do ALTO_B200_BLOCK_L1_BYTES=$b timeout 600 python tools/kbench.py c2 dview > gpurun_out/kb_blk_$b.log 2>&1; done
ALTO_B200_BLOCK=0 timeout 600 python tools/kbench.py c2 dview > gpurun_out/kb_blk_0.log 2>&1
