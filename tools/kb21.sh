for b in 16384 32768 65536 131072; do
  ALTO_B200_BLOCK_L1_BYTES=$b ALTO_B200_BLOCK_MIN_RUN=16 python tools/kbench.py c2 dview mttkrp 2>&1 | grep sum_ms | sed "s/^/$b /"
done
ALTO_B200_BLOCK=0 python tools/kbench.py c2 dview mttkrp 2>&1 | grep sum_ms | sed "s/^/noblock /"
