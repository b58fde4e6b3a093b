python -m pytest tests -x -q -m gpu -k "phi or apr or drivers or scale" 2>&1 | tail -2
for i in 1 2; do
python tools/kbench.py c4 dview phi > gpurun_out/kb16.log 2>&1; grep sum_ms gpurun_out/kb16.log
ALTO_B200_LIB=paper_2403_06348_b200/libalto_b200_ieee.so python tools/kbench.py c4 dview phi > gpurun_out/kb16.log 2>&1; grep sum_ms gpurun_out/kb16.log
done
