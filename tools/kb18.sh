ALTO_B200_LIB=paper_2403_06348_b200/libalto_b200_u4m2.so timeout 900 python -m pytest tests -x -q -m gpu -k "phi or apr or drivers" 2>&1 | tail -2
for i in 1 2; do
for lib in default nods u4m2 u4m2nods; do
  if [ $lib = default ]; then L=""; else L="ALTO_B200_LIB=paper_2403_06348_b200/libalto_b200_$lib.so"; fi
  env $L python tools/kbench.py c4 dview phi > gpurun_out/kb18.log 2>&1; grep sum_ms gpurun_out/kb18.log
done
done
