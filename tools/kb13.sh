for lib in default b128m5 b128m6 b128m5u2; do
  if [ $lib = default ]; then L=""; else L="ALTO_B200_LIB=paper_2403_06348_b200/libalto_b200_$lib.so"; fi
  env $L python tools/kbench.py c2 dview mttkrp
done > gpurun_out/kb13.log 2>&1
grep sum_ms gpurun_out/kb13.log
