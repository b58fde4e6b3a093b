for lib in default sef sefel; do
  if [ $lib = default ]; then L=""; else L="ALTO_B200_LIB=paper_2403_06348_b200/libalto_b200_$lib.so"; fi
  env $L python tools/kbench.py c3 dview mttkrp > gpurun_out/kb17.log 2>&1; grep sum_ms gpurun_out/kb17.log
  env $L python tools/kbench.py c2 dview mttkrp > gpurun_out/kb17.log 2>&1; grep sum_ms gpurun_out/kb17.log
done
