ALTO_B200_LIB=paper_2403_06348_b200/libalto_b200_pf.so timeout 900 python -m pytest tests -x -q -m gpu -k "dview" 2>&1 | tail -2
for lib in default pf; do
  if [ $lib = default ]; then L=""; else L="ALTO_B200_LIB=paper_2403_06348_b200/libalto_b200_$lib.so"; fi
  env $L python tools/kbench.py c2 dview mttkrp > gpurun_out/kb18.log 2>&1; grep sum_ms gpurun_out/kb18.log
  env $L python tools/kbench.py c4 dview phi > gpurun_out/kb18.log 2>&1; grep sum_ms gpurun_out/kb18.log
  env $L python tools/kbench.py c3 dview mttkrp > gpurun_out/kb18.log 2>&1; grep sum_ms gpurun_out/kb18.log
done
