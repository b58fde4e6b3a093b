python tools/memo_split_prof.py > gpurun_out/msp_base.log 2>&1
for m in 3 4; do ALTO_B200_LIB=paper_2403_06348_b200/libalto_b200_minb$m.so python tools/memo_split_prof.py > gpurun_out/msp_minb$m.log 2>&1; done
