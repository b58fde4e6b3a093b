timeout 600 python tools/kbench.py c2 dview > gpurun_out/abl_base.log 2>&1
for v in nogather nostage both; do ALTO_B200_LIB=paper_2403_06348_b200/libalto_b200_$v.so timeout 600 python tools/kbench.py c2 dview > gpurun_out/abl_$v.log 2>&1; done
