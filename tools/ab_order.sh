for c in c5 c3 c2; do ALTO_B200_VIEW_ORDER=alto timeout 900 python tools/kbench.py $c dview > gpurun_out/ord_alto_$c.log 2>&1; done
ALTO_B200_VIEW_ORDER=alto timeout 600 python tools/kbench.py c4 dview mttkrp,phi > gpurun_out/ord_alto_c4.log 2>&1
