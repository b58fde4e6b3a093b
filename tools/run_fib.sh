for c in c3 c5; do
for f in short long; do
ALTO_B200_FUSED_MODES=5 ALTO_B200_FUSED_FIBER=$f timeout 900 python tools/kbench.py $c dview 2>&1 | tail -6 | sed "s/^/$f /"
done
done
