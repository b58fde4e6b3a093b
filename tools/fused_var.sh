for v in default fu2 fu1; do
  if [ $v = default ]; then L=""; else L=paper_2403_06348_b200/libalto_b200_$v.so; fi
  echo "== $v" >> gpurun_out/fused_var.log
  ALTO_B200_LIB=$L python tools/il_ab.py c2 --sums-only --no-hot >> gpurun_out/fused_var.log 2>&1
done
