# session-5 refresh: single-stage A/B, then launch list + full ncu capture of the final fused producer / consumer
run() { L=""; [ "$2" != default ] && L=paper_2403_06348_b200/libalto_b200_$2.so
  ALTO_B200_LIB=$L timeout 400 python bench.py --steps 30 --warmup 5 --no-apr --mttkrp-configs "" --no-cpu-baseline --no-drivers > gpurun_out/s5ab_$1.json 2>gpurun_out/s5ab_$1.err
  python -c "
import json
d=json.loads(open('gpurun_out/s5ab_$1.json').read().strip().splitlines()[-1])
print('$1', d['ms_per_step'], d['mttkrp_ms_per_mode'], d['e2e']['ms_per_step'])"; }
run default_a default
run st1 st1
run st1c43 st1c43
run default_b default
python bench.py --steps 2 --warmup 3 --no-apr --mttkrp-configs "" --no-cpu-baseline --no-drivers --no-e2e > gpurun_out/p_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"memo_|als_" --csv --log-file gpurun_out/r02_launches_bench_c2_final.csv python bench.py --steps 2 --warmup 3 --no-apr --mttkrp-configs "" --no-cpu-baseline --no-drivers --no-e2e > gpurun_out/p_ncu1.log 2>&1
python tools/prof_fused.py > gpurun_out/p_f.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"memo_fused|memo_consume" -s 2 -c 2 -o gpurun_out/r02_fused_consume_final python tools/prof_fused.py > gpurun_out/p_ncu2.log 2>&1
ls -la gpurun_out | tail -5
