# launch list (time + DRAM bytes per kernel) of the bench's c2 sweep with the fused producer and streaming
# consumer, then one full capture of each
python bench.py --steps 2 --warmup 3 --no-apr --mttkrp-configs "" --no-cpu-baseline --no-drivers --no-e2e > gpurun_out/p_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"memo_|als_" --csv --log-file gpurun_out/r02_launches_bench_c2_fused.csv python bench.py --steps 2 --warmup 3 --no-apr --mttkrp-configs "" --no-cpu-baseline --no-drivers --no-e2e > gpurun_out/p_ncu1.log 2>&1
python tools/prof_fused.py > gpurun_out/p_f.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"memo_fused|memo_consume" -s 2 -c 2 -o gpurun_out/r02_fused_consume python tools/prof_fused.py > gpurun_out/p_ncu2.log 2>&1
