# launch list (time + DRAM bytes) of the bench's timed sweeps, then one full capture of the piece-sum kernel
python bench.py --steps 2 --warmup 3 --no-apr --mttkrp-configs "" --no-cpu-baseline --no-drivers --no-e2e > gpurun_out/p_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"dview3_kernel|memo1_kernel|als_" --csv --log-file gpurun_out/r02_launches_bench_c2.csv python bench.py --steps 2 --warmup 3 --no-apr --mttkrp-configs "" --no-cpu-baseline --no-drivers --no-e2e > gpurun_out/p_ncu1.log 2>&1
python tools/prof_sums.py > gpurun_out/p_sums.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"dview3_kernel|memo1_kernel" -s 1 -c 4 -o gpurun_out/r02_sums python tools/prof_sums.py > gpurun_out/p_ncu2.log 2>&1
python -m pytest tests/test_gpu_drivers.py -q -x > gpurun_out/t_drv.log 2>&1; tail -1 gpurun_out/t_drv.log
