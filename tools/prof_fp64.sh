# fp64-pipe utilisation, DRAM and L2->L1 bytes of the c3 / c5 per-mode MTTKRP kernels (fp64 co-bound)
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__m_xbar2l1tex_read_bytes.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"
python tools/prof_one.py c3 140e6 dview > gpurun_out/pf_c3.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:"memo_fused|dview3" --csv --log-file gpurun_out/r02_c3_fp64.csv python tools/prof_one.py c3 140e6 dview > gpurun_out/pf_c3n.log 2>&1
python tools/prof_one.py c5 500e6 dview > gpurun_out/pf_c5.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:"memo_fused|dview3" --csv --log-file gpurun_out/r02_c5_fp64.csv python tools/prof_one.py c5 500e6 dview > gpurun_out/pf_c5n.log 2>&1
python tools/prof_one.py c2 76e6 dview > gpurun_out/pf_c2.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:"memo_fused|dview3" --csv --log-file gpurun_out/r02_c2_fp64.csv python tools/prof_one.py c2 76e6 dview > gpurun_out/pf_c2n.log 2>&1
tail -2 gpurun_out/pf_c*.log
