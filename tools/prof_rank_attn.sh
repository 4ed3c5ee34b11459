mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"fwd_tc|dkdv|dq_tc" -c 3 --csv --log-file gpurun_out/rank_attn.csv python tools/attn_rank_bench.py > /dev/null 2>&1
