# SURVEY §8(d) measurement rows: config F sweep, measured max sequence per GPU, per-rank attention of
# L8/Q8, and per-launch DRAM traffic of every kernel class in one L1 step (ncu, for roofline.traffic).
mkdir -p gpurun_out
timeout 900 python tools/flce_sweep.py --out gpurun_out/flce_sweep.json > gpurun_out/flce_sweep.log 2>&1; tail -2 gpurun_out/flce_sweep.log
timeout 1200 python tools/max_seq.py --attn --out gpurun_out/max_seq.json > gpurun_out/max_seq.log 2>&1; tail -4 gpurun_out/max_seq.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
ls -la gpurun_out | tail -5
