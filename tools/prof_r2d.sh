# Round-2 final evidence pass (gpurun from the repo root): outputs in gpurun_out/r2d_*, summaries copied to profiles/.
# Every step has its own timeout so one hang cannot eat the whole call.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r2d_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d_fin_bench_L1.json 2> gpurun_out/r2d_fin_bench_L1.err; tail -c 300 gpurun_out/r2d_fin_bench_L1.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2d_fin_bench_ref.json 2>/dev/null; tail -c 200 gpurun_out/r2d_fin_bench_ref.json
timeout 600 python bench.py --workload tiny --steps 20 --warmup 5 > gpurun_out/r2d_fin_bench_tiny.json 2>/dev/null; tail -c 200 gpurun_out/r2d_fin_bench_tiny.json
timeout 900 python bench.py --workload tiny --impl reference --steps 20 --warmup 5 > gpurun_out/r2d_fin_bench_tiny_ref.json 2>/dev/null; tail -c 200 gpurun_out/r2d_fin_bench_tiny_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2d_fin_launches.csv python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
for k in fwd_tc128 dkdv dq_tmem ce_rows_exp rmsnorm_bwd; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/r2d_fin_$k -f python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 40 -c 1 -o gpurun_out/r2d_fin_gemm -f python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
timeout 900 python tools/attn_rank_bench.py > gpurun_out/r2d_fin_attn_rank_L8.txt 2>&1; tail -1 gpurun_out/r2d_fin_attn_rank_L8.txt
timeout 900 python tools/attn_rank_bench.py 1048576 8 1 > gpurun_out/r2d_fin_attn_rank_Q8.txt 2>&1; tail -1 gpurun_out/r2d_fin_attn_rank_Q8.txt
timeout 900 python tools/attn_fa4_bench.py 32768:32:8 524288:4:1 > gpurun_out/r2d_fin_fa4.txt 2>&1; tail -2 gpurun_out/r2d_fin_fa4.txt
timeout 1200 python tools/l8_emulation.py --out gpurun_out/r2d_fin_l8_emulation.json > gpurun_out/r2d_fin_l8_emulation.log 2>&1; tail -3 gpurun_out/r2d_fin_l8_emulation.log
timeout 600 python tools/shape_bench.py > gpurun_out/r2d_fin_qwen_shape_32k.json 2>&1; tail -c 300 gpurun_out/r2d_fin_qwen_shape_32k.json
timeout 1500 python tools/max_seq.py --n 786432,1048576,1179648,1310720 --out gpurun_out/r2d_fin_max_seq.json > gpurun_out/r2d_fin_max_seq.log 2>&1; tail -5 gpurun_out/r2d_fin_max_seq.log
ls gpurun_out/r2d_fin_*
