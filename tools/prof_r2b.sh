# Round-2 session-2 evidence pass (gpurun from the repo root): GPU tests, bench, library yardstick, launch list.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r2b_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_pytest_gpu.log 2>&1; tail -3 gpurun_out/r2b_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; tail -c 600 gpurun_out/r2b_bench.json
timeout 900 python tools/attn_fa4_bench.py 32768:32:8 524288:4:1 > gpurun_out/r2b_fa4.txt 2>&1; cat gpurun_out/r2b_fa4.txt | tail -5
timeout 600 python tools/attn_rank_bench.py > gpurun_out/r2b_attn_rank.txt 2>&1; tail -3 gpurun_out/r2b_attn_rank.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2b_launches.csv python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
ls -la gpurun_out/
