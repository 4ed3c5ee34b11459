# Round-2 closing pass (r2f) on the final code: GPU suite + smoke, bench (both arms, L1 and tiny), config F sweep,
# attention yardsticks at the L1 / L8-rank shapes, launch list with DRAM bytes.  Each step under its own timeout.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r2f_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2f_pytest_gpu.txt 2>&1; tail -2 gpurun_out/r2f_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.txt 2>&1; tail -1 gpurun_out/r2f_smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench_L1.json 2> gpurun_out/r2f_bench_L1.err; tail -c 300 gpurun_out/r2f_bench_L1.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2f_bench_ref.json 2>/dev/null; tail -c 200 gpurun_out/r2f_bench_ref.json
timeout 600 python bench.py --workload tiny --steps 20 --warmup 5 > gpurun_out/r2f_bench_tiny.json 2>/dev/null; tail -c 200 gpurun_out/r2f_bench_tiny.json
timeout 1500 python tools/flce_sweep.py --n 65536,262144,1048576 --tiles 2048,4096,8192 --out gpurun_out/r2f_flce_sweep.json > gpurun_out/r2f_flce_sweep.log 2>&1; tail -4 gpurun_out/r2f_flce_sweep.log
timeout 900 python tools/attn_rank_bench.py 32768 32 8 > gpurun_out/r2f_attn_L1.txt 2>&1; tail -1 gpurun_out/r2f_attn_L1.txt
timeout 900 python tools/attn_rank_bench.py > gpurun_out/r2f_attn_L8rank.txt 2>&1; tail -1 gpurun_out/r2f_attn_L8rank.txt
timeout 900 python tools/attn_fa4_bench.py 32768:32:8 524288:4:1 > gpurun_out/r2f_fa4.txt 2>&1; tail -2 gpurun_out/r2f_fa4.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2f_launches.csv python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
ls gpurun_out/r2f_*
