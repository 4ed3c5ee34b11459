set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r2d_gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_pytest_gpu.txt 2>&1; tail -3 gpurun_out/r2d_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.txt 2>&1; tail -2 gpurun_out/r2d_smoke.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2d_bench_L1.json 2> gpurun_out/r2d_bench_L1.err; tail -c 400 gpurun_out/r2d_bench_L1.json
