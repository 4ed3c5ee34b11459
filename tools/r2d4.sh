# checkpoint after the forward register split: full GPU suite, smoke, bench (both arms)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2d4_pytest_gpu.txt 2>&1; tail -3 gpurun_out/r2d4_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d4_smoke.txt 2>&1; tail -1 gpurun_out/r2d4_smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d4_bench_L1.json 2> gpurun_out/r2d4_bench_L1.err; tail -c 300 gpurun_out/r2d4_bench_L1.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2d4_bench_ref.json 2> gpurun_out/r2d4_bench_ref.err; tail -c 600 gpurun_out/r2d4_bench_ref.json
