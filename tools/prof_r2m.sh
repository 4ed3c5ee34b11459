# Round-2 last check on the final commit (r2m): the driver's round-end sequence (GPU suite, smoke, bench both arms).
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2m_pytest_gpu.txt 2>&1; tail -2 gpurun_out/r2m_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2m_smoke.txt 2>&1; tail -1 gpurun_out/r2m_smoke.txt
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2m_bench_L1.json 2> gpurun_out/r2m_bench_L1.err; tail -c 300 gpurun_out/r2m_bench_L1.json
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2m_bench_ref.json 2>/dev/null; tail -c 300 gpurun_out/r2m_bench_ref.json
timeout 600 python bench.py --workload tiny --steps 20 --warmup 5 > gpurun_out/r2m_bench_tiny.json 2>/dev/null; tail -c 200 gpurun_out/r2m_bench_tiny.json
timeout 900 python bench.py --workload tiny --impl reference --steps 20 --warmup 5 > gpurun_out/r2m_bench_tiny_ref.json 2>/dev/null; tail -c 400 gpurun_out/r2m_bench_tiny_ref.json
timeout 600 python bench.py --workload qwen --steps 10 --warmup 3 > gpurun_out/r2m_bench_qwen.json 2>/dev/null; tail -c 300 gpurun_out/r2m_bench_qwen.json
