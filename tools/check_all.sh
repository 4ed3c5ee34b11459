# Full GPU parity suite + attention timing + GEMM site timing of the current build.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python tools/attn_bench.py 2>&1 | tee gpurun_out/attn_bench.txt
python tools/gemm_sites.py 2>&1 | tail -1
