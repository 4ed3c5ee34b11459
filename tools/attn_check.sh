# Attention parity tests + timing of the current build.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "attention or layer or fullsize" > gpurun_out/attn_tests.log 2>&1; tail -1 gpurun_out/attn_tests.log
python tools/attn_bench.py 2>&1 | tee gpurun_out/attn_bench.txt
