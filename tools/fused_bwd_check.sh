# First validation of the fused dK/dV/dQ backward: watchdog build, bounded time, attention tests then bench.
mkdir -p gpurun_out
rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
SPT_WATCHDOG=1 python -c "from paper_2506_13996_b200 import build as B; B.build()"
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k attention > gpurun_out/fused_tests_wd.log 2>&1; echo "rc=$?"; tail -15 gpurun_out/fused_tests_wd.log
rm -f paper_2506_13996_b200/_build/attention_tc.cu.o
python -c "from paper_2506_13996_b200 import build as B; B.build()"
timeout 300 python -m pytest tests -m gpu -q -x -k "attention or layer" > gpurun_out/fused_tests.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/fused_tests.log
timeout 120 python tools/attn_bench.py
SPT_ATTN_BWD=2pass timeout 120 python tools/attn_bench.py
