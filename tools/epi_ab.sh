mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "gemm or flce or mlp or layer or fullsize" > gpurun_out/epi_tests.log 2>&1; tail -1 gpurun_out/epi_tests.log
for M in 2 1 2 1; do SPT_EPI_TSTORE=$M python tools/gemm_sites.py flce_dW mlp_dWgu mlp_dWd qkv_dW o_dW 2>&1 | tail -1; done
