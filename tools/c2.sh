set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py tests/test_memest.py -m gpu -q -x > gpurun_out/c2_pytest.log 2>&1; tail -5 gpurun_out/c2_pytest.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2_reduce tools/micro/l2_reduce.cu && timeout 120 /tmp/l2_reduce > gpurun_out/c2_l2_reduce.txt 2>&1; cat gpurun_out/c2_l2_reduce.txt
bash tools/flce_ab.sh 2>&1 | tee gpurun_out/c2_flce_ab.txt
