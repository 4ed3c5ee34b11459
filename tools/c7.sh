mkdir -p gpurun_out
timeout 900 python tools/step_ab.py gemm_raster=0,1,2 --group 12 --rounds 3 > gpurun_out/c7_raster_ab.txt 2>&1; tail -2 gpurun_out/c7_raster_ab.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "attention" > gpurun_out/c7_pytest.log 2>&1; tail -15 gpurun_out/c7_pytest.log
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_multilayer.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/c7_pytest2.log 2>&1; tail -5 gpurun_out/c7_pytest2.log
