mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "gemm or flce or mlp" > gpurun_out/c6_pytest.log 2>&1; tail -2 gpurun_out/c6_pytest.log
timeout 900 python tools/step_ab.py gemm_raster=0,1 --group 12 --rounds 4 > gpurun_out/c6_raster_ab.txt 2>&1; tail -4 gpurun_out/c6_raster_ab.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c6_launches.csv python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
timeout 900 python tools/attn_fwd_ab.py 1,13,16 32768:32:8 524288:4:1 --rounds 8 > gpurun_out/c6_fwd_ab.txt 2>&1; grep -v " O rel" gpurun_out/c6_fwd_ab.txt
