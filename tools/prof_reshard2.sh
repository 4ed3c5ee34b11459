mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_cpp_api.py -m gpu -q > gpurun_out/cpp_gpu.log 2>&1; tail -1 gpurun_out/cpp_gpu.log
timeout 900 ncu --set full --clock-control none -k regex:reshard -c 4 -o gpurun_out/reshard_sp8_256k python tools/prof_step.py --seq 262144 --sp 8 --steps 1 --warmup 0 > gpurun_out/reshard_run.log 2>&1
tail -2 gpurun_out/reshard_run.log
