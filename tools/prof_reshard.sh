mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_cpp_api.py -m gpu -q 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none -k regex:reshard -c 4 -o gpurun_out/reshard_sp8 python tools/prof_step.py --sp 8 --steps 1 --warmup 0 > /dev/null 2>&1
ls -la gpurun_out/reshard_sp8.ncu-rep
