mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "reshard or ulysses or sp or layer or q8 or multilayer or cpp" > gpurun_out/resh_tests.log 2>&1; tail -1 gpurun_out/resh_tests.log
timeout 900 ncu --set full --clock-control none -k regex:reshard -c 6 -o gpurun_out/reshard_rows_256k python tools/prof_step.py --seq 262144 --sp 8 --steps 1 --warmup 0 > /dev/null 2>&1
ls gpurun_out/reshard_rows_256k.ncu-rep
