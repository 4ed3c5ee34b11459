# Round-1 evidence pass: GPU tests, bench (device + e2e + CPU baseline), launch list, ncu full captures.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 12 -c 4 -o gpurun_out/gemm_r1c python tools/prof_step.py --steps 1 --warmup 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"fwd_tc|dkdv|dq_tc|ce_rows|rmsnorm" -c 5 -o gpurun_out/attn_r1c python tools/prof_step.py --steps 1 --warmup 0 > /dev/null 2>&1
ls -la gpurun_out
