# Round-1 re-entry evidence pass: GPU tests, smoke, bench, launch list, ncu full captures.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 1000 gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1d.csv python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_tc|dkdv|dq_tc|ce_rows|rmsnorm" -c 5 -o gpurun_out/attn_r1d python tools/prof_step.py --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 12 -c 6 -o gpurun_out/gemm_r1d python tools/prof_step.py --steps 1 --warmup 0 > /dev/null 2>&1
ls -la gpurun_out
