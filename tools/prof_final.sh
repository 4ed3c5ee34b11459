# Round-1 final evidence pass: GPU tests, smoke, bench (ours + reference arm), launch list, traffic, ncu full.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1; tail -2 gpurun_out/final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -c 400 gpurun_out/final_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc_kernel" -s 2 -c 4 -o gpurun_out/final_gemm1sm python tools/prof_step.py --steps 1 --warmup 0 > /dev/null 2>&1
for k in fwd_tc dkdv dq_tc ce_rows; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/final_$k python tools/prof_step.py --steps 1 --warmup 0 > /dev/null 2>&1
done
ls gpurun_out/final_*
