# Round-2 evidence pass (run under gpurun from the repo root); outputs in gpurun_out/r2_*, summaries copied to
# profiles/ by hand.  Every step has its own timeout so one hang cannot eat the whole call.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bench_contract.py -q -m gpu > gpurun_out/r2_bench_contract.log 2>&1; tail -1 gpurun_out/r2_bench_contract.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -c 1 -o gpurun_out/r2_gemm python tools/prof_step.py --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 python tools/l8_emulation.py --out gpurun_out/r2_l8_emulation.json > /dev/null 2>&1
timeout 900 python tools/attn_rank_bench.py > gpurun_out/r2_attn_rank_L8.txt 2>&1
timeout 1500 python tools/max_seq.py --n 786432,917504,1048576,1179648 --out gpurun_out/r2_max_seq.json > gpurun_out/r2_max_seq.log 2>&1
ls gpurun_out/r2_*
