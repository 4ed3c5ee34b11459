# Final evidence pass #4 (128-key forward, packed fast path, fused RoPE, embedding).
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f4_pytest_gpu.log 2>&1; tail -1 gpurun_out/f4_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; tail -1 gpurun_out/f4_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/f4_bench.json 2> gpurun_out/f4_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f4_bench_ref.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/f4_launches.csv python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
for k in dq_tmem dkdv fwd_tc; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/f4_$k python tools/prof_step.py --steps 1 --warmup 0 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:gemm_tc_kernel -c 1 -o gpurun_out/f4_gemm1sm python tools/prof_step.py --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 python tools/l8_emulation.py --out gpurun_out/f4_l8_emulation.json > /dev/null 2>&1
timeout 600 python tools/attn_rank_bench.py > gpurun_out/f4_attn_rank.txt 2>&1
timeout 900 python tools/attn_rank_bench.py 1048576 8 1 > gpurun_out/f4_attn_rank_q8.txt 2>&1
timeout 300 python tools/packed_attn_bench.py --out gpurun_out/f4_packed_attn.json > /dev/null 2>&1
ls gpurun_out/f4_*
