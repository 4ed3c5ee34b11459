# Round-2 refresh of the widened rows on the final code: multi-layer stack with device / offloaded
# checkpoints, RoPE, packed-sequence attention.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --layers 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_bench_L4_device_ckpt.json 2>/dev/null; tail -c 200 gpurun_out/r2g_bench_L4_device_ckpt.json
timeout 900 python bench.py --layers 4 --offload --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_bench_L4_offload.json 2>/dev/null; tail -c 200 gpurun_out/r2g_bench_L4_offload.json
timeout 600 python bench.py --rope 500000 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_bench_L1_rope.json 2>/dev/null; tail -c 200 gpurun_out/r2g_bench_L1_rope.json
SPT_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --seq 16384 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_bench_sp2_same_gpu.json 2>gpurun_out/r2g_bench_sp2_same_gpu.err; tail -c 300 gpurun_out/r2g_bench_sp2_same_gpu.json
timeout 900 python tools/packed_attn_bench.py > gpurun_out/r2g_packed_attn.txt 2>&1; tail -5 gpurun_out/r2g_packed_attn.txt
ls gpurun_out/r2g_*
