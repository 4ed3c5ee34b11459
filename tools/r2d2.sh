# fwd_tc128 on 12 warps with setmaxnreg (no spills) + rmsnorm prefetch: tests + forward A/B + FA4 yardstick
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention or rmsnorm" > gpurun_out/r2d2_pytest.txt 2>&1; tail -2 gpurun_out/r2d2_pytest.txt
timeout 600 python tools/attn_fwd_ab.py 1,13,16,18 32768:32:8 524288:4:1 --rounds 4 > gpurun_out/r2d2_fwd_ab.txt 2>&1; tail -2 gpurun_out/r2d2_fwd_ab.txt
timeout 600 python tools/attn_fa4_bench.py 32768:32:8 > gpurun_out/r2d2_fa4.txt 2>&1; tail -1 gpurun_out/r2d2_fa4.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2d2_bench.json 2>gpurun_out/r2d2_bench.err; python -c "
import json;d=json.load(open('gpurun_out/r2d2_bench.json'));print(d['value'],d['ms_per_step'],d['breakdown_ms_per_step'],d['clocks'])"
