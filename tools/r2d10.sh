# early-exponential forward: correctness/bitwise tests, standalone A/B, sustained step A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention_fwd" > gpurun_out/r2d10_pytest.txt 2>&1; tail -2 gpurun_out/r2d10_pytest.txt
timeout 900 python tools/attn_fwd_ab.py 13,23,11,21 32768:32:8 131072:4:1 524288:4:1 65536:8:2 --rounds 4 > gpurun_out/r2d10_fwd_ab.txt 2>&1; grep -v "O rel" gpurun_out/r2d10_fwd_ab.txt; grep "v=23\|v=21" gpurun_out/r2d10_fwd_ab.txt | grep "O rel" | head -4
timeout 900 python tools/step_ab.py attn_fwd_bk128=13,23 --rounds 3 --group 12 2>&1 | tail -1
