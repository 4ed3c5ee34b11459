mkdir -p gpurun_out
timeout 900 python tools/attn_fwd_ab.py 1,12,13,14,16,18 32768:32:8 131072:4:1 524288:4:1 --rounds 3 > gpurun_out/c4_fwd_ab.txt 2>&1; cat gpurun_out/c4_fwd_ab.txt
