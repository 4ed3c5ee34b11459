mkdir -p gpurun_out
timeout 900 python tools/attn_fwd_ab.py 1,13,16 32768:32:8 32768:4:1 65536:8:2 131072:4:1 131072:32:8 524288:4:1 --rounds 5 > gpurun_out/c5_fwd_ab.txt 2>&1; grep -v " O rel" gpurun_out/c5_fwd_ab.txt
