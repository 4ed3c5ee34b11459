python tools/step_ab.py gemm_bn=0,2 --rounds 3 --group 12 > gpurun_out/r2d19_a.txt 2>&1; tail -1 gpurun_out/r2d19_a.txt
python tools/step_ab.py mlp_bwd_group=1,2 --rounds 3 --group 12 > gpurun_out/r2d19_b.txt 2>&1; tail -1 gpurun_out/r2d19_b.txt
python tools/step_ab.py attn_kv_group=0,1 --rounds 3 --group 12 > gpurun_out/r2d19_c.txt 2>&1; tail -1 gpurun_out/r2d19_c.txt
