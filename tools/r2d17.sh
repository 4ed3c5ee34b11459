python tools/step_ab.py gemm_pair_colgroup=0,4,8,16 --rounds 3 --group 12 > gpurun_out/r2d17_a.txt 2>&1; tail -1 gpurun_out/r2d17_a.txt
python tools/step_ab.py gemm_group_m=0,8,32 --rounds 3 --group 12 > gpurun_out/r2d17_b.txt 2>&1; tail -1 gpurun_out/r2d17_b.txt
