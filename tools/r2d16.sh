python tools/step_ab.py gemm_colgroup=0,8,16,1008 --rounds 3 --group 12 > gpurun_out/r2d16_a.txt 2>&1; tail -1 gpurun_out/r2d16_a.txt
python tools/step_ab.py gemm_colgroup=8,0,2,1016 --rounds 3 --group 12 > gpurun_out/r2d16_b.txt 2>&1; tail -1 gpurun_out/r2d16_b.txt
