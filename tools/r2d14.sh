timeout 1500 python tools/step_ab.py gemm_group_m=0,16,-1 --rounds 3 --group 12 2>&1 | tail -1
timeout 900 python tools/step_ab.py gemm_group_m=0,16,-1 --rounds 3 --group 12 2>&1 | tail -1
