for i in 1 2; do python tools/gemm_one.py 128256 4096 8192 1 1 --f32; python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --pair; python tools/gemm_one.py 32768 4096 6144 0 1; python tools/gemm_one.py 32768 4096 6144 0 1 --pair; done
timeout 1500 python tools/step_ab.py gemm_pair_mn=0,3,4 --rounds 3 --group 12 2>&1 | tail -1
