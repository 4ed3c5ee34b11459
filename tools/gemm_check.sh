python tools/gemm_sites.py 2>&1 | tail -1
python tools/gemm_sites.py 2>&1 | tail -1
SPT_GEMM_PAIR_MN=1 python tools/gemm_sites.py 2>&1 | tail -1
