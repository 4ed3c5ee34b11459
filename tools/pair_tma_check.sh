SPT_GEMM_PAIR_MN=1 timeout 600 python -m pytest tests -m gpu -q -x -k "gemm or flce or mlp or layer_step" 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -q -x -k "gemm or flce or mlp" 2>&1 | tail -1
python tools/step_ab.py gemm_pair_mn=0,1 --rounds 5 2>&1 | tail -1
python tools/step_ab.py gemm_pair_mn=0,1 --rounds 5 2>&1 | tail -1
