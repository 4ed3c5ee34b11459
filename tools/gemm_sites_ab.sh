# A/B the GEMM tile configurations on every layer-step GEMM site (tools/gemm_sites.py).
mkdir -p gpurun_out
python tools/gemm_sites.py --check > gpurun_out/gs_default.txt 2>&1
SPT_GEMM_PAIR_MN=1 python tools/gemm_sites.py --check > gpurun_out/gs_pairmn.txt 2>&1
SPT_GEMM_PAIR_MN=1 SPT_GEMM_BN=128 python tools/gemm_sites.py --check > gpurun_out/gs_pairmn_bn128.txt 2>&1
SPT_GEMM_BN=128 python tools/gemm_sites.py > gpurun_out/gs_bn128.txt 2>&1
SPT_GEMM_1SM=1 python tools/gemm_sites.py > gpurun_out/gs_1sm.txt 2>&1
SPT_EPI_TSTORE=0 python tools/gemm_sites.py > gpurun_out/gs_notstore.txt 2>&1
tail -n 20 gpurun_out/gs_*.txt
