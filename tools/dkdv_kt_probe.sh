set -x
SPT_ATTN_DKDV_KT=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:dkdv_tc_kernel -c 1 -o gpurun_out/kt_dkdv -f python tools/attn_rank_bench.py 32768 32 8 > gpurun_out/kt_ncu.log 2>&1
SPT_ATTN_DKDV_KT=0 timeout 300 ncu --set full --clock-control none -k regex:dkdv_tc_kernel -c 1 -o gpurun_out/def_dkdv -f python tools/attn_rank_bench.py 32768 32 8 > gpurun_out/def_ncu.log 2>&1
touch paper_2506_13996_b200/csrc/attention_tc.cu
SPT_EXTRA_DEFS=SPT_EXP_NO_ELEM python paper_2506_13996_b200/build.py
timeout 300 python tools/attn_bwd_ab.py attn_dkdv_kt=0,1 --shapes 32768x32x8,131072x4x1 --rounds 3 2>&1 | tail -3
