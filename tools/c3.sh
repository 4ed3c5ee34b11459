set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_tc128 -c 1 -o gpurun_out/c3_fwd128 python tools/attn_rank_bench.py 131072 4 1 > gpurun_out/c3_ncu.log 2>&1; tail -3 gpurun_out/c3_ncu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dkdv_tc -c 1 -o gpurun_out/c3_dkdv python tools/attn_rank_bench.py 131072 4 1 > gpurun_out/c3_ncu2.log 2>&1; tail -3 gpurun_out/c3_ncu2.log
ls -la gpurun_out
