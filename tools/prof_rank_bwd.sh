# ncu of the attention backward kernels at the L8 rank shape (s=524288, 4q/1kv): dK/dV (K in TMEM) and dQ.
mkdir -p gpurun_out
for k in dkdv dq_tmem fwd_tc; do
timeout 900 ncu --set full --clock-control none -k regex:$k -c 1 -o gpurun_out/rank_$k -f python tools/attn_rank_bench.py 524288 4 1 > /dev/null 2>&1
done
ls gpurun_out/rank_*
