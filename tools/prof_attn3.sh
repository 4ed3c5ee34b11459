mkdir -p gpurun_out
for k in fwd_tc dkdv dq_tc; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/a4_$k python tools/attn_bench.py > /dev/null 2>&1
done
ls gpurun_out/a3_*
