mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dkdv -c 1 -o gpurun_out/attn_dkdv python tools/attn_bench.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dq_tc -c 1 -o gpurun_out/attn_dq python tools/attn_bench.py > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
