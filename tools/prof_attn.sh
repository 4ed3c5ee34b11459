mkdir -p gpurun_out
python tools/attn_bench.py > gpurun_out/attn_bench.txt 2>&1
python tools/attn_lib_bench.py > gpurun_out/attn_lib.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_tc|dkdv|dq_tc" -c 3 -o gpurun_out/attn_full python tools/attn_bench.py > /dev/null 2>&1
cat gpurun_out/attn_bench.txt gpurun_out/attn_lib.txt
