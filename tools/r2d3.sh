# forward exp split A/B after the register fix: standalone shapes + sustained L1 step
mkdir -p gpurun_out
timeout 900 python tools/attn_fwd_ab.py 1,12,13,14 32768:32:8 131072:4:1 524288:4:1 65536:8:2 --rounds 4 > gpurun_out/r2d3_fwd_ab.txt 2>&1; grep ": v=1 " gpurun_out/r2d3_fwd_ab.txt
timeout 900 python tools/step_ab.py attn_fwd_bk128=1,13 --rounds 3 --group 12 > gpurun_out/r2d3_step_ab.txt 2>&1; tail -3 gpurun_out/r2d3_step_ab.txt
