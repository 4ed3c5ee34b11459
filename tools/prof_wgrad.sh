mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -c 1 -o gpurun_out/wgrad_mlp python tools/gemm_sites.py mlp_dWgu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -c 1 -o gpurun_out/dgrad_mlp python tools/gemm_sites.py mlp_dx_gu > /dev/null 2>&1
ls gpurun_out/wgrad_mlp.ncu-rep gpurun_out/dgrad_mlp.ncu-rep
