# Refresh after the GEMM tile-order change (r2e): launch list with DRAM bytes (-> profiles/traffic.json), ncu --set full
# of the two lm_head backward GEMMs in the step, the L8 emulation, the Qwen shape.
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2e_launches.csv python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc_kernel<256, 1, 1, 1>" -s 10 -c 1 -o gpurun_out/r2e_gemm_dw -f python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc_kernel<256, 0, 1, 0>" -s 10 -c 1 -o gpurun_out/r2e_gemm_dx -f python tools/prof_step.py --steps 1 --warmup 1 > /dev/null 2>&1
timeout 1200 python tools/l8_emulation.py --out gpurun_out/r2e_l8_emulation.json > gpurun_out/r2e_l8_emulation.log 2>&1; tail -2 gpurun_out/r2e_l8_emulation.log
timeout 600 python tools/shape_bench.py > gpurun_out/r2e_qwen_shape_32k.json 2>&1; tail -c 300 gpurun_out/r2e_qwen_shape_32k.json
ls gpurun_out/r2e_*
