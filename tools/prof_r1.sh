set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python tools/prof_step.py --steps 1 --warmup 1 > gpurun_out/launch_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bwd_dkdv -c 1 -o gpurun_out/attn_dkdv python tools/prof_step.py --steps 1 --warmup 0 > gpurun_out/p1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 20 -c 2 -o gpurun_out/gemm python tools/prof_step.py --steps 1 --warmup 0 > gpurun_out/p2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -c 1 -o gpurun_out/attn_fwd python tools/prof_step.py --steps 1 --warmup 0 > gpurun_out/p3.log 2>&1
ls -la gpurun_out
