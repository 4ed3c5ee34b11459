set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python tools/prof_step.py --steps 1 --warmup 1 > gpurun_out/launch_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fwd_tc_kernel -c 1 -o gpurun_out/attn_fwd_tc python tools/prof_step.py --steps 1 --warmup 0 > gpurun_out/p1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dkdv_tc_kernel -c 1 -o gpurun_out/attn_dkdv_tc python tools/prof_step.py --steps 1 --warmup 0 > gpurun_out/p2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dq_tc_kernel -c 1 -o gpurun_out/attn_dq_tc python tools/prof_step.py --steps 1 --warmup 0 > gpurun_out/p3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 12 -c 3 -o gpurun_out/gemm_b python tools/prof_step.py --steps 1 --warmup 0 > gpurun_out/p4.log 2>&1
ls -la gpurun_out
