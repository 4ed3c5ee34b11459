# L2 policy A/B on the lm_head / TiledMLP weight-gradient GEMMs: timing and ncu DRAM bytes per raster mode
mkdir -p gpurun_out
for r in 0 4 8 12; do for i in 1 2; do python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --raster $r --reps 10; done; done
for r in 0 4 8 12; do timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 2 -c 1 --csv python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --raster $r --reps 1 2>/dev/null | grep -E "dram__|duration|cycles_elapsed" | awk -F'","' -v r=$r '{print "raster " r ": " $(NF-2) " " $(NF)}'; done
timeout 1200 python tools/step_ab.py gemm_raster=0,4,8,12 --rounds 3 --group 12 2>&1 | tail -2
