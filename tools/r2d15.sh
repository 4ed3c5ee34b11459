run() { timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 2 -c 1 --csv python tools/gemm_one.py "$@" --reps 1 2>/dev/null | grep -E "dram__|duration|cycles" | awk -F'","' -v a="$*" '{printf "%s | %s %s\n", a, $(NF-2), $(NF)}'; }
run 128256 4096 8192 1 1 --f32
for g in 2 4 8; do run 128256 4096 8192 1 1 --f32 --raster 19 --group $g; done
for g in 2 4 8; do run 8192 4096 128256 0 1 --raster 19 --group $g; done
for i in 1 2; do python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --reps 10; python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --reps 10 --raster 19 --group 8; python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --reps 10 --raster 19 --group 4; done
