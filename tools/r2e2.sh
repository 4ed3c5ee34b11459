run() { timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 2 -c 1 --csv python tools/gemm_one.py "$@" --reps 1 2>/dev/null | grep -E "dram__|duration|cycles" | awk -F'","' -v a="$*" '{printf "%s | %s %s\n", a, $(NF-2), $(NF)}'; }
for g in 4 8 16 32; do run 16384 28672 4096 0 0 --group $g; done
for g in 4 8 16 32; do run 16384 28672 4096 0 0 --raster 19 --group $g; done
for g in 8 16 32; do run 16384 4096 14336 0 0 --group $g; done
for g in 4 8 16; do run 16384 4096 14336 0 0 --raster 19 --group $g; done
