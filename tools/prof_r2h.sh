# compute-sanitizer memcheck / racecheck on the final code (12-warp forward, RMSNorm prefetch, GEMM tile orders)
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/r2h_memcheck.txt 2>&1; tail -3 gpurun_out/r2h_memcheck.txt
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_cases.py > gpurun_out/r2h_racecheck.txt 2>&1; tail -3 gpurun_out/r2h_racecheck.txt
