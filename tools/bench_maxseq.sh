mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r1f.json 2> gpurun_out/bench_r1f.err; tail -c 600 gpurun_out/bench_r1f.json
timeout 1500 python tools/max_seq.py --n 786432,1048576,1310720 --out gpurun_out/max_seq_big.json > gpurun_out/max_seq_big.log 2>&1; cat gpurun_out/max_seq_big.log
