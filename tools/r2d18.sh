mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2d18_pytest_gpu.txt 2>&1; tail -2 gpurun_out/r2d18_pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d18_bench_L1.json 2> gpurun_out/r2d18_bench_L1.err; python -c "
import json;d=json.load(open('gpurun_out/r2d18_bench_L1.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],d['breakdown_ms_per_step'],d['clocks'])
for k,v in d['gemm_sites'].items(): print(k,v)"
