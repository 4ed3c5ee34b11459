mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multilayer.py tests/test_cpp_api.py -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --layers 4 > gpurun_out/bench_l4.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/bench_l4.json').read().splitlines()[-1]);print('L4 dev', d['value'], d['ms_per_step'], d['peak_hbm_bytes'])"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --layers 4 --offload > gpurun_out/bench_l4o.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/bench_l4o.json').read().splitlines()[-1]);print('L4 offload', d['value'], d['ms_per_step'], d['peak_hbm_bytes'])"
