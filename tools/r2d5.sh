# loss tile A/B at L1 (8192 = current rule, 16384 = the same 4 GiB budget counted at the exp form's 2 bytes/logit)
mkdir -p gpurun_out
for r in 1 2; do for t in 8192 16384; do
timeout 600 python bench.py --steps 12 --warmup 3 --no-cpu-baseline --loss-tile $t > gpurun_out/r2d5_lt${t}_$r.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/r2d5_lt${t}_$r.json'));print('tile $t run $r', round(d['value']), round(d['ms_per_step'],2), d['peak_hbm_bytes'], d['breakdown_ms_per_step'], d['clocks']['sm_mhz'])"
done; done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2d5_bench_ref.json 2>/dev/null; tail -c 250 gpurun_out/r2d5_bench_ref.json
