# FLCE A/B on the L1 bench step (separate processes: SPT_FLCE_EXP is read at load), interleaved twice.
mkdir -p gpurun_out
for r in 1 2; do
  for cfg in "0 8192" "1 8192" "1 16384"; do
    set -- $cfg
    SPT_FLCE_EXP=$1 timeout 400 python bench.py --steps 12 --warmup 3 --no-cpu-baseline --loss-tile $2 2>/dev/null | tail -1 > gpurun_out/flce_ab_$1_$2_$r.json
    python3 -c "import json,sys; d=json.load(open('gpurun_out/flce_ab_$1_$2_$r.json')); print('exp=$1 tile=$2 round $r', round(d['ms_per_step'],2), 'ms', d['breakdown_ms_per_step'], d['peak_hbm_bytes'], d['clocks']['sm_mhz'])"
  done
done
