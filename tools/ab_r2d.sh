# Round-2 (r2d) A/B and check invocations, in the order they ran under gpurun (each was its own call; the
# profiles/r2d_*.txt files cite them as r2dN).  Kept as one record instead of twenty one-off scripts; run any
# block by hand.  Outputs went to gpurun_out/ (scratch); the summaries are in profiles/.
# Switches that measured worse were removed from the library afterwards, so those blocks no longer run as-is:
# gemm_raster hint bits 4 / 8 (r2d6), gemm_one --persist / gemm_l2_persist (r2d8), attn_fwd_bk128 21 / 23 and
# tools/fwd_det_check.py (r2d10-11), gemm_pair_mn 3 / 4 (r2d12), gemm_pair_colgroup (r2d17).

# ---- r2d1
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r2d_gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_pytest_gpu.txt 2>&1; tail -3 gpurun_out/r2d_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.txt 2>&1; tail -2 gpurun_out/r2d_smoke.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2d_bench_L1.json 2> gpurun_out/r2d_bench_L1.err; tail -c 400 gpurun_out/r2d_bench_L1.json

# ---- r2d2
# fwd_tc128 on 12 warps with setmaxnreg (no spills) + rmsnorm prefetch: tests + forward A/B + FA4 yardstick
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention or rmsnorm" > gpurun_out/r2d2_pytest.txt 2>&1; tail -2 gpurun_out/r2d2_pytest.txt
timeout 600 python tools/attn_fwd_ab.py 1,13,16,18 32768:32:8 524288:4:1 --rounds 4 > gpurun_out/r2d2_fwd_ab.txt 2>&1; tail -2 gpurun_out/r2d2_fwd_ab.txt
timeout 600 python tools/attn_fa4_bench.py 32768:32:8 > gpurun_out/r2d2_fa4.txt 2>&1; tail -1 gpurun_out/r2d2_fa4.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2d2_bench.json 2>gpurun_out/r2d2_bench.err; python -c "
import json;d=json.load(open('gpurun_out/r2d2_bench.json'));print(d['value'],d['ms_per_step'],d['breakdown_ms_per_step'],d['clocks'])"

# ---- r2d3
# forward exp split A/B after the register fix: standalone shapes + sustained L1 step
timeout 900 python tools/attn_fwd_ab.py 1,12,13,14 32768:32:8 131072:4:1 524288:4:1 65536:8:2 --rounds 4 > gpurun_out/r2d3_fwd_ab.txt 2>&1; grep ": v=1 " gpurun_out/r2d3_fwd_ab.txt
timeout 900 python tools/step_ab.py attn_fwd_bk128=1,13 --rounds 3 --group 12 > gpurun_out/r2d3_step_ab.txt 2>&1; tail -3 gpurun_out/r2d3_step_ab.txt

# ---- r2d4
# checkpoint after the forward register split: full GPU suite, smoke, bench (both arms)
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2d4_pytest_gpu.txt 2>&1; tail -3 gpurun_out/r2d4_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d4_smoke.txt 2>&1; tail -1 gpurun_out/r2d4_smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d4_bench_L1.json 2> gpurun_out/r2d4_bench_L1.err; tail -c 300 gpurun_out/r2d4_bench_L1.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2d4_bench_ref.json 2> gpurun_out/r2d4_bench_ref.err; tail -c 600 gpurun_out/r2d4_bench_ref.json

# ---- r2d5
# loss tile A/B at L1 (8192 = current rule, 16384 = the same 4 GiB budget counted at the exp form's 2 bytes/logit)
for r in 1 2; do for t in 8192 16384; do
timeout 600 python bench.py --steps 12 --warmup 3 --no-cpu-baseline --loss-tile $t > gpurun_out/r2d5_lt${t}_$r.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/r2d5_lt${t}_$r.json'));print('tile $t run $r', round(d['value']), round(d['ms_per_step'],2), d['peak_hbm_bytes'], d['breakdown_ms_per_step'], d['clocks']['sm_mhz'])"
done; done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2d5_bench_ref.json 2>/dev/null; tail -c 250 gpurun_out/r2d5_bench_ref.json

# ---- r2d6
# L2 policy A/B on the lm_head / TiledMLP weight-gradient GEMMs: timing and ncu DRAM bytes per raster mode
for r in 0 4 8 12; do for i in 1 2; do python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --raster $r --reps 10; done; done
for r in 0 4 8 12; do timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 2 -c 1 --csv python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --raster $r --reps 1 2>/dev/null | grep -E "dram__|duration|cycles_elapsed" | awk -F'","' -v r=$r '{print "raster " r ": " $(NF-2) " " $(NF)}'; done
timeout 1200 python tools/step_ab.py gemm_raster=0,4,8,12 --rounds 3 --group 12 2>&1 | tail -2

# ---- r2d7
for r in 0 1; do for i in 1 2; do python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --raster $r --reps 10; done; done
for r in 0 1; do timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 2 -c 1 --csv python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --raster $r --reps 1 2>/dev/null | grep -E "dram__|duration|cycles_elapsed" | awk -F'","' -v r=$r '{print "raster " r ": " $(NF-2) " " $(NF)}'; done

# ---- r2d8
for p in 0 80; do for i in 1 2; do python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --persist $p --reps 10; done; done
for p in 0 80; do timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 2 -c 1 --csv python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --persist $p --reps 1 2>/dev/null | grep -E "dram__|duration|cycles_elapsed" | awk -F'","' -v r=$p '{print "persist " r ": " $(NF-2) " " $(NF)}'; done
timeout 1200 python tools/step_ab.py gemm_l2_persist=0,80 --rounds 3 --group 12 2>&1 | tail -1

# ---- r2d9
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size/2**20, 'MB')
import ctypes; rt=ctypes.CDLL('libcudart.so.12') if False else None
" 2>&1
python - <<'PY'
import ctypes
cudart = None
for n in ("libcudart.so.12", "libcudart.so"):
    try:
        cudart = ctypes.CDLL(n); break
    except OSError: pass
import torch; torch.cuda.init()
v = ctypes.c_int()
if cudart is not None:
    print("persistingL2CacheMaxSize", cudart.cudaDeviceGetAttribute(ctypes.byref(v), 108, 0), v.value / 2**20, "MB")
PY
for k in 2048 4096 8192; do timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 2 -c 1 --csv python tools/gemm_one.py 128256 4096 $k 1 1 --f32 --reps 1 2>/dev/null | grep -E "dram__|duration" | awk -F'","' -v r=$k '{print "K " r ": " $(NF-2) " " $(NF)}'; done

# ---- r2d10
# early-exponential forward: correctness/bitwise tests, standalone A/B, sustained step A/B
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention_fwd" > gpurun_out/r2d10_pytest.txt 2>&1; tail -2 gpurun_out/r2d10_pytest.txt
timeout 900 python tools/attn_fwd_ab.py 13,23,11,21 32768:32:8 131072:4:1 524288:4:1 65536:8:2 --rounds 4 > gpurun_out/r2d10_fwd_ab.txt 2>&1; grep -v "O rel" gpurun_out/r2d10_fwd_ab.txt; grep "v=23\|v=21" gpurun_out/r2d10_fwd_ab.txt | grep "O rel" | head -4
timeout 900 python tools/step_ab.py attn_fwd_bk128=13,23 --rounds 3 --group 12 2>&1 | tail -1

# ---- r2d11
python tools/fwd_det_check.py 4096 8 2 2.5 11,21,13,23
timeout 900 python tools/attn_fwd_ab.py 13,11 32768:32:8 524288:4:1 --rounds 3 2>&1 | grep -v "O rel"
timeout 900 python tools/attn_fwd_ab.py 13,11 32768:32:8 524288:4:1 --rounds 3 --lib=ab_old/libsptrain_b200.so 2>&1 | grep -v "O rel"

# ---- r2d12
for i in 1 2; do python tools/gemm_one.py 128256 4096 8192 1 1 --f32; python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --pair; python tools/gemm_one.py 32768 4096 6144 0 1; python tools/gemm_one.py 32768 4096 6144 0 1 --pair; done
timeout 1500 python tools/step_ab.py gemm_pair_mn=0,3,4 --rounds 3 --group 12 2>&1 | tail -1

# ---- r2d13
# raster-0 group size vs HBM bytes and time on the lm_head GEMM shapes (logits as bf16 out, dgrad, dW)
run() { timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 2 -c 1 --csv python tools/gemm_one.py "$@" --reps 1 2>/dev/null | grep -E "dram__|duration|cycles" | awk -F'","' -v a="$*" '{printf "%s | %s %s\n", a, $(NF-2), $(NF)}'; }
for g in 4 8 16 32; do run 8192 128256 4096 0 0 --group $g; done
for g in 4 8 16 32 64; do run 8192 4096 128256 0 1 --group $g; done
for g in 4 8 16 32; do run 128256 4096 8192 1 1 --f32 --group $g; done

# ---- r2d14
timeout 1500 python tools/step_ab.py gemm_group_m=0,16,-1 --rounds 3 --group 12 2>&1 | tail -1
timeout 900 python tools/step_ab.py gemm_group_m=0,16,-1 --rounds 3 --group 12 2>&1 | tail -1

# ---- r2d15
run() { timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 2 -c 1 --csv python tools/gemm_one.py "$@" --reps 1 2>/dev/null | grep -E "dram__|duration|cycles" | awk -F'","' -v a="$*" '{printf "%s | %s %s\n", a, $(NF-2), $(NF)}'; }
run 128256 4096 8192 1 1 --f32
for g in 2 4 8; do run 128256 4096 8192 1 1 --f32 --raster 19 --group $g; done
for g in 2 4 8; do run 8192 4096 128256 0 1 --raster 19 --group $g; done
for i in 1 2; do python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --reps 10; python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --reps 10 --raster 19 --group 8; python tools/gemm_one.py 128256 4096 8192 1 1 --f32 --reps 10 --raster 19 --group 4; done

# ---- r2d16
python tools/step_ab.py gemm_colgroup=0,8,16,1008 --rounds 3 --group 12 > gpurun_out/r2d16_a.txt 2>&1; tail -1 gpurun_out/r2d16_a.txt
python tools/step_ab.py gemm_colgroup=8,0,2,1016 --rounds 3 --group 12 > gpurun_out/r2d16_b.txt 2>&1; tail -1 gpurun_out/r2d16_b.txt

# ---- r2d17
python tools/step_ab.py gemm_pair_colgroup=0,4,8,16 --rounds 3 --group 12 > gpurun_out/r2d17_a.txt 2>&1; tail -1 gpurun_out/r2d17_a.txt
python tools/step_ab.py gemm_group_m=0,8,32 --rounds 3 --group 12 > gpurun_out/r2d17_b.txt 2>&1; tail -1 gpurun_out/r2d17_b.txt

# ---- r2d18
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2d18_pytest_gpu.txt 2>&1; tail -2 gpurun_out/r2d18_pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d18_bench_L1.json 2> gpurun_out/r2d18_bench_L1.err; python -c "
import json;d=json.load(open('gpurun_out/r2d18_bench_L1.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],d['breakdown_ms_per_step'],d['clocks'])
for k,v in d['gemm_sites'].items(): print(k,v)"

# ---- r2d19
python tools/step_ab.py gemm_bn=0,2 --rounds 3 --group 12 > gpurun_out/r2d19_a.txt 2>&1; tail -1 gpurun_out/r2d19_a.txt
python tools/step_ab.py mlp_bwd_group=1,2 --rounds 3 --group 12 > gpurun_out/r2d19_b.txt 2>&1; tail -1 gpurun_out/r2d19_b.txt
python tools/step_ab.py attn_kv_group=0,1 --rounds 3 --group 12 > gpurun_out/r2d19_c.txt 2>&1; tail -1 gpurun_out/r2d19_c.txt

# ---- r2d20
python tools/config_ab.py mlp_tiles=0,1,4 --rounds 3 --group 12 > gpurun_out/r2d20_a.txt 2>&1; tail -1 gpurun_out/r2d20_a.txt
python tools/config_ab.py loss_tile=0,16384,4096 --rounds 3 --group 12 > gpurun_out/r2d20_b.txt 2>&1; tail -1 gpurun_out/r2d20_b.txt

# ---- r2e2: MLP-shaped pair GEMMs, row groups vs column groups (standalone DRAM bytes; defaults kept)
run() { timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 2 -c 1 --csv python tools/gemm_one.py "$@" --reps 1 2>/dev/null | grep -E "dram__|duration|cycles" | awk -F'","' -v a="$*" '{printf "%s | %s %s\n", a, $(NF-2), $(NF)}'; }
for g in 4 8 16 32; do run 16384 28672 4096 0 0 --group $g; done
for g in 4 8 16 32; do run 16384 28672 4096 0 0 --raster 19 --group $g; done
for g in 8 16 32; do run 16384 4096 14336 0 0 --group $g; done
for g in 4 8 16; do run 16384 4096 14336 0 0 --raster 19 --group $g; done

# ---- r2e3: forward P hand-off variants as separate builds (SPT_EXTRA_DEFS=SPT_FWD2_NPART=2 / a deferred-arrive
# form, since removed), interleaved in one process with tools/lib_ab_fwd.py: all within +-0.5% (bitwise equal)
for i in 1 2; do timeout 900 python tools/lib_ab_fwd.py paper_2506_13996_b200/libsptrain_b200.so ab_var/libsptrain_b200.so ab_var2/libsptrain_b200.so ab_var3/libsptrain_b200.so --rounds 5; done
