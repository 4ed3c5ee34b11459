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
