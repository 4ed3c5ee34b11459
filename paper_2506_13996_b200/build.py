"""Build libsptrain_b200.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed)."""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")

LIB = os.path.join(HERE, "libsptrain_b200.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = (["-DSPT_WATCHDOG"] if os.environ.get("SPT_WATCHDOG") else []) + \
        [f"-D{x}" for x in os.environ.get("SPT_EXTRA_DEFS", "").split(",") if x] + ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include"), "-I/usr/include"]
SOURCES = ["util.cpp", "plan.cpp", "memest.cpp", "comm.cpp", "peer.cu", "ulysses.cpp", "gemm.cu", "kernels.cu",
           "attention.cu", "attention_tc.cu", "tiled.cu", "embed.cu", "engine.cu"]
# Objects live in a directory keyed by the compile flags, so a build with different -D switches (the A/B
# scripts' SPT_EXTRA_DEFS, SPT_WATCHDOG) never reuses objects of another configuration.
FLAG_KEY = hashlib.sha1(" ".join(ARCH + FLAGS).encode()).hexdigest()[:10]
OBJ = os.path.join(HERE, "_build", FLAG_KEY)
DEPS_HDR = [f for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))] + ["../../include/sptrain_b200.h"]


def _newest_header() -> float:
    return max(os.path.getmtime(os.path.join(CSRC, f)) for f in DEPS_HDR)


def _compile(src: str, verbose: bool) -> str:
    out = os.path.join(OBJ, src + ".o")
    s = os.path.join(CSRC, src)
    if os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(s), _newest_header()):
        return out
    cmd = [NVCC, *ARCH, *FLAGS, "-c", s, "-o", out]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr)
    return out


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    stamp = LIB + ".flags"
    same_flags = os.path.exists(stamp) and open(stamp).read() == FLAG_KEY
    if not same_flags or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        with open(stamp, "w") as f:
            f.write(FLAG_KEY)
    return LIB




# ---------------------------------------------------------------------------------------------------------
# The reference-API drop-in (include/sptrain/gpu.hpp): sptrain::gpu ops and the autograd.hpp definitions,
# compiled against the reference's own headers and linked with the reference's own tensor.cpp / ledger.cpp,
# both compiled in place from /root/reference (never copied into this repo).  Built here, where the reference
# exists; the outputs in _ext/ travel to the GPU box with the snapshot (git-ignored, not gpurun-ignored).
REF = "/root/reference/proj"
EXT = os.path.join(HERE, "_ext")
EXT_LIB = os.path.join(EXT, "libsptrain_ext.so")
EXT_TEST = os.path.join(EXT, "tensor_ext_test")
CUDA = "/usr/local/cuda"


def build_ext() -> str | None:
    """Build _ext/libsptrain_ext.so and the C++ test program; None when the reference is not present."""
    if not os.path.isdir(os.path.join(REF, "include", "sptrain")):
        return None
    os.makedirs(EXT, exist_ok=True)
    srcs = [os.path.join(REF, "src", "tensor.cpp"), os.path.join(REF, "src", "ledger.cpp"),
            os.path.join(HERE, "sptrain_ext", "autograd.cpp"), os.path.join(HERE, "sptrain_ext", "gpu_ops.cpp")]
    hdrs = [os.path.join(ROOT, "include", "sptrain", "gpu.hpp"), os.path.join(ROOT, "include", "sptrain_b200.h")]
    inc = ["-I", os.path.join(REF, "include"), "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include")]
    link = ["-L", HERE, "-lsptrain_b200", f"-Wl,-rpath,{HERE}", "-L", os.path.join(CUDA, "lib64"), "-lcudart",
            f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}", "-lpthread"]

    def stale(out, deps):
        return not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(d) for d in deps)

    if stale(EXT_LIB, srcs + hdrs + [LIB]):
        cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", *inc, *srcs, "-o", EXT_LIB, *link]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"libsptrain_ext build failed:\n{r.stderr}")
    test_src = os.path.join(ROOT, "tests", "cpp", "tensor_ext_test.cpp")
    if stale(EXT_TEST, [test_src, EXT_LIB] + hdrs):
        cmd = ["g++", "-std=c++20", "-O2", *inc, test_src, "-o", EXT_TEST, "-L", EXT, "-lsptrain_ext",
               f"-Wl,-rpath,{EXT}", *link]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"tensor_ext_test build failed:\n{r.stderr}")
    return EXT_LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
    print(build_ext())
