// Device side of the peer-memory transport (comm.h, peer mode): the cross-rank barrier and the fixed-order
// all-reduce / all-gather / all-to-all over buffers mapped from the other ranks (NVLink / NVSwitch loads and
// stores; CUDA IPC mappings between processes, plain pointers between threads of one process).
//
// Barrier protocol.  Rank r keeps a device counter `epoch` of barriers entered.  Entering barrier e, one
// thread per peer p stores e into peer p's flags[r] with st.release.sys (after a system-scope fence that
// orders every write this rank's stream made before the barrier, including remote stores of the fused K1),
// then spins with ld.acquire.sys on its own flags[p] until it reads >= e.  Flags only grow and no rank can
// run more than one barrier ahead of another, so ">= e" is exact.  A wait longer than timeout_ns (read from
// %globaltimer) sets the group's error flag (pinned host memory, visible to the host without a sync) and
// leaves the barrier, so a dead or diverged peer turns into ProtocolError rather than a hang.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.h"
#include "launch.h"

namespace spt {

struct PeerBufs {
    void* p[kMaxSP];
};

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void peer_barrier_kernel(PeerBufs flags, int rank, int P, uint64_t* epoch, int64_t timeout_ns,
                                    int32_t* err) {
    __shared__ uint64_t e;
    if (threadIdx.x == 0) {
        e = *epoch + 1;
        *epoch = e;
        __threadfence_system();
    }
    __syncthreads();
    const int p = threadIdx.x;
    if (p >= P || p == rank) return;
    st_release_sys(static_cast<uint64_t*>(flags.p[p]) + rank, e);  // "rank arrived at e", in peer p's flags
    const uint64_t* mine = static_cast<const uint64_t*>(flags.p[rank]) + p;
    const uint64_t t0 = global_ns();
    uint32_t spins = 0;
    while (ld_acquire_sys(mine) < e) {
        if ((++spins & 1023) == 0) {
            if ((int64_t)(global_ns() - t0) > timeout_ns) {
                *(volatile int32_t*)err = 1;
                __threadfence_system();
                break;
            }
            __nanosleep(256);
        }
    }
}

void peer_barrier(void* const* flag_bufs, int rank, int P, uint64_t* epoch, int64_t timeout_ns, int32_t* err,
                  cudaStream_t st) {
    PeerBufs f{};
    for (int i = 0; i < P; ++i) f.p[i] = flag_bufs[i];
    peer_barrier_kernel<<<1, 64, 0, st>>>(f, rank, P, epoch, timeout_ns, err);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

// ---- reduce-scatter (rank r owns chunk r) then all-gather, summing every element over ranks 0..P-1 in
// ascending order.  Elements are processed 16 bytes at a time; chunk bounds are multiples of
// 64 elements so every chunk but the last is 16-byte aligned.
template <class T>
struct Vec16 {
    static constexpr int N = 16 / sizeof(T);
    T v[N];
};

template <class T>
__global__ void __launch_bounds__(256) peer_reduce_chunk_kernel(PeerBufs bufs, int P, int rank, int64_t lo,
                                                                int64_t hi) {
    using V = Vec16<T>;
    constexpr int NV = V::N;
    const int64_t n = hi - lo;
    const int64_t nvec = n / NV;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    T* out = static_cast<T*>(bufs.p[rank]) + lo;
    for (int64_t i = tid; i < nvec; i += nth) {
        V acc = reinterpret_cast<const V*>(static_cast<const T*>(bufs.p[0]) + lo)[i];
        for (int q = 1; q < P; ++q) {
            const V x = reinterpret_cast<const V*>(static_cast<const T*>(bufs.p[q]) + lo)[i];
#pragma unroll
            for (int k = 0; k < NV; ++k) acc.v[k] += x.v[k];
        }
        reinterpret_cast<V*>(out)[i] = acc;
    }
    for (int64_t i = nvec * NV + tid; i < n; i += nth) {  // tail
        T acc = static_cast<const T*>(bufs.p[0])[lo + i];
        for (int q = 1; q < P; ++q) acc += static_cast<const T*>(bufs.p[q])[lo + i];
        out[i] = acc;
    }
}

// dst[lo_q, hi_q) = rank q's copy for every q != rank (bytes; 16-byte granules where aligned)
__global__ void __launch_bounds__(256) peer_gather_chunks_kernel(PeerBufs bufs, int P, int rank, int64_t chunk_bytes,
                                                                 int64_t total_bytes) {
    char* dst = static_cast<char*>(bufs.p[rank]);
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int q = 0; q < P; ++q) {
        if (q == rank) continue;
        const int64_t lo = q * chunk_bytes;
        if (lo >= total_bytes) break;
        const int64_t n = min(chunk_bytes, total_bytes - lo);
        const char* src = static_cast<const char*>(bufs.p[q]);
        const int64_t nv = n / 16;
        for (int64_t i = tid; i < nv; i += nth)
            reinterpret_cast<uint4*>(dst + lo)[i] = reinterpret_cast<const uint4*>(src + lo)[i];
        for (int64_t i = nv * 16 + tid; i < n; i += nth) dst[lo + i] = src[lo + i];
    }
}

static int peer_grid(int64_t work16) {
    const int64_t b = (work16 + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms() * 4));
}

// one rank's part of an all-reduce: reduce its chunk, (barrier), gather the others' chunks.  The caller
// brackets the two kernels with barriers.
int64_t peer_chunk_elems(int64_t count, int P) { return ((count + P - 1) / P + 63) / 64 * 64; }

void peer_reduce_chunk(void* const* bufs, int P, int rank, int64_t count, int elem_kind, cudaStream_t st) {
    PeerBufs b{};
    for (int i = 0; i < P; ++i) b.p[i] = bufs[i];
    const int64_t ce = peer_chunk_elems(count, P);
    const int64_t lo = std::min<int64_t>(count, rank * ce), hi = std::min<int64_t>(count, lo + ce);
    if (hi <= lo) return;
    switch (elem_kind) {
        case 0:
            peer_reduce_chunk_kernel<float><<<peer_grid((hi - lo) / 4), 256, 0, st>>>(b, P, rank, lo, hi);
            break;
        case 1:
            peer_reduce_chunk_kernel<double><<<peer_grid((hi - lo) / 2), 256, 0, st>>>(b, P, rank, lo, hi);
            break;
        case 2:
            peer_reduce_chunk_kernel<int64_t><<<peer_grid((hi - lo) / 2), 256, 0, st>>>(b, P, rank, lo, hi);
            break;
        default:
            SPT_THROW(SPT_ERR_INTERNAL, "peer_reduce_chunk: bad element kind");
    }
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

void peer_gather_chunks(void* const* bufs, int P, int rank, int64_t chunk_bytes, int64_t total_bytes,
                        cudaStream_t st) {
    PeerBufs b{};
    for (int i = 0; i < P; ++i) b.p[i] = bufs[i];
    peer_gather_chunks_kernel<<<peer_grid(total_bytes / 16), 256, 0, st>>>(b, P, rank, chunk_bytes, total_bytes);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

// pull copy: dst[q * bytes .. (q+1) * bytes) = src_q[src_off .. src_off + bytes) for every rank q (all-gather
// with src_off = 0; all-to-all with src_off = rank * bytes)
__global__ void __launch_bounds__(256) peer_pull_kernel(PeerBufs src, int P, int64_t src_off, int64_t bytes,
                                                        char* dst) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int q = 0; q < P; ++q) {
        const char* s = static_cast<const char*>(src.p[q]) + src_off;
        char* d = dst + q * bytes;
        const bool al = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0;
        const int64_t nv = al ? bytes / 16 : 0;
        for (int64_t i = tid; i < nv; i += nth) reinterpret_cast<uint4*>(d)[i] = reinterpret_cast<const uint4*>(s)[i];
        for (int64_t i = nv * 16 + tid; i < bytes; i += nth) d[i] = s[i];
    }
}

void peer_pull(void* const* src, int P, int64_t src_off, int64_t bytes, void* dst, cudaStream_t st) {
    PeerBufs b{};
    for (int i = 0; i < P; ++i) b.p[i] = src[i];
    peer_pull_kernel<<<peer_grid(bytes * P / 16), 256, 0, st>>>(b, P, src_off, bytes, (char*)dst);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

}  // namespace spt
