// Token embedding (SURVEY.md §8(f) f4; SPEC.md:205 "embedding", :223-227 forward(model, input_ids, ...)
// with "token id >= V -> validation error").
//
//   forward : x[t, :] = E[ids[t], :]                       (bf16 rows, 16-byte accesses)
//   backward: dE[v, :] (+)= sum over t with ids[t] == v of dx[t, :], summed in ascending t (fp32)
//
// The backward is deterministic without atomics: the (id, t) pairs are sorted by id with a stable radix sort
// (CUB, from the CUDA toolkit; this is plumbing, not the measured hot path), so equal ids come out in
// ascending t, and the CTA that finds the head of a run owns that vocab row and sums the run in order.
// Rows of E that no token touches are left as they are (accumulate) or zeroed (overwrite).
#include <algorithm>
#include <cub/device/device_radix_sort.cuh>

#include "common.h"
#include "launch.h"
#include "sm100.cuh"

namespace spt {

namespace {

__global__ void embed_gather_kernel(const int64_t* __restrict__ ids, int64_t n, int64_t V, int64_t h,
                                    const bf16* __restrict__ E, bf16* __restrict__ x, int32_t* __restrict__ err) {
    const int64_t vec = h / 8;  // 16-byte chunks per row
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * vec; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / vec, c = i - t * vec;
        int64_t id = ids[t];
        if (id < 0 || id >= V) {
            if (c == 0) *err = 3;
            id = 0;  // keep the access in bounds; the step reports the error
        }
        reinterpret_cast<uint4*>(x + t * h)[c] = reinterpret_cast<const uint4*>(E + id * h)[c];
    }
}

__global__ void embed_keys_kernel(const int64_t* __restrict__ ids, int64_t n, int64_t V, int32_t* __restrict__ keys,
                                  int32_t* __restrict__ vals, int32_t* __restrict__ err) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t id = ids[t];
        if (id < 0 || id >= V) {
            *err = 3;
            id = 0;
        }
        keys[t] = (int32_t)id;
        vals[t] = (int32_t)t;
    }
}

// One CTA per run head (grid-stride over sorted positions): sums the run's dx rows in sorted (= ascending t)
// order into fp32 and writes / adds the vocab row once.
__global__ void __launch_bounds__(256) embed_segsum_kernel(const int32_t* __restrict__ skeys,
                                                            const int32_t* __restrict__ svals, int64_t n, int64_t h,
                                                            const bf16* __restrict__ dx, float* __restrict__ dE,
                                                            int accumulate) {
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const int32_t v = skeys[i];
        if (i > 0 && skeys[i - 1] == v) continue;  // not a run head
        int64_t end = i + 1;
        while (end < n && skeys[end] == v) ++end;
        float* row = dE + (int64_t)v * h;
        for (int64_t c = threadIdx.x * 8; c < h; c += 256 * 8) {
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            for (int64_t j = i; j < end; ++j) {
                const uint4 u = *reinterpret_cast<const uint4*>(dx + (int64_t)svals[j] * h + c);
                const bf16* b = reinterpret_cast<const bf16*>(&u);
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[e] += __bfloat162float(b[e]);
            }
            float4* r4 = reinterpret_cast<float4*>(row + c);
            float4 a = make_float4(acc[0], acc[1], acc[2], acc[3]), b = make_float4(acc[4], acc[5], acc[6], acc[7]);
            if (accumulate) {
                const float4 o0 = r4[0], o1 = r4[1];
                a.x += o0.x; a.y += o0.y; a.z += o0.z; a.w += o0.w;
                b.x += o1.x; b.y += o1.y; b.z += o1.z; b.w += o1.w;
            }
            r4[0] = a;
            r4[1] = b;
        }
    }
}

int sort_bits(int64_t V) {
    int b = 1;
    while ((int64_t(1) << b) < V) ++b;
    return b;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t cub_temp_bytes(int64_t n, int64_t V) {
    size_t bytes = 0;
    SPT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                             (const int32_t*)nullptr, (int32_t*)nullptr, (int)n, 0, sort_bits(V)));
    return bytes;
}

int grid_stride_blocks(int64_t work, int threads) {
    const int64_t b = (work + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

}  // namespace

size_t embed_bwd_workspace(int64_t n, int64_t V) {
    return 4 * align256((size_t)n * 4) + align256(cub_temp_bytes(n, V));
}

void embed_fwd(const int64_t* ids, int64_t n, int64_t V, int64_t h, const void* E, void* x, int32_t* err,
               cudaStream_t st) {
    SPT_CHECK(h % 8 == 0, SPT_ERR_SHAPE, "embedding: hidden size must be a multiple of 8");
    SPT_CHECK(n < (int64_t(1) << 31) && V < (int64_t(1) << 31), SPT_ERR_SHAPE, "embedding: n and V must be < 2^31");
    if (n == 0) return;
    embed_gather_kernel<<<grid_stride_blocks(n * (h / 8), 256), 256, 0, st>>>(ids, n, V, h, (const bf16*)E, (bf16*)x,
                                                                             err);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

void embed_bwd(const int64_t* ids, int64_t n, int64_t V, int64_t h, const void* dx, float* dE, bool accumulate,
               int32_t* err, void* ws, cudaStream_t st) {
    SPT_CHECK(h % 8 == 0, SPT_ERR_SHAPE, "embedding: hidden size must be a multiple of 8");
    SPT_CHECK(n < (int64_t(1) << 31) && V < (int64_t(1) << 31), SPT_ERR_SHAPE, "embedding: n and V must be < 2^31");
    if (!accumulate) SPT_CUDA(cudaMemsetAsync(dE, 0, (size_t)V * h * 4, st));
    if (n == 0) return;
    uint8_t* p = (uint8_t*)ws;
    int32_t* keys = (int32_t*)p;
    p += align256((size_t)n * 4);
    int32_t* vals = (int32_t*)p;
    p += align256((size_t)n * 4);
    int32_t* skeys = (int32_t*)p;
    p += align256((size_t)n * 4);
    int32_t* svals = (int32_t*)p;
    p += align256((size_t)n * 4);
    size_t temp = cub_temp_bytes(n, V);
    embed_keys_kernel<<<grid_stride_blocks(n, 256), 256, 0, st>>>(ids, n, V, keys, vals, err);
    count_launch();
    SPT_CUDA(cudaGetLastError());
    SPT_CUDA(cub::DeviceRadixSort::SortPairs(p, temp, keys, skeys, vals, svals, (int)n, 0, sort_bits(V), st));
    embed_segsum_kernel<<<(int)std::min<int64_t>(n, 148 * 8), 256, 0, st>>>(skeys, svals, n, h, (const bf16*)dx, dE,
                                                                           1);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

}  // namespace spt

using namespace spt;

extern "C" {
size_t spt_embed_bwd_workspace(int64_t n, int64_t vocab) {
    try {
        return embed_bwd_workspace(n, vocab);
    } catch (...) {
        return 0;
    }
}
spt_status spt_embed_fwd(const int64_t* input_ids, int64_t n, int64_t vocab, int64_t h, const void* table, void* x,
                         int32_t* err_flag, void* stream) {
    return capi_guard([&] { embed_fwd(input_ids, n, vocab, h, table, x, err_flag, (cudaStream_t)stream); });
}
spt_status spt_embed_bwd(const int64_t* input_ids, int64_t n, int64_t vocab, int64_t h, const void* dx, float* dtable,
                         int32_t accumulate, int32_t* err_flag, void* workspace, void* stream) {
    return capi_guard([&] {
        embed_bwd(input_ids, n, vocab, h, dx, dtable, accumulate != 0, err_flag, workspace, (cudaStream_t)stream);
    });
}
}
