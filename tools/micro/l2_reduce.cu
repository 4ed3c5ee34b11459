// L2 reduction throughput on B200: how fast can fp32 partial sums be added into an L2-resident accumulator?
// (the budget of a single-pass attention backward whose dQ partials reach global memory as reductions).
// Variants, all 148 x k CTAs, each adding `chunk` bytes per op into a footprint of F bytes (fits L2):
//   0 bulk      cp.reduce.async.bulk.global.shared::cta.add.f32 (smem -> L2, one op per chunk)
//   1 red.v4    red.global.add.v4.f32 from registers (16 B per thread-op)
//   2 red.v8    red.global.add.v8.f32? (not on sm_100: falls back to 2x v4)
//   3 store     cp.async.bulk.global.shared::cta (plain bulk store, the write-bandwidth yardstick)
//   4 st.v4     st.global.v4.f32
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_reduce l2_reduce.cu && ./l2_reduce
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(256) kern(float* acc, int64_t foot_floats, int chunk_floats, int iters, int overlap) {
    extern __shared__ __align__(128) float sm[];
    for (int i = threadIdx.x; i < chunk_floats; i += blockDim.x) sm[i] = 1.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int64_t nchunks = foot_floats / chunk_floats;
    // overlap = how many CTAs share a target chunk at a time (contention): CTA b targets chunk (b / overlap + it * G)
    const int64_t G = gridDim.x / overlap;
    for (int it = 0; it < iters; ++it) {
        const int64_t c = ((int64_t)(blockIdx.x / overlap) + (int64_t)it * G) % nchunks;
        float* g = acc + c * chunk_floats;
        if (MODE == 0 || MODE == 3) {
            if (threadIdx.x == 0) {
                if (MODE == 0)
                    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(g),
                                 "r"(smem_u32(sm)), "r"(chunk_floats * 4) : "memory");
                else
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g),
                                 "r"(smem_u32(sm)), "r"(chunk_floats * 4) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
            }
        } else {
            for (int i = threadIdx.x * 4; i < chunk_floats; i += blockDim.x * 4) {
                float4 v = *reinterpret_cast<float4*>(sm + i);
                if (MODE == 1 || MODE == 2)
                    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(g + i), "f"(v.x), "f"(v.y), "f"(v.z),
                                 "f"(v.w) : "memory");
                else
                    asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(g + i), "f"(v.x), "f"(v.y), "f"(v.z),
                                 "f"(v.w) : "memory");
            }
        }
    }
    if ((MODE == 0 || MODE == 3) && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int MODE>
static void run(const char* name, float* acc, int64_t foot, int chunk, int ctas_per_sm, int overlap) {
    const int grid = 148 * ctas_per_sm, iters = 400;
    const int smem = chunk * 4;
    cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<MODE><<<grid, 256, smem>>>(acc, foot / 4, chunk, 20, overlap);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<MODE><<<grid, 256, smem>>>(acc, foot / 4, chunk, iters, overlap);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)grid * iters * chunk * 4;
    printf("%-8s foot %6.1f MB chunk %6d B ctas/SM %d overlap %2d: %8.1f GB/s  (%s)\n", name, foot / 1e6, chunk * 4,
           ctas_per_sm, overlap, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int64_t foot_max = 512ll << 20;
    float* acc;
    cudaMalloc(&acc, foot_max);
    cudaMemset(acc, 0, foot_max);
    for (int64_t foot : {16ll << 20, 64ll << 20, 512ll << 20}) {
        for (int chunk : {4096, 8192}) {  // floats: 16 KiB, 32 KiB
            for (int cps : {1, 2}) {
                run<0>("bulk", acc, foot, chunk, cps, 1);
                run<1>("red.v4", acc, foot, chunk, cps, 1);
                run<3>("bstore", acc, foot, chunk, cps, 1);
                run<4>("st.v4", acc, foot, chunk, cps, 1);
            }
        }
    }
    // contention: several CTAs adding into the same chunk at once (a q block's dQ from several key blocks)
    for (int ov : {2, 4, 8}) {
        run<0>("bulk", acc, 64ll << 20, 8192, 1, ov);
        run<1>("red.v4", acc, 64ll << 20, 8192, 1, ov);
    }
    return 0;
}
