// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1, M=128, N=256, K=16, bf16) throughput for each operand
// major, with the GEMM kernel's own SW128 descriptors (K-major: 16-byte LBO, +32 B per K step; MN-major: 64-wide
// column regions 8 KiB apart, +2 KiB per K step).  One CTA per SM, one thread issues back-to-back MMAs over a
// 4-step K block (like one GEMM stage), one commit at the end.  Are MN-major operands slower in the MMA itself?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2506_13996_b200/csrc tools/micro/mma_major_rate.cu
#include <cstdio>
#include "sm100.cuh"
using namespace spt;

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) { tmem_alloc(&slot, 256); tmem_relinquish(); }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    constexpr uint32_t idesc = make_idesc_bf16(128, 256, A_MN, B_MN);
    const uint32_t a = smem_u32(smem), b = a + 16384;  // A: 128 x 64 (16 KiB), B: 256 x 64 (32 KiB)
    const uint64_t ad = A_MN ? make_sdesc_sw128(a, 8192, 1024) : make_sdesc_sw128(a, 16, 1024);
    const uint64_t bd = B_MN ? make_sdesc_sw128(b, 8192, 1024) : make_sdesc_sw128(b, 16, 1024);
    if (threadIdx.x == 0) {
        const unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                mma_bf16_ss(tmem, ad + (A_MN ? 128 : 2) * kk, bd + (B_MN ? 128 : 2) * kk, idesc, 1);
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        out[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 256); }
}

template <bool A_MN, bool B_MN>
void run(unsigned long long* d) {
    const int iters = 4096;
    cudaFuncSetAttribute(k<A_MN, B_MN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<A_MN, B_MN><<<148, 128, 64 * 1024>>>(iters, d);
    k<A_MN, B_MN><<<148, 128, 64 * 1024>>>(iters, d);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double mmas = iters * 4.0, ideal = 128.0 * 256 * 16 / 4096.0;  // 4096 bf16 MAC/clk/SM
    printf("A %s x B %s  M=128 N=256 K=16: %.1f cycles/MMA (ideal %.0f) -> %.1f%% of peak  [%s]\n",
           A_MN ? "MN-major" : "K-major ", B_MN ? "MN-major" : "K-major ", mx / mmas, ideal, 100.0 * ideal * mmas / mx,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    run<false, false>(d);
    run<false, true>(d);
    run<true, false>(d);
    run<true, true>(d);
    return 0;
}
