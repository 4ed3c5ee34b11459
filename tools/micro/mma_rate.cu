// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1, M=128, K=16, bf16) issue-limited throughput vs N.
// One CTA per SM, one elected thread issues back-to-back MMAs (SW128 K-major smem operands, accumulate in
// TMEM), one commit at the end; cycles per MMA and the achieved fraction of the M*N*K/8192 ideal cycles.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2506_13996_b200/csrc tools/micro/mma_rate.cu
#include <cstdio>
#include "sm100.cuh"
using namespace spt;

template <int N, bool UNIFORM>
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
    constexpr uint32_t idesc = make_idesc_bf16(128, N, false, false);
    const uint32_t a = smem_u32(smem), b = a + 16384;
    const uint64_t ad = make_sdesc_sw128(a, 16, 1024), bd = make_sdesc_sw128(b, 16, 1024);
    unsigned long long t0 = 0, t1 = 0;
    if (UNIFORM) {  // whole warp converged, elect.sync inside the wrapper: descriptors on the uniform datapath
        if (warp_id() == 0) {
            t0 = clock64();
            for (int i = 0; i < iters; ++i) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) mma_bf16_ss_w(tmem, ad + 2 * kk, bd + 2 * kk, idesc, 1);
            }
            mma_commit_w(&bar);
            mbar_wait(&bar, 0);
            t1 = clock64();
            if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
        }
    } else if (threadIdx.x == 0) {
        t0 = clock64();
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(tmem, ad + 2 * kk, bd + 2 * kk, idesc, 1);
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 256); }
}

template <int N, bool U>
void run(unsigned long long* d) {
    const int iters = 4096 * 64 / N;  // same flops for every N
    cudaFuncSetAttribute(k<N, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<N, U><<<148, 128, 64 * 1024>>>(iters, d);
    k<N, U><<<148, 128, 64 * 1024>>>(iters, d);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double mmas = iters * 4.0, ideal = mmas * 128.0 * N * 16 / 4096.0;  // 4096 bf16 MAC/clk/SM
    printf("%s M=128 N=%3d K=16: %.1f cycles/MMA (ideal %.0f) -> %.1f%% of peak  [%s]\n", U ? "uniform" : "lane0  ", N,
           h[0] / mmas, 128.0 * N * 16 / 4096.0, 100.0 * ideal / h[0], cudaGetErrorString(cudaGetLastError()));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    run<32, false>(d);
    run<64, false>(d);
    run<128, false>(d);
    run<256, false>(d);
    run<32, true>(d);
    run<64, true>(d);
    run<128, true>(d);
    run<256, true>(d);
    return 0;
}
