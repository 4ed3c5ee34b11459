// Microbenchmark: tcgen05.mma kind::f16 (bf16, K=16) throughput, cta_group::1 (M=128) vs cta_group::2
// (M=256 over a CTA pair, B split across the pair), smem A ("ss") or TMEM A ("ts"), for several N.
// One CTA (pair) per SM (pair), one converged warp issues back-to-back MMAs, one commit at the end.
// Reports cycles per MMA per SM against the 128*N*16/4096 ideal (4096 bf16 MAC/clk/SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2506_13996_b200/csrc tools/micro/mma_pair_rate.cu
#include <cstdio>
#include "sm100.cuh"
using namespace spt;

template <int N, bool PAIR, bool TS>
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    const int warp = warp_id();
    const uint32_t rank = PAIR ? cluster_ctarank() : 0;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) {
        if (PAIR) { tmem_alloc_pair(&slot, 512); tmem_relinquish_pair(); }
        else { tmem_alloc(&slot, 512); tmem_relinquish(); }
    }
    tc_fence_before();
    if (PAIR) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, slot, 0);
    constexpr uint32_t idesc = make_idesc_bf16(PAIR ? 256 : 128, N, false, false);
    const uint32_t a = smem_u32(smem), b = a + 16384;
    const uint64_t ad = make_sdesc_sw128(a, 16, 1024), bd = make_sdesc_sw128(b, 16, 1024);
    const uint32_t d_t = tmem + 256, a_t = tmem;  // TS: A (bf16, 8 columns per K=16) in columns [0, 32)
    if (warp == 0 && rank == 0) {
        const unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (PAIR) {
                    if (TS) mma_bf16_ts_pair_w(d_t, a_t + 8 * kk, bd + 2 * kk, idesc, 1);
                    else mma_bf16_ss_pair_w(d_t, ad + 2 * kk, bd + 2 * kk, idesc, 1);
                } else {
                    if (TS) mma_bf16_ts_w(d_t, a_t + 8 * kk, bd + 2 * kk, idesc, 1);
                    else mma_bf16_ss_w(d_t, ad + 2 * kk, bd + 2 * kk, idesc, 1);
                }
            }
        }
        if (PAIR) mma_commit_pair_w(&bar, 0x3);
        else mma_commit_w(&bar);
        mbar_wait(&bar, 0);
        if (lane_id() == 0) out[blockIdx.x] = clock64() - t0;
    } else if (PAIR && warp == 0) {
        mbar_wait(&bar, 0);
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();
    if (warp == 0) {
        tc_fence_after();
        if (PAIR) tmem_dealloc_pair(tmem, 512); else tmem_dealloc(tmem, 512);
    }
}

template <int N, bool PAIR, bool TS>
void run(unsigned long long* d) {
    const int iters = 4096 * 64 / N;
    auto kern = k<N, PAIR, TS>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 64 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = PAIR ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    for (int r = 0; r < 2; ++r) cudaLaunchKernelEx(&cfg, kern, iters, d);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double mmas = iters * 4.0, ideal = 128.0 * N * 16 / 4096.0;  // per SM (pair: 256 rows over 2 SMs)
    printf("%s %s M=%d N=%3d K=16: %.1f cycles/MMA (ideal %.0f per SM) -> %.1f%% of peak  [%s]\n",
           PAIR ? "cta_group::2" : "cta_group::1", TS ? "ts" : "ss", PAIR ? 256 : 128, N, h[0] / mmas, ideal,
           100.0 * ideal * mmas / h[0], cudaGetErrorString(cudaGetLastError()));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    cudaMemset(d, 0, 148 * 8);
    run<64, false, false>(d);
    run<64, true, false>(d);
    run<128, false, false>(d);
    run<128, true, false>(d);
    run<256, true, false>(d);
    run<64, false, true>(d);
    run<64, true, true>(d);
    run<128, false, true>(d);
    run<128, true, true>(d);
    return 0;
}
