// Microbenchmark: tcgen05.ld (32x32b.x32 / .x16) throughput per SM vs number of loading warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2506_13996_b200/csrc tools/micro/tmem_bw.cu -o /tmp/tmem_bw
#include <cstdio>
#include "sm100.cuh"
using namespace spt;

template <int X>
__global__ void __launch_bounds__(512, 1) k(int iters, int nwarps, unsigned long long* out, uint32_t* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) { tmem_alloc(&slot, 512); tmem_relinquish(); }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    uint32_t acc = 0;
    unsigned long long t0 = clock64();
    if (warp < nwarps) {
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t col = (uint32_t)((warp >> 2) * 32) & 511;
        for (int i = 0; i < iters; ++i) {
            uint32_t r[32];
            if constexpr (X == 32) {
                tmem_ld32(tmem + lane_off + ((col + i * 32) & 511), r);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) acc ^= r[j];
            } else {
                uint32_t (&r16)[16] = *reinterpret_cast<uint32_t(*)[16]>(r);
                tmem_ld16(tmem + lane_off + ((col + i * 16) & 511), r16);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 16; ++j) acc ^= r16[j];
            }
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 0x12345678) sink[threadIdx.x] = acc;
    tc_fence_before(); __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
    unsigned long long* d; uint32_t* s;
    cudaMalloc(&d, 148 * 8); cudaMalloc(&s, 4096);
    const int iters = 4096;
    for (int x : {32, 16})
    for (int nw : {4, 8, 16}) {
        unsigned long long h[148];
        for (int rep = 0; rep < 2; ++rep) {
            if (x == 32) k<32><<<148, 512>>>(iters, nw, d, s); else k<16><<<148, 512>>>(iters, nw, d, s);
            cudaDeviceSynchronize();
        }
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double bytes = (double)nw * iters * 32 * x * 4;  // per SM
        printf("x%d warps=%2d: %.1f B/clk/SM (%llu clk)  err=%s\n", x, nw, bytes / h[0], h[0],
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
