// Causal / block-causal GQA flash attention, forward + deterministic backward (K3/K4).
//
// Inner AttentionCallback of ulysses_attention: each rank runs it over the
// full sequence for its local heads.  Masking is evaluated lazily from per-token run starts
// (derive_block_causal_mask_predicate): key j is visible to query i iff
// start[i] <= j <= i.  No [s,s] tensor is ever materialised.
//
// Layout: qkv [s][hq + 2*hkv][D] (q heads, k heads, v heads — the fused-QKV GEMM output at SP=1
// and the seq_to_head receive buffer at SP>1), o [s][hq][D], lse [hq][s] (natural log).
//
// v1 kernels use warp-level mma.sync m16n8k16 (bf16 -> fp32) with ldmatrix from XOR-swizzled
// shared memory and cp.async double buffering.  Backward = dK/dV pass (KV-outer, loops over the GQA
// group's q heads and the visible q blocks) + dQ pass (Q-outer): no atomics, bitwise deterministic
// (SPEC.md:102).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.h"
#include "launch.h"
#include "sm100.cuh"

namespace spt {

namespace fa {

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Tile of R rows x D bf16, rows of D*2 bytes, 16-byte chunks XOR-swizzled by row.
template <int D>
struct Tile {
    static constexpr int CH = D / 8;  // 16B chunks per row
    static constexpr int SW = CH >= 8 ? 8 : CH;
    __device__ static __forceinline__ uint32_t off(int row, int chunk) {
        return (uint32_t)(row * D * 2 + ((chunk ^ (row % SW)) * 16));
    }
};

// Cooperative async copy of `rows` rows (global row pitch gstride elements) into a swizzled tile.
template <int D, int NT>
__device__ __forceinline__ void load_tile(uint32_t sbase, const bf16* g, int64_t gstride, int rows, int64_t row0,
                                          int64_t nrows_total) {
    constexpr int CH = D / 8;
    for (int i = threadIdx.x; i < rows * CH; i += NT) {
        const int r = i / CH, c = i % CH;
        int64_t gr = row0 + r;
        if (gr >= nrows_total) gr = nrows_total - 1;  // clamp (masked anyway)
        cp_async16(sbase + Tile<D>::off(r, c), g + gr * gstride + c * 8);
    }
}

// A fragments (16 rows x 16 cols at (r0, k0)) from a swizzled tile.
template <int D>
__device__ __forceinline__ void ld_a(uint32_t sbase, int r0, int k0, uint32_t (&a)[4]) {
    const int lane = threadIdx.x & 31;
    const int row = r0 + (lane & 7) + 8 * ((lane >> 3) & 1);
    const int chunk = (k0 >> 3) + (lane >> 4);
    ldsm_x4(sbase + Tile<D>::off(row, chunk), a[0], a[1], a[2], a[3]);
}
// B fragments for two n-tiles (n0, n0+8) x k16 at k0 from a tile stored [n][k] (non-transposed).
template <int D>
__device__ __forceinline__ void ld_b_nk(uint32_t sbase, int n0, int k0, uint32_t& b00, uint32_t& b01, uint32_t& b10,
                                        uint32_t& b11) {
    const int lane = threadIdx.x & 31;
    const int row = n0 + (lane & 7) + 8 * (lane >> 4);
    const int chunk = (k0 >> 3) + ((lane >> 3) & 1);
    ldsm_x4(sbase + Tile<D>::off(row, chunk), b00, b01, b10, b11);
}
// B fragments for two n-tiles (n0, n0+8) x k16 at k0 from a tile stored [k][n] (transposed load).
template <int D>
__device__ __forceinline__ void ld_b_kn(uint32_t sbase, int n0, int k0, uint32_t& b00, uint32_t& b01, uint32_t& b10,
                                        uint32_t& b11) {
    const int lane = threadIdx.x & 31;
    const int row = k0 + (lane & 7) + 8 * ((lane >> 3) & 1);
    const int chunk = (n0 >> 3) + (lane >> 4);
    ldsm_x4_t(sbase + Tile<D>::off(row, chunk), b00, b01, b10, b11);
}

__device__ __forceinline__ float quad_max(float v) {
    v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
    return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
__device__ __forceinline__ float quad_sum(float v) {
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    return v + __shfl_xor_sync(0xffffffffu, v, 2);
}

constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

// ------------------------------------------------------------------ forward
template <int D>
__global__ void __launch_bounds__(256) fwd_kernel(const bf16* __restrict__ qkv, int64_t s, int hq, int hkv,
                                                  const int32_t* __restrict__ seg, float scale, bf16* __restrict__ o,
                                                  float* __restrict__ lse) {
    constexpr int BM = 128, BN = 64, NT = 256;
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sQ = smem_u32(smem);
    const uint32_t sK0 = sQ + BM * D * 2;
    const uint32_t sV0 = sK0 + 2 * BN * D * 2;
    const int nqb = (int)((s + BM - 1) / BM);
    const int qb = nqb - 1 - blockIdx.x;  // longest causal rows first
    const int h = blockIdx.y;
    const int kvh = h / (hq / hkv);
    const int64_t rs = (int64_t)(hq + 2 * hkv) * D;
    const bf16* Qg = qkv + (int64_t)h * D;
    const bf16* Kg = qkv + (int64_t)(hq + kvh) * D;
    const bf16* Vg = qkv + (int64_t)(hq + hkv + kvh) * D;
    const int64_t q0 = (int64_t)qb * BM;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;

    const int64_t kmin = seg ? (int64_t)seg[q0] : 0;
    const int kb0 = (int)(kmin / BN);
    const int kb1 = (int)(std::min<int64_t>(q0 + BM, s) - 1) / BN;

    load_tile<D, NT>(sQ, Qg, rs, BM, q0, s);
    load_tile<D, NT>(sK0, Kg, rs, BN, (int64_t)kb0 * BN, s);
    load_tile<D, NT>(sV0, Vg, rs, BN, (int64_t)kb0 * BN, s);
    cp_async_commit();

    const int64_t row_a = q0 + warp * 16 + g, row_b = row_a + 8;
    const int start_a = seg ? (row_a < s ? seg[row_a] : 0) : 0;
    const int start_b = seg ? (row_b < s ? seg[row_b] : 0) : 0;

    uint32_t qf[D / 16][4];
    float oacc[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
    float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
    const float sl2 = scale * LOG2E;

    for (int kb = kb0; kb <= kb1; ++kb) {
        const int buf = (kb - kb0) & 1;
        if (kb < kb1) {
            load_tile<D, NT>(sK0 + (buf ^ 1) * BN * D * 2, Kg, rs, BN, (int64_t)(kb + 1) * BN, s);
            load_tile<D, NT>(sV0 + (buf ^ 1) * BN * D * 2, Vg, rs, BN, (int64_t)(kb + 1) * BN, s);
        }
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        if (kb == kb0) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) ld_a<D>(sQ, warp * 16, kk * 16, qf[kk]);
        }
        const uint32_t sK = sK0 + buf * BN * D * 2, sV = sV0 + buf * BN * D * 2;
        float sacc[BN / 8][4];
#pragma unroll
        for (int i = 0; i < BN / 8; ++i) sacc[i][0] = sacc[i][1] = sacc[i][2] = sacc[i][3] = 0.f;
#pragma unroll
        for (int np = 0; np < BN / 16; ++np) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                uint32_t b00, b01, b10, b11;
                ld_b_nk<D>(sK, np * 16, kk * 16, b00, b01, b10, b11);
                mma16816(sacc[2 * np], qf[kk], b00, b01);
                mma16816(sacc[2 * np + 1], qf[kk], b10, b11);
            }
        }
        // mask + online softmax (log2 domain)
        const int64_t key0 = (int64_t)kb * BN;
        const bool need_mask = seg != nullptr || key0 + BN - 1 > q0 + warp * 16;
        float mx_a = -INFINITY, mx_b = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < BN / 8; ++nt) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int64_t key = key0 + nt * 8 + 2 * t4 + (e & 1);
                const bool rb = e >= 2;
                float v = sacc[nt][e] * sl2;
                if (need_mask) {
                    const int64_t qi = rb ? row_b : row_a;
                    const int st = rb ? start_b : start_a;
                    if (key > qi || key < st) v = -INFINITY;
                }
                sacc[nt][e] = v;
                if (rb) mx_b = fmaxf(mx_b, v);
                else mx_a = fmaxf(mx_a, v);
            }
        }
        mx_a = quad_max(mx_a);
        mx_b = quad_max(mx_b);
        const float mn_a = fmaxf(m_a, mx_a), mn_b = fmaxf(m_b, mx_b);
        const float mu_a = mn_a == -INFINITY ? 0.f : mn_a, mu_b = mn_b == -INFINITY ? 0.f : mn_b;
        const float al_a = exp2f(m_a - mu_a), al_b = exp2f(m_b - mu_b);
        m_a = mn_a;
        m_b = mn_b;
        float rs_a = 0.f, rs_b = 0.f;
        uint32_t pf[BN / 16][4];
#pragma unroll
        for (int nt = 0; nt < BN / 8; ++nt) {
            const float p0 = exp2f(sacc[nt][0] - mu_a), p1 = exp2f(sacc[nt][1] - mu_a);
            const float p2 = exp2f(sacc[nt][2] - mu_b), p3 = exp2f(sacc[nt][3] - mu_b);
            rs_a += p0 + p1;
            rs_b += p2 + p3;
            const int j = nt >> 1, hi = nt & 1;
            pf[j][hi ? 2 : 0] = pack_bf16x2(p0, p1);
            pf[j][hi ? 3 : 1] = pack_bf16x2(p2, p3);
        }
        l_a = l_a * al_a + quad_sum(rs_a);
        l_b = l_b * al_b + quad_sum(rs_b);
#pragma unroll
        for (int i = 0; i < D / 8; ++i) {
            oacc[i][0] *= al_a;
            oacc[i][1] *= al_a;
            oacc[i][2] *= al_b;
            oacc[i][3] *= al_b;
        }
#pragma unroll
        for (int j = 0; j < BN / 16; ++j) {
#pragma unroll
            for (int dp = 0; dp < D / 16; ++dp) {
                uint32_t b00, b01, b10, b11;
                ld_b_kn<D>(sV, dp * 16, j * 16, b00, b01, b10, b11);
                mma16816(oacc[2 * dp], pf[j], b00, b01);
                mma16816(oacc[2 * dp + 1], pf[j], b10, b11);
            }
        }
        __syncthreads();
    }
    // epilogue
    const float inv_a = l_a > 0.f ? 1.f / l_a : 0.f, inv_b = l_b > 0.f ? 1.f / l_b : 0.f;
    if (row_a < s) {
        bf16* orow = o + (row_a * hq + h) * D;
#pragma unroll
        for (int i = 0; i < D / 8; ++i)
            *reinterpret_cast<uint32_t*>(orow + i * 8 + 2 * t4) = pack_bf16x2(oacc[i][0] * inv_a, oacc[i][1] * inv_a);
        if (t4 == 0) lse[(int64_t)h * s + row_a] = (m_a + __log2f(l_a)) * LN2;
    }
    if (row_b < s) {
        bf16* orow = o + (row_b * hq + h) * D;
#pragma unroll
        for (int i = 0; i < D / 8; ++i)
            *reinterpret_cast<uint32_t*>(orow + i * 8 + 2 * t4) = pack_bf16x2(oacc[i][2] * inv_b, oacc[i][3] * inv_b);
        if (t4 == 0) lse[(int64_t)h * s + row_b] = (m_b + __log2f(l_b)) * LN2;
    }
}

// ------------------------------------------------------------------ backward
// D_i = sum_d dO_i * O_i  per (token, head), fp32 [hq][s]
template <int D>
__global__ void bwd_dot_kernel(const bf16* __restrict__ o, const bf16* __restrict__ dout, const float* __restrict__ lse,
                               int64_t s, int hq, float* __restrict__ Dv, float* __restrict__ lse2) {
    const int64_t n = s * hq;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / hq;
        const int h = (int)(i % hq);
        const bf16* a = o + i * D;
        const bf16* b = dout + i * D;
        float acc = 0.f;
#pragma unroll 4
        for (int c = 0; c < D; c += 8) {
            float x[8], y[8];
            load8(a + c, x);
            load8(b + c, y);
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += x[k] * y[k];
        }
        Dv[(int64_t)h * s + t] = acc;
        lse2[(int64_t)h * s + t] = lse[(int64_t)h * s + t] * LOG2E;
    }
}

// dK/dV: CTA = (kv head, 128-key block); 8 warps x 16 keys.  Loops over the GQA group's q heads and
// the 64-query blocks that can see the key block; accumulates dK, dV in registers.
template <int D>
__global__ void __launch_bounds__(256, 1) bwd_dkdv_kernel(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                                          const float* __restrict__ lse, const float* __restrict__ Dv,
                                                          int64_t s, int hq, int hkv, const int32_t* __restrict__ seg,
                                                          float scale, bf16* __restrict__ dqkv) {
    constexpr int BKEY = 128, BQ = 64, NT = 256;
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sK = smem_u32(smem);
    const uint32_t sV = sK + BKEY * D * 2;
    const uint32_t sQ0 = sV + BKEY * D * 2;        // [2][BQ][D]
    const uint32_t sO0 = sQ0 + 2 * BQ * D * 2;     // dO tiles [2][BQ][D]
    float* sL = reinterpret_cast<float*>(smem + (size_t)(2 * BKEY + 4 * BQ) * D * 2);  // [2][BQ] lse
    float* sD = sL + 2 * BQ;                                                         // [2][BQ] D
    const int nkb = (int)((s + BKEY - 1) / BKEY);
    const int kb = blockIdx.x;
    const int kvh = blockIdx.y;
    const int grp = hq / hkv;
    const int64_t rs = (int64_t)(hq + 2 * hkv) * D;
    const int64_t k0 = (int64_t)kb * BKEY;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    (void)nkb;

    load_tile<D, NT>(sK, qkv + (int64_t)(hq + kvh) * D, rs, BKEY, k0, s);
    load_tile<D, NT>(sV, qkv + (int64_t)(hq + hkv + kvh) * D, rs, BKEY, k0, s);
    cp_async_commit();

    // visible q range: q >= k0 (causal) and start[q] <= k0 + BKEY - 1 (starts are monotone)
    const int qb_first = (int)(k0 / BQ);
    int qb_last = (int)((s - 1) / BQ);
    if (seg) {
        // binary search last q with seg[q] <= k_last
        const int64_t klast = std::min<int64_t>(k0 + BKEY, s) - 1;
        int64_t lo = k0, hi = s - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) / 2;
            if (seg[mid] <= klast) lo = mid;
            else hi = mid - 1;
        }
        qb_last = (int)(lo / BQ);
    }
    const int nq = qb_last - qb_first + 1;
    const int total = nq * grp;

    float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;

    const int64_t key_a = k0 + warp * 16 + g, key_b = key_a + 8;  // rows of S^T owned by this thread
    auto issue = [&](int it, int buf) {
        const int hh = kvh * grp + it / nq;
        const int64_t q0 = (int64_t)(qb_first + it % nq) * BQ;
        load_tile<D, NT>(sQ0 + buf * BQ * D * 2, qkv + (int64_t)hh * D, rs, BQ, q0, s);
        load_tile<D, NT>(sO0 + buf * BQ * D * 2, dout + (int64_t)hh * D, (int64_t)hq * D, BQ, q0, s);
        for (int i = threadIdx.x; i < BQ; i += NT) {
            const int64_t q = std::min<int64_t>(q0 + i, s - 1);
            sL[buf * BQ + i] = lse[(int64_t)hh * s + q];
            sD[buf * BQ + i] = Dv[(int64_t)hh * s + q];
        }
    };
    if (total > 0) issue(0, 0);
    cp_async_commit();
    const float sl2 = scale * LOG2E;
    for (int it = 0; it < total; ++it) {
        const int buf = it & 1;
        if (it + 1 < total) issue(it + 1, buf ^ 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const int64_t q0 = (int64_t)(qb_first + it % nq) * BQ;
        const uint32_t sQ = sQ0 + buf * BQ * D * 2, sO = sO0 + buf * BQ * D * 2;
        // S^T = K Q^T  (16 keys x 64 queries per warp), dP^T = V dO^T
        float st[BQ / 8][4], dpt[BQ / 8][4];
#pragma unroll
        for (int i = 0; i < BQ / 8; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) st[i][e] = dpt[i][e] = 0.f;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
            uint32_t ka[4], va[4];
            ld_a<D>(sK, warp * 16, kk * 16, ka);
            ld_a<D>(sV, warp * 16, kk * 16, va);
#pragma unroll
            for (int np = 0; np < BQ / 16; ++np) {
                uint32_t b00, b01, b10, b11;
                ld_b_nk<D>(sQ, np * 16, kk * 16, b00, b01, b10, b11);
                mma16816(st[2 * np], ka, b00, b01);
                mma16816(st[2 * np + 1], ka, b10, b11);
                ld_b_nk<D>(sO, np * 16, kk * 16, b00, b01, b10, b11);
                mma16816(dpt[2 * np], va, b00, b01);
                mma16816(dpt[2 * np + 1], va, b10, b11);
            }
        }
        // P^T, dS^T
        uint32_t pa[BQ / 16][4], dsa[BQ / 16][4];
#pragma unroll
        for (int nt = 0; nt < BQ / 8; ++nt) {
            float pv[4], dsv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int qi = nt * 8 + 2 * t4 + (e & 1);
                const int64_t q = q0 + qi;
                const int64_t key = (e >= 2) ? key_b : key_a;
                bool ok = key <= q && q < s;
                if (seg && ok) ok = key >= seg[q];
                const float p = ok ? exp2f(st[nt][e] * sl2 - sL[buf * BQ + qi] * LOG2E) : 0.f;
                pv[e] = p;
                dsv[e] = p * (dpt[nt][e] - sD[buf * BQ + qi]);
            }
            const int j = nt >> 1, hi = nt & 1;
            pa[j][hi ? 2 : 0] = pack_bf16x2(pv[0], pv[1]);
            pa[j][hi ? 3 : 1] = pack_bf16x2(pv[2], pv[3]);
            dsa[j][hi ? 2 : 0] = pack_bf16x2(dsv[0], dsv[1]);
            dsa[j][hi ? 3 : 1] = pack_bf16x2(dsv[2], dsv[3]);
        }
        // dV += P^T dO ; dK += dS^T Q   (k = queries)
#pragma unroll
        for (int j = 0; j < BQ / 16; ++j) {
#pragma unroll
            for (int dp = 0; dp < D / 16; ++dp) {
                uint32_t b00, b01, b10, b11;
                ld_b_kn<D>(sO, dp * 16, j * 16, b00, b01, b10, b11);
                mma16816(dv[2 * dp], pa[j], b00, b01);
                mma16816(dv[2 * dp + 1], pa[j], b10, b11);
                ld_b_kn<D>(sQ, dp * 16, j * 16, b00, b01, b10, b11);
                mma16816(dk[2 * dp], dsa[j], b00, b01);
                mma16816(dk[2 * dp + 1], dsa[j], b10, b11);
            }
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    // write dK (scaled), dV
    bf16* dK = dqkv + (int64_t)(hq + kvh) * D;
    bf16* dV = dqkv + (int64_t)(hq + hkv + kvh) * D;
    if (key_a < s) {
#pragma unroll
        for (int i = 0; i < D / 8; ++i) {
            *reinterpret_cast<uint32_t*>(dK + key_a * rs + i * 8 + 2 * t4) = pack_bf16x2(dk[i][0] * scale, dk[i][1] * scale);
            *reinterpret_cast<uint32_t*>(dV + key_a * rs + i * 8 + 2 * t4) = pack_bf16x2(dv[i][0], dv[i][1]);
        }
    }
    if (key_b < s) {
#pragma unroll
        for (int i = 0; i < D / 8; ++i) {
            *reinterpret_cast<uint32_t*>(dK + key_b * rs + i * 8 + 2 * t4) = pack_bf16x2(dk[i][2] * scale, dk[i][3] * scale);
            *reinterpret_cast<uint32_t*>(dV + key_b * rs + i * 8 + 2 * t4) = pack_bf16x2(dv[i][2], dv[i][3]);
        }
    }
}

// dQ: CTA = (q head, 128-query block); loops over visible 64-key blocks.
template <int D>
__global__ void __launch_bounds__(256, 1) bwd_dq_kernel(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                                        const float* __restrict__ lse, const float* __restrict__ Dv,
                                                        int64_t s, int hq, int hkv, const int32_t* __restrict__ seg,
                                                        float scale, bf16* __restrict__ dqkv) {
    constexpr int BM = 128, BN = 64, NT = 256;
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sQ = smem_u32(smem);
    const uint32_t sO = sQ + BM * D * 2;
    const uint32_t sK0 = sO + BM * D * 2;
    const uint32_t sV0 = sK0 + 2 * BN * D * 2;
    const int nqb = (int)((s + BM - 1) / BM);
    const int qb = nqb - 1 - blockIdx.x;
    const int h = blockIdx.y;
    const int kvh = h / (hq / hkv);
    const int64_t rs = (int64_t)(hq + 2 * hkv) * D;
    const bf16* Kg = qkv + (int64_t)(hq + kvh) * D;
    const bf16* Vg = qkv + (int64_t)(hq + hkv + kvh) * D;
    const int64_t q0 = (int64_t)qb * BM;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const int64_t kmin = seg ? (int64_t)seg[q0] : 0;
    const int kb0 = (int)(kmin / BN);
    const int kb1 = (int)((std::min<int64_t>(q0 + BM, s) - 1) / BN);

    load_tile<D, NT>(sQ, qkv + (int64_t)h * D, rs, BM, q0, s);
    load_tile<D, NT>(sO, dout + (int64_t)h * D, (int64_t)hq * D, BM, q0, s);
    load_tile<D, NT>(sK0, Kg, rs, BN, (int64_t)kb0 * BN, s);
    load_tile<D, NT>(sV0, Vg, rs, BN, (int64_t)kb0 * BN, s);
    cp_async_commit();

    const int64_t row_a = q0 + warp * 16 + g, row_b = row_a + 8;
    const int64_t ra = std::min<int64_t>(row_a, s - 1), rb = std::min<int64_t>(row_b, s - 1);
    const float lse_a = lse[(int64_t)h * s + ra] * LOG2E, lse_b = lse[(int64_t)h * s + rb] * LOG2E;
    const float D_a = Dv[(int64_t)h * s + ra], D_b = Dv[(int64_t)h * s + rb];
    const int start_a = seg ? seg[ra] : 0, start_b = seg ? seg[rb] : 0;
    const float sl2 = scale * LOG2E;

    uint32_t qf[D / 16][4], of[D / 16][4];
    float dq[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;

    for (int kb = kb0; kb <= kb1; ++kb) {
        const int buf = (kb - kb0) & 1;
        if (kb < kb1) {
            load_tile<D, NT>(sK0 + (buf ^ 1) * BN * D * 2, Kg, rs, BN, (int64_t)(kb + 1) * BN, s);
            load_tile<D, NT>(sV0 + (buf ^ 1) * BN * D * 2, Vg, rs, BN, (int64_t)(kb + 1) * BN, s);
        }
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        if (kb == kb0) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                ld_a<D>(sQ, warp * 16, kk * 16, qf[kk]);
                ld_a<D>(sO, warp * 16, kk * 16, of[kk]);
            }
        }
        const uint32_t sK = sK0 + buf * BN * D * 2, sV = sV0 + buf * BN * D * 2;
        float sacc[BN / 8][4], dp[BN / 8][4];
#pragma unroll
        for (int i = 0; i < BN / 8; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) sacc[i][e] = dp[i][e] = 0.f;
#pragma unroll
        for (int np = 0; np < BN / 16; ++np) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                uint32_t b00, b01, b10, b11;
                ld_b_nk<D>(sK, np * 16, kk * 16, b00, b01, b10, b11);
                mma16816(sacc[2 * np], qf[kk], b00, b01);
                mma16816(sacc[2 * np + 1], qf[kk], b10, b11);
                ld_b_nk<D>(sV, np * 16, kk * 16, b00, b01, b10, b11);
                mma16816(dp[2 * np], of[kk], b00, b01);
                mma16816(dp[2 * np + 1], of[kk], b10, b11);
            }
        }
        const int64_t key0 = (int64_t)kb * BN;
        uint32_t dsf[BN / 16][4];
#pragma unroll
        for (int nt = 0; nt < BN / 8; ++nt) {
            float dsv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int64_t key = key0 + nt * 8 + 2 * t4 + (e & 1);
                const bool b = e >= 2;
                const int64_t qi = b ? row_b : row_a;
                const bool ok = key <= qi && key >= (b ? start_b : start_a);
                const float p = ok ? exp2f(sacc[nt][e] * sl2 - (b ? lse_b : lse_a)) : 0.f;
                dsv[e] = p * (dp[nt][e] - (b ? D_b : D_a));
            }
            const int j = nt >> 1, hi = nt & 1;
            dsf[j][hi ? 2 : 0] = pack_bf16x2(dsv[0], dsv[1]);
            dsf[j][hi ? 3 : 1] = pack_bf16x2(dsv[2], dsv[3]);
        }
#pragma unroll
        for (int j = 0; j < BN / 16; ++j) {
#pragma unroll
            for (int dpi = 0; dpi < D / 16; ++dpi) {
                uint32_t b00, b01, b10, b11;
                ld_b_kn<D>(sK, dpi * 16, j * 16, b00, b01, b10, b11);
                mma16816(dq[2 * dpi], dsf[j], b00, b01);
                mma16816(dq[2 * dpi + 1], dsf[j], b10, b11);
            }
        }
        __syncthreads();
    }
    bf16* dQ = dqkv + (int64_t)h * D;
    if (row_a < s) {
#pragma unroll
        for (int i = 0; i < D / 8; ++i)
            *reinterpret_cast<uint32_t*>(dQ + row_a * rs + i * 8 + 2 * t4) = pack_bf16x2(dq[i][0] * scale, dq[i][1] * scale);
    }
    if (row_b < s) {
#pragma unroll
        for (int i = 0; i < D / 8; ++i)
            *reinterpret_cast<uint32_t*>(dQ + row_b * rs + i * 8 + 2 * t4) = pack_bf16x2(dq[i][2] * scale, dq[i][3] * scale);
    }
}

}  // namespace fa

template <int D>
static void attn_fwd_t(const void* qkv, int64_t s, int hq, int hkv, const int32_t* seg, float scale, void* o,
                       float* lse, cudaStream_t st) {
    constexpr int smem = (128 + 4 * 64) * D * 2;
    auto k = fa::fwd_kernel<D>;
    static bool attr = false;
    if (!attr) {
        SPT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    dim3 grid((unsigned)((s + 127) / 128), (unsigned)hq);
    k<<<grid, 256, smem, st>>>((const bf16*)qkv, s, hq, hkv, seg, scale, (bf16*)o, lse);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

bool attn_bwd_tc(const void* qkv, const void* dout, const float* lse, const float* Dv, int64_t s, int hq, int hkv,
                 int d, const int32_t* seg, float scale, void* dqkv, void* ws, cudaStream_t st);
size_t attn_bwd_tc_workspace(int64_t s, int hq);
static int attn_impl();

template <int D>
static void attn_bwd_t(const void* qkv, const void* o, const float* lse, const void* dout, int64_t s, int hq, int hkv,
                       const int32_t* seg, float scale, void* dqkv, void* ws, cudaStream_t st) {
    float* Dv = (float*)ws;
    float* lse2 = Dv + s * hq;
    fa::bwd_dot_kernel<D><<<(unsigned)std::min<int64_t>((s * hq + 255) / 256, 148 * 16), 256, 0, st>>>(
        (const bf16*)o, (const bf16*)dout, lse, s, hq, Dv, lse2);
    count_launch();
    SPT_CUDA(cudaGetLastError());
    if (attn_impl() == 1 && attn_bwd_tc(qkv, dout, lse2, Dv, s, hq, hkv, D, seg, scale, dqkv, lse2 + s * hq, st)) return;
    {
        constexpr int smem = (2 * 128 + 4 * 64) * D * 2 + 4 * 64 * 4;
        auto k = fa::bwd_dkdv_kernel<D>;
        static bool attr = false;
        if (!attr) {
            SPT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            attr = true;
        }
        dim3 grid((unsigned)((s + 127) / 128), (unsigned)hkv);
        k<<<grid, 256, smem, st>>>((const bf16*)qkv, (const bf16*)dout, lse, Dv, s, hq, hkv, seg, scale, (bf16*)dqkv);
        count_launch();
        SPT_CUDA(cudaGetLastError());
    }
    {
        constexpr int smem = (2 * 128 + 4 * 64) * D * 2;
        auto k = fa::bwd_dq_kernel<D>;
        static bool attr = false;
        if (!attr) {
            SPT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            attr = true;
        }
        dim3 grid((unsigned)((s + 127) / 128), (unsigned)hq);
        k<<<grid, 256, smem, st>>>((const bf16*)qkv, (const bf16*)dout, lse, Dv, s, hq, hkv, seg, scale, (bf16*)dqkv);
        count_launch();
        SPT_CUDA(cudaGetLastError());
    }
}

static void check_attn(int64_t s, int hq, int hkv, int d) {
    SPT_CHECK(hq > 0 && hkv > 0 && hq % hkv == 0, SPT_ERR_SHAPE, "attention: hq must be a multiple of hkv");
    SPT_CHECK(s > 0 && s % 128 == 0, SPT_ERR_SHAPE, "attention: sequence length must be a multiple of 128");
    SPT_CHECK(d == 32 || d == 64 || d == 128, SPT_ERR_SHAPE, "attention: head_dim must be 32, 64 or 128");
}

bool attn_fwd_tc(const void* qkv, int64_t s, int hq, int hkv, int d, const int32_t* seg, float scale, void* o,
                 float* lse, cudaStream_t st);

static int attn_impl() {
    static int v = [] {
        const char* e = getenv("SPT_ATTN_IMPL");  // "mma" forces the mma.sync kernels (A/B comparisons)
        return (e && std::string(e) == "mma") ? 0 : 1;
    }();
    return v;
}

void attn_fwd(const void* qkv, int64_t s, int hq, int hkv, int d, const int32_t* seg, float scale, void* o, float* lse,
              cudaStream_t st) {
    check_attn(s, hq, hkv, d);
    if (attn_impl() == 1 && attn_fwd_tc(qkv, s, hq, hkv, d, seg, scale, o, lse, st)) return;
    if (d == 128) attn_fwd_t<128>(qkv, s, hq, hkv, seg, scale, o, lse, st);
    else if (d == 64) attn_fwd_t<64>(qkv, s, hq, hkv, seg, scale, o, lse, st);
    else attn_fwd_t<32>(qkv, s, hq, hkv, seg, scale, o, lse, st);
}

size_t attn_bwd_workspace(int64_t s, int hq, int hkv, int d) {
    (void)hkv;
    // D = rowsum(dO*O) and lse*log2(e), then (head_dim 128, tcgen05 path) the fp32 dQ accumulator and the
    // dQ ordering counters of the fused backward
    return (size_t)s * hq * 4 * 2 + (d == 128 ? attn_bwd_tc_workspace(s, hq) : 0);
}

void attn_bwd(const void* qkv, const void* o, const float* lse, const void* dout, int64_t s, int hq, int hkv, int d,
              const int32_t* seg, float scale, void* dqkv, void* ws, cudaStream_t st) {
    check_attn(s, hq, hkv, d);
    if (d == 128) attn_bwd_t<128>(qkv, o, lse, dout, s, hq, hkv, seg, scale, dqkv, ws, st);
    else if (d == 64) attn_bwd_t<64>(qkv, o, lse, dout, s, hq, hkv, seg, scale, dqkv, ws, st);
    else attn_bwd_t<32>(qkv, o, lse, dout, s, hq, hkv, seg, scale, dqkv, ws, st);
}

}  // namespace spt
