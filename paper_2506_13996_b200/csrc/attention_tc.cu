// tcgen05 / TMEM / TMA flash-attention forward for head_dim 128 (K3, Blackwell-native).
//
// CTA = (pair of consecutive 128-row query tiles, q head); 10 warps:
//   warps 0-3  softmax warpgroup for tile 0, warps 4-7 for tile 1 (thread = query row)
//   warp 8     MMA issuer (one lane) + TMEM owner (512 columns: S0 | S1 | O0 | O1)
//   warp 9     TMA producer: Q tiles once, then K_j / V_j through a 3-slot ring
// Per 128-key block j and tile t:  S_t = Q_t K_j^T (TMEM) -> softmax warps read S_t, mask
// (causal / block-causal runs), online max with lazy rescale (only when the running
// max grows by > 2^8, then O_t is rescaled in TMEM), P_t (bf16) -> swizzled smem -> O_t += P_t V_j.
// MMA order S0 S1 | PV0 S0' PV1 S1' | ... keeps one tile's softmax overlapped with the other tile's
// MMAs.  tcgen05 ops complete in issue order, so the commit that signals S_t(j+1) also certifies
// PV_t(j) is done (P_t buffer reusable, O_t stable for a rescale).
#include <algorithm>

#include "common.h"
#include "launch.h"
#include "sm100.cuh"

namespace spt {
namespace fatc {

constexpr int D = 128;
constexpr int BQ = 128;   // rows per query tile
constexpr int BK = 128;   // keys per block
constexpr int TILE_BYTES = BQ * D * 2;  // 32 KiB (two 16 KiB SW128 column regions)
constexpr int NSLOT = 3;
constexpr int SMEM_Q = 0;
constexpr int SMEM_P = 2 * TILE_BYTES;
constexpr int SMEM_KV = 4 * TILE_BYTES;
constexpr int SMEM_BAR = SMEM_KV + NSLOT * TILE_BYTES;
constexpr int SMEM_BYTES = SMEM_BAR + 256 + 1024;
constexpr int THREADS = 320;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;
constexpr float RESCALE_THRESHOLD = 8.f;  // log2 units

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

// K-major SW128 descriptor over a [128 rows][128 cols] bf16 tile stored as two 16 KiB column regions.
__device__ __forceinline__ uint64_t kdesc(uint32_t tile, int kk) {
    return make_sdesc_sw128(tile + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
}
// MN-major SW128 descriptor (rows = K, 64-wide MN blocks 16 KiB apart) advanced by kk*16 rows.
__device__ __forceinline__ uint64_t mndesc(uint32_t tile, int kk) {
    return make_sdesc_sw128(tile + kk * 2048, 16384, 1024);
}

__global__ void __launch_bounds__(THREADS, 1)
    fwd_tc_kernel(const __grid_constant__ CUtensorMap tm, int64_t s, int hq, int hkv, const int32_t* __restrict__ seg,
                  float scale_log2, bf16* __restrict__ o, float* __restrict__ lse) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SMEM_BAR);
    uint64_t* q_full = bar;
    uint64_t* kv_full = bar + 1;
    uint64_t* kv_empty = bar + 1 + NSLOT;
    uint64_t* s_full = bar + 1 + 2 * NSLOT;  // [2]
    uint64_t* p_full = s_full + 2;           // [2]
    uint64_t* o_done = p_full + 2;           // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

    const int warp = warp_id(), lane = lane_id();
    const int npairs = (int)(s / (2 * BQ));
    const int pair = npairs - 1 - (int)blockIdx.x;  // longest causal rows first
    const int h = blockIdx.y;
    const int kvh = h / (hq / hkv);
    const int64_t q0 = (int64_t)pair * 2 * BQ;
    // key-block ranges per tile
    int jb[2], je[2];
    for (int t = 0; t < 2; ++t) {
        const int64_t first = q0 + t * BQ;
        je[t] = (int)((first + BQ - 1) / BK);
        jb[t] = seg ? (int)(seg[first] / BK) : 0;
    }
    const int jlo = min(jb[0], jb[1]), jhi = max(je[0], je[1]);

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < NSLOT; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&s_full[t], 1);
            mbar_init(&p_full[t], 128);
            mbar_init(&o_done[t], 1);
        }
        fence_barrier_init();
    }
    if (warp == 8) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sbase = smem_u32(smem);

    if (warp == 9) {
        if (lane == 0) {
            tma_prefetch_desc(&tm);
            mbar_arrive_expect_tx(q_full, 2 * TILE_BYTES);
            for (int t = 0; t < 2; ++t)
                for (int r = 0; r < 2; ++r)
                    tma_load_2d(&tm, q_full, smem + SMEM_Q + t * TILE_BYTES + r * 16384, h * D + 64 * r,
                                (int)(q0 + t * BQ));
            int li = 0;
            for (int j = jlo; j <= jhi; ++j) {
                for (int w = 0; w < 2; ++w, ++li) {  // w=0: K_j, w=1: V_j
                    const int slot = li % NSLOT;
                    const uint32_t ph = (li / NSLOT) & 1;
                    mbar_wait(&kv_empty[slot], ph ^ 1);
                    mbar_arrive_expect_tx(&kv_full[slot], TILE_BYTES);
                    const int col = (hq + (w ? hkv : 0) + kvh) * D;
                    for (int r = 0; r < 2; ++r)
                        tma_load_2d(&tm, &kv_full[slot], smem + SMEM_KV + slot * TILE_BYTES + r * 16384, col + 64 * r,
                                    j * BK);
                }
            }
        }
    } else if (warp == 8) {
        if (lane == 0) {
            constexpr uint32_t idesc_s = make_idesc_bf16(BQ, BK, false, false);
            constexpr uint32_t idesc_o = make_idesc_bf16(BQ, D, false, true);
            mbar_wait(q_full, 0);
            int pv_count[2] = {0, 0};
            auto uses = [&](int t, int j) { return j >= jb[t] && j <= je[t]; };
            auto slot_of = [&](int j, int w) { return (2 * (j - jlo) + w) % NSLOT; };
            auto phase_of = [&](int j, int w) { return (uint32_t)(((2 * (j - jlo) + w) / NSLOT) & 1); };
            auto issue_s = [&](int t, int j) {
                mbar_wait(&kv_full[slot_of(j, 0)], phase_of(j, 0));
                tc_fence_after();
                const uint32_t qa = sbase + SMEM_Q + t * TILE_BYTES;
                const uint32_t kb = sbase + SMEM_KV + slot_of(j, 0) * TILE_BYTES;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) mma_bf16_ss(tmem + t * BK, kdesc(qa, kk), kdesc(kb, kk), idesc_s, kk > 0);
                mma_commit(&s_full[t]);
            };
            auto issue_pv = [&](int t, int j) {
                mbar_wait(&p_full[t], pv_count[t] & 1);
                mbar_wait(&kv_full[slot_of(j, 1)], phase_of(j, 1));
                tc_fence_after();
                const uint32_t pa = sbase + SMEM_P + t * TILE_BYTES;
                const uint32_t vb = sbase + SMEM_KV + slot_of(j, 1) * TILE_BYTES;
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk)
                    mma_bf16_ss(tmem + 256 + t * D, kdesc(pa, kk), mndesc(vb, kk), idesc_o, (pv_count[t] > 0 || kk > 0));
                ++pv_count[t];
            };
            if (uses(0, jlo)) issue_s(0, jlo);
            if (uses(1, jlo)) issue_s(1, jlo);
            mma_commit(&kv_empty[slot_of(jlo, 0)]);
            for (int j = jlo; j <= jhi; ++j) {
                if (uses(0, j)) issue_pv(0, j);
                if (j + 1 <= jhi && uses(0, j + 1)) issue_s(0, j + 1);
                if (uses(1, j)) issue_pv(1, j);
                mma_commit(&kv_empty[slot_of(j, 1)]);
                if (j + 1 <= jhi) {
                    if (uses(1, j + 1)) issue_s(1, j + 1);
                    mma_commit(&kv_empty[slot_of(j + 1, 0)]);
                }
            }
            mma_commit(&o_done[0]);
            mma_commit(&o_done[1]);
        }
    } else {
        // ---------------- softmax warpgroups
        const int t = warp >> 2;
        const int sub = warp & 3;
        const int r = sub * 32 + lane;
        const int64_t q = q0 + t * BQ + r;
        const int start = seg ? seg[q] : 0;
        const uint32_t lane_off = (uint32_t)(sub * 32) << 16;
        const uint32_t s_tm = tmem + lane_off + t * BK;
        const uint32_t o_tm = tmem + lane_off + 256 + t * D;
        const uint32_t prow = sbase + SMEM_P + t * TILE_BYTES + r * 128;
        float m_use = -INFINITY, l = 0.f;  // running max in log2 units (scaled)
        int n = 0;
        const int jb_t = t ? jb[1] : jb[0], je_t = t ? je[1] : je[0];
        for (int j = jb_t; j <= je_t; ++j, ++n) {
            mbar_wait(&s_full[t], n & 1);
            tc_fence_after();
            const int64_t k0 = (int64_t)j * BK;
            const bool need_mask = seg != nullptr || (k0 + BK - 1 > q0 + t * BQ);  // warp-uniform
            // pass 1: row max of raw scores (scale > 0 commutes with max)
            float mraw = -INFINITY;
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                uint32_t v[2][32];
                tmem_ld32(s_tm + h2 * 64, v[0]);
                tmem_ld32(s_tm + h2 * 64 + 32, v[1]);
                tmem_ld_wait();
                if (need_mask) {
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const int64_t key = k0 + h2 * 64 + c * 32 + i;
                            const float x = (key > q || key < start) ? -INFINITY : __uint_as_float(v[c][i]);
                            mraw = fmaxf(mraw, x);
                        }
                } else {
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int i = 0; i < 32; ++i) mraw = fmaxf(mraw, __uint_as_float(v[c][i]));
                }
            }
            const float mx = mraw * scale_log2;
            // lazy rescale; tcgen05.ld/st are warp-collective, so the O rescale runs warp-uniformly
            const bool grow = mx > m_use + RESCALE_THRESHOLD;
            const bool resc = grow && m_use != -INFINITY && n > 0;
            const float alpha = resc ? ex2(m_use - mx) : 1.f;
            if (__any_sync(0xffffffffu, resc)) {
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    uint32_t ov[32];
                    tmem_ld32(o_tm + c * 32, ov);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
                    tmem_st32(o_tm + c * 32, ov);
                }
                tmem_st_wait();
            }
            l *= alpha;
            if (grow) m_use = mx;
            const float nbase = m_use == -INFINITY ? 0.f : -m_use;
            // pass 2: p = 2^(s*scale_log2 - m) -> bf16 -> swizzled smem (K-major SW128 A operand)
            float rs = 0.f;
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                uint32_t v[2][32];
                tmem_ld32(s_tm + h2 * 64, v[0]);
                tmem_ld32(s_tm + h2 * 64 + 32, v[1]);
                tmem_ld_wait();
                const uint32_t reg = prow + h2 * 16384;  // keys [64*h2, 64*h2+64) -> column region h2
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    float p[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int col = 8 * k + e;
                        p[e] = ex2(fmaf(__uint_as_float(v[col >> 5][col & 31]), scale_log2, nbase));
                        if (need_mask) {
                            const int64_t key = k0 + h2 * 64 + col;
                            if (key > q || key < start) p[e] = 0.f;
                        }
                        rs += p[e];
                    }
                    sts128(reg + ((k ^ (r & 7)) << 4), pack_bf16x2(p[0], p[1]), pack_bf16x2(p[2], p[3]),
                           pack_bf16x2(p[4], p[5]), pack_bf16x2(p[6], p[7]));
                }
            }
            l += rs;
            fence_proxy_async();
            tc_fence_before();
            mbar_arrive(&p_full[t]);
        }
        // epilogue: O_t / l -> global, lse
        mbar_wait(&o_done[t], 0);
        tc_fence_after();
        const float inv = l > 0.f ? 1.f / l : 0.f;
        bf16* orow = o + (q * hq + h) * D;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t ov[32];
            tmem_ld32(o_tm + c * 32, ov);
            tmem_ld_wait();
            float f[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(ov[i]) * inv;
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint4 w;
                w.x = pack_bf16x2(f[8 * k + 0], f[8 * k + 1]);
                w.y = pack_bf16x2(f[8 * k + 2], f[8 * k + 3]);
                w.z = pack_bf16x2(f[8 * k + 4], f[8 * k + 5]);
                w.w = pack_bf16x2(f[8 * k + 6], f[8 * k + 7]);
                dst[k] = w;
            }
        }
        lse[(int64_t)h * s + q] = l > 0.f ? (m_use + __log2f(l)) * LN2 : -INFINITY;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}


// ===================================================================================== backward
// Generic SW128 descriptors for tiles made of 128 B-wide column regions `region` bytes apart.
__device__ __forceinline__ uint64_t kdesc_r(uint32_t tile, int kk, uint32_t region) {
    return make_sdesc_sw128(tile + (kk >> 2) * region + (kk & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t mndesc_r(uint32_t tile, int kk, uint32_t region) {
    return make_sdesc_sw128(tile + kk * 2048, region, 1024);
}

// ------------------------------------------------------------------ dQ pass
// CTA = (128-row q tile, q head).  Per 64-key block j (double-buffered in TMEM):
//   S_j = Q K_j^T, dP_j = dO V_j^T -> dS_j = P (dP - D) (bf16, smem, double-buffered) -> dQ += dS_j K_j.
// 8 elementwise warps (2 per TMEM lane quarter, each owning 32 of the 64 key columns), 6-slot K/V ring.
namespace dq {
constexpr int BKB = 64;
constexpr int Q_BYTES = 128 * D * 2;        // 32 KiB
constexpr int KV_BYTES = BKB * D * 2;       // 16 KiB (two 8 KiB regions)
constexpr int DS_BYTES = 128 * BKB * 2;     // 16 KiB (one region)
constexpr int NSL = 6;
constexpr int OFF_Q = 0, OFF_DO = Q_BYTES, OFF_DS = 2 * Q_BYTES, OFF_KV = OFF_DS + 2 * DS_BYTES;
constexpr int OFF_BAR = OFF_KV + NSL * KV_BYTES;
constexpr int SMEM = OFF_BAR + 256 + 1024;
}  // namespace dq

__global__ void __launch_bounds__(THREADS, 1)
    dq_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tkv,
                 const __grid_constant__ CUtensorMap tdo, int64_t s, int hq, int hkv, const int32_t* __restrict__ seg,
                 const float* __restrict__ lse2v, const float* __restrict__ Dv, float scale, bf16* __restrict__ dqkv) {
    using namespace dq;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* q_full = bar;
    uint64_t* kv_full = bar + 1;
    uint64_t* kv_empty = kv_full + NSL;
    uint64_t* s_full = kv_empty + NSL;  // [2]
    uint64_t* ds_full = s_full + 2;      // [2]
    uint64_t* dq_done = ds_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_done + 1);
    const int warp = warp_id(), lane = lane_id();
    const int nqb = (int)(s / 128);
    const int qb = nqb - 1 - (int)blockIdx.x;  // longest rows first
    const int h = blockIdx.y;
    const int kvh = h / (hq / hkv);
    const int64_t q0 = (int64_t)qb * 128;
    const int jb = seg ? (int)(seg[q0] / BKB) : 0;
    const int je = (int)((q0 + 127) / BKB);
    const int nblk = je - jb + 1;
    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < NSL; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&s_full[t], 1);
            mbar_init(&ds_full[t], 256);
        }
        mbar_init(dq_done, 1);
        fence_barrier_init();
    }
    if (warp == 8) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sbase = smem_u32(smem);
    if (warp == 9) {
        if (lane == 0) {
            mbar_arrive_expect_tx(q_full, 2 * Q_BYTES);
            for (int r = 0; r < 2; ++r) {
                tma_load_2d(&tq, q_full, smem + OFF_Q + r * 16384, h * D + 64 * r, (int)q0);
                tma_load_2d(&tdo, q_full, smem + OFF_DO + r * 16384, h * D + 64 * r, (int)q0);
            }
            for (int li = 0; li < 2 * nblk; ++li) {  // K_j, V_j, K_j+1, ...
                const int j = jb + li / 2, w = li & 1;
                const int slot = li % NSL;
                mbar_wait(&kv_empty[slot], ((li / NSL) & 1) ^ 1);
                mbar_arrive_expect_tx(&kv_full[slot], KV_BYTES);
                const int col = (hq + (w ? hkv : 0) + kvh) * D;
                for (int r = 0; r < 2; ++r)
                    tma_load_2d(&tkv, &kv_full[slot], smem + OFF_KV + slot * KV_BYTES + r * 8192, col + 64 * r,
                                j * BKB);
            }
        }
    } else if (warp == 8) {
        if (lane == 0) {
            constexpr uint32_t id_s = make_idesc_bf16(128, BKB, false, false);
            constexpr uint32_t id_q = make_idesc_bf16(128, D, false, true);
            mbar_wait(q_full, 0);
            const uint32_t qa = sbase + OFF_Q, da = sbase + OFF_DO;
            auto issue_sdp = [&](int it) {
                const int ks = (2 * it) % NSL, vs = (2 * it + 1) % NSL;
                mbar_wait(&kv_full[ks], ((2 * it) / NSL) & 1);
                mbar_wait(&kv_full[vs], ((2 * it + 1) / NSL) & 1);
                tc_fence_after();
                const uint32_t kb = sbase + OFF_KV + ks * KV_BYTES, vb = sbase + OFF_KV + vs * KV_BYTES;
                const uint32_t d_s = tmem + (it & 1) * 128;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    mma_bf16_ss(d_s, kdesc_r(qa, kk, 16384), kdesc_r(kb, kk, 8192), id_s, kk > 0);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    mma_bf16_ss(d_s + 64, kdesc_r(da, kk, 16384), kdesc_r(vb, kk, 8192), id_s, kk > 0);
                mma_commit(&s_full[it & 1]);
                mma_commit(&kv_empty[vs]);  // V_j only feeds dP
            };
            auto issue_dq = [&](int it) {
                mbar_wait(&ds_full[it & 1], (it >> 1) & 1);
                tc_fence_after();
                const int ks = (2 * it) % NSL;
                const uint32_t dsa = sbase + OFF_DS + (it & 1) * DS_BYTES;
                const uint32_t kb = sbase + OFF_KV + ks * KV_BYTES;
#pragma unroll
                for (int kk = 0; kk < BKB / 16; ++kk)
                    mma_bf16_ss(tmem + 256, kdesc_r(dsa, kk, 8192), mndesc_r(kb, kk, 8192), id_q, (it > 0 || kk > 0));
                mma_commit(&kv_empty[ks]);
            };
            issue_sdp(0);
            if (nblk > 1) issue_sdp(1);
            for (int it = 0; it < nblk; ++it) {
                issue_dq(it);
                if (it + 2 < nblk) issue_sdp(it + 2);
            }
            mma_commit(dq_done);
        }
    } else {
        const int sub = warp & 3, half = warp >> 2;
        const int r = sub * 32 + lane;
        const int64_t q = q0 + r;
        const int start = seg ? seg[q] : 0;
        const float nlse2 = -lse2v[(int64_t)h * s + q];  // -(lse * log2 e), precomputed
        const float Dq = Dv[(int64_t)h * s + q];
        const float sl2 = scale * LOG2E;
        const uint32_t lo = (uint32_t)(sub * 32) << 16;
        for (int it = 0; it < nblk; ++it) {
            const int b = it & 1;
            mbar_wait(&s_full[b], (it >> 1) & 1);
            tc_fence_after();
            uint32_t sv[32], dv[32];
            tmem_ld32(tmem + lo + b * 128 + half * 32, sv);
            tmem_ld32(tmem + lo + b * 128 + 64 + half * 32, dv);
            tmem_ld_wait();
            const int64_t k0 = (int64_t)(jb + it) * BKB + half * 32;
            const bool need_mask = seg != nullptr || (k0 + 31 > q0);
            const uint32_t dsrow = sbase + OFF_DS + b * DS_BYTES + r * 128;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float d8[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int i = 8 * k + e;
                    float p = ex2(fmaf(__uint_as_float(sv[i]), sl2, nlse2));
                    if (need_mask) {
                        const int64_t key = k0 + i;
                        if (key > q || key < start) p = 0.f;
                    }
                    d8[e] = p * (__uint_as_float(dv[i]) - Dq);
                }
                const int chunk = half * 4 + k;
                sts128(dsrow + ((chunk ^ (r & 7)) << 4), pack_bf16x2(d8[0], d8[1]), pack_bf16x2(d8[2], d8[3]),
                       pack_bf16x2(d8[4], d8[5]), pack_bf16x2(d8[6], d8[7]));
            }
            fence_proxy_async();
            tc_fence_before();
            mbar_arrive(&ds_full[b]);
        }
        mbar_wait(dq_done, 0);
        tc_fence_after();
        bf16* dst = dqkv + (q * (hq + 2 * hkv) + h) * D + half * 64;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
            uint32_t v[32];
            tmem_ld32(tmem + lo + 256 + half * 64 + c * 32, v);
            tmem_ld_wait();
            uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint4 w;
                w.x = pack_bf16x2(__uint_as_float(v[8 * k + 0]) * scale, __uint_as_float(v[8 * k + 1]) * scale);
                w.y = pack_bf16x2(__uint_as_float(v[8 * k + 2]) * scale, __uint_as_float(v[8 * k + 3]) * scale);
                w.z = pack_bf16x2(__uint_as_float(v[8 * k + 4]) * scale, __uint_as_float(v[8 * k + 5]) * scale);
                w.w = pack_bf16x2(__uint_as_float(v[8 * k + 6]) * scale, __uint_as_float(v[8 * k + 7]) * scale);
                d4[k] = w;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ dK / dV pass
// CTA = (128-key block, kv head).  Iterations over (q head of the GQA group, 64-row q block):
//   S^T = K Q^T, dP^T = V dO^T (TMEM, double-buffered) -> P^T, dS^T (bf16 smem, double-buffered)
//   -> dV += P^T dO, dK += dS^T Q (TMEM accumulators for the whole CTA).  No atomics.
namespace dkv {
constexpr int BQB = 64;
constexpr int KB_BYTES = 128 * D * 2;              // K or V block, 32 KiB
constexpr int QS_BYTES = BQB * D * 2;              // Q or dO tile, 16 KiB (two 8 KiB regions)
constexpr int PT_BYTES = 128 * BQB * 2;            // P^T / dS^T, 16 KiB
constexpr int NQS = 3;                                              // Q/dO ring stages
constexpr int OFF_K = 0, OFF_V = KB_BYTES, OFF_QS = 2 * KB_BYTES;  // NQS stages x (Q, dO)
constexpr int OFF_PT = OFF_QS + NQS * 2 * QS_BYTES;                 // [2 bufs] x (P^T, dS^T)
constexpr int OFF_BAR = OFF_PT + 4 * PT_BYTES;
constexpr int SMEM = OFF_BAR + 256 + 1024;
}  // namespace dkv

__global__ void __launch_bounds__(THREADS, 1)
    dkdv_tc_kernel(const __grid_constant__ CUtensorMap tkv, const __grid_constant__ CUtensorMap tq,
                   const __grid_constant__ CUtensorMap tdo, int64_t s, int hq, int hkv, const int32_t* __restrict__ seg,
                   const float* __restrict__ lse2v, const float* __restrict__ Dv, float scale, bf16* __restrict__ dqkv) {
    using namespace dkv;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* kv_full = bar;
    uint64_t* qs_full = bar + 1;          // [NQS]
    uint64_t* qs_empty = qs_full + NQS;   // [NQS]
    uint64_t* s_full = qs_empty + NQS;    // [2]
    uint64_t* pd_full = s_full + 2;       // [2]
    uint64_t* acc_done = pd_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);
    const int warp = warp_id(), lane = lane_id();
    const int nkb = (int)(s / 128);
    const int kb = (int)blockIdx.x;  // small kb = most work: launched first
    const int kvh = blockIdx.y;
    const int grp = hq / hkv;
    const int64_t k0 = (int64_t)kb * 128;
    (void)nkb;
    // visible q range: q >= k0 and (block-causal) start[q] <= k0 + 127
    const int qb_first = (int)(k0 / BQB);
    int qb_last = (int)((s - 1) / BQB);
    if (seg) {
        const int64_t klast = k0 + 127;
        int64_t lo = k0, hi = s - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) / 2;
            if (seg[mid] <= klast) lo = mid;
            else hi = mid - 1;
        }
        qb_last = (int)(lo / BQB);
    }
    const int nqb = qb_last - qb_first + 1;
    const int total = nqb * grp;
    if (threadIdx.x == 0) {
        mbar_init(kv_full, 1);
        for (int i = 0; i < NQS; ++i) {
            mbar_init(&qs_full[i], 1);
            mbar_init(&qs_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&pd_full[i], 256);
        }
        mbar_init(acc_done, 1);
        fence_barrier_init();
    }
    if (warp == 8) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sbase = smem_u32(smem);
    auto it_head = [&](int it) { return kvh * grp + it / nqb; };
    auto it_q0 = [&](int it) { return (int64_t)(qb_first + it % nqb) * BQB; };
    if (warp == 9) {
        if (lane == 0) {
            mbar_arrive_expect_tx(kv_full, 2 * KB_BYTES);
            for (int r = 0; r < 2; ++r) {
                tma_load_2d(&tkv, kv_full, smem + OFF_K + r * 16384, (hq + kvh) * D + 64 * r, (int)k0);
                tma_load_2d(&tkv, kv_full, smem + OFF_V + r * 16384, (hq + hkv + kvh) * D + 64 * r, (int)k0);
            }
            for (int it = 0; it < total; ++it) {
                const int st = it % NQS;
                mbar_wait(&qs_empty[st], ((it / NQS) & 1) ^ 1);
                mbar_arrive_expect_tx(&qs_full[st], 2 * QS_BYTES);
                const int hh = it_head(it);
                const int qq = (int)it_q0(it);
                uint8_t* base = smem + OFF_QS + st * 2 * QS_BYTES;
                for (int r = 0; r < 2; ++r) {
                    tma_load_2d(&tq, &qs_full[st], base + r * 8192, hh * D + 64 * r, qq);
                    tma_load_2d(&tdo, &qs_full[st], base + QS_BYTES + r * 8192, hh * D + 64 * r, qq);
                }
            }
        }
    } else if (warp == 8) {
        if (lane == 0) {
            constexpr uint32_t id_s = make_idesc_bf16(128, BQB, false, false);
            constexpr uint32_t id_a = make_idesc_bf16(128, D, false, true);
            mbar_wait(kv_full, 0);
            const uint32_t ka = sbase + OFF_K, va = sbase + OFF_V;
            auto issue_sdp = [&](int it) {
                const int st = it % NQS;
                mbar_wait(&qs_full[st], (it / NQS) & 1);
                tc_fence_after();
                const uint32_t qb_ = sbase + OFF_QS + st * 2 * QS_BYTES, dob = qb_ + QS_BYTES;
                const uint32_t d_s = tmem + (it & 1) * 128;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    mma_bf16_ss(d_s, kdesc_r(ka, kk, 16384), kdesc_r(qb_, kk, 8192), id_s, kk > 0);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    mma_bf16_ss(d_s + 64, kdesc_r(va, kk, 16384), kdesc_r(dob, kk, 8192), id_s, kk > 0);
                mma_commit(&s_full[it & 1]);
            };
            auto issue_acc = [&](int it) {
                const int b = it & 1, st = it % NQS;
                mbar_wait(&pd_full[b], (it >> 1) & 1);
                tc_fence_after();
                const uint32_t pt = sbase + OFF_PT + b * 2 * PT_BYTES, dst_ = pt + PT_BYTES;
                const uint32_t qb_ = sbase + OFF_QS + st * 2 * QS_BYTES, dob = qb_ + QS_BYTES;
#pragma unroll
                for (int kk = 0; kk < BQB / 16; ++kk)
                    mma_bf16_ss(tmem + 256, kdesc_r(pt, kk, 8192), mndesc_r(dob, kk, 8192), id_a, (it > 0 || kk > 0));
#pragma unroll
                for (int kk = 0; kk < BQB / 16; ++kk)
                    mma_bf16_ss(tmem + 384, kdesc_r(dst_, kk, 8192), mndesc_r(qb_, kk, 8192), id_a, (it > 0 || kk > 0));
                mma_commit(&qs_empty[st]);
            };
            if (total > 0) issue_sdp(0);
            if (total > 1) issue_sdp(1);
            for (int it = 0; it < total; ++it) {
                issue_acc(it);
                if (it + 2 < total) issue_sdp(it + 2);
            }
            mma_commit(acc_done);
        }
    } else {
        // elementwise: warp w: TMEM lanes (w&3)*32.., columns half (w>>2)*32 of the 64 q columns
        const int sub = warp & 3, half = warp >> 2;
        const int r = sub * 32 + lane;  // key row
        const int64_t key = k0 + r;
        const uint32_t lo = (uint32_t)(sub * 32) << 16;
        const float sl2 = scale * LOG2E;
        for (int it = 0; it < total; ++it) {
            const int b = it & 1;
            const int hh = it_head(it);
            const int64_t qq = it_q0(it) + half * 32;
            mbar_wait(&s_full[b], (it >> 1) & 1);
            tc_fence_after();
            uint32_t sv[32], dv[32];
            tmem_ld32(tmem + lo + b * 128 + half * 32, sv);
            tmem_ld32(tmem + lo + b * 128 + 64 + half * 32, dv);
            tmem_ld_wait();
            const float4* l4 = reinterpret_cast<const float4*>(lse2v + (int64_t)hh * s + qq);
            const float4* d4 = reinterpret_cast<const float4*>(Dv + (int64_t)hh * s + qq);
            const bool need_mask = seg != nullptr || qq < k0 + 127;
            const uint32_t prow = sbase + OFF_PT + b * 2 * PT_BYTES + r * 128;
            const uint32_t drow = prow + PT_BYTES;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float4 la = __ldg(l4 + 2 * k), lb = __ldg(l4 + 2 * k + 1);
                const float4 da = __ldg(d4 + 2 * k), db = __ldg(d4 + 2 * k + 1);
                const float lv[8] = {la.x, la.y, la.z, la.w, lb.x, lb.y, lb.z, lb.w};
                const float dd[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
                float p8[8], s8[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int i = 8 * k + e;
                    float p = ex2(fmaf(__uint_as_float(sv[i]), sl2, -lv[e]));
                    if (need_mask) {
                        const int64_t qi = qq + i;
                        if (key > qi || (seg && key < seg[qi])) p = 0.f;
                    }
                    p8[e] = p;
                    s8[e] = p * (__uint_as_float(dv[i]) - dd[e]);
                }
                const int chunk = half * 4 + k;
                const uint32_t off = (uint32_t)((chunk ^ (r & 7)) << 4);
                sts128(prow + off, pack_bf16x2(p8[0], p8[1]), pack_bf16x2(p8[2], p8[3]), pack_bf16x2(p8[4], p8[5]),
                       pack_bf16x2(p8[6], p8[7]));
                sts128(drow + off, pack_bf16x2(s8[0], s8[1]), pack_bf16x2(s8[2], s8[3]), pack_bf16x2(s8[4], s8[5]),
                       pack_bf16x2(s8[6], s8[7]));
            }
            fence_proxy_async();
            tc_fence_before();
            mbar_arrive(&pd_full[b]);
        }
        // epilogue: half 0 writes dV, half 1 writes dK (scaled)
        mbar_wait(acc_done, 0);
        tc_fence_after();
        const int64_t rs = (int64_t)(hq + 2 * hkv) * D;
        bf16* dst = dqkv + key * rs + (int64_t)(half ? (hq + kvh) : (hq + hkv + kvh)) * D;
        const float mul = half ? scale : 1.f;
        const uint32_t acc_tm = tmem + lo + (half ? 384 : 256);
        if (total == 0) {
            uint4* d4 = reinterpret_cast<uint4*>(dst);
            for (int k = 0; k < D / 8; ++k) d4[k] = make_uint4(0, 0, 0, 0);
        } else {
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                uint32_t v[32];
                tmem_ld32(acc_tm + c * 32, v);
                tmem_ld_wait();
                uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    uint4 w;
                    w.x = pack_bf16x2(__uint_as_float(v[8 * k + 0]) * mul, __uint_as_float(v[8 * k + 1]) * mul);
                    w.y = pack_bf16x2(__uint_as_float(v[8 * k + 2]) * mul, __uint_as_float(v[8 * k + 3]) * mul);
                    w.z = pack_bf16x2(__uint_as_float(v[8 * k + 4]) * mul, __uint_as_float(v[8 * k + 5]) * mul);
                    w.w = pack_bf16x2(__uint_as_float(v[8 * k + 6]) * mul, __uint_as_float(v[8 * k + 7]) * mul);
                    d4[k] = w;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace fatc

bool attn_fwd_tc(const void* qkv, int64_t s, int hq, int hkv, int d, const int32_t* seg, float scale, void* o,
                 float* lse, cudaStream_t st) {
    if (d != fatc::D || s % 256 != 0) return false;
    const int64_t width = (int64_t)(hq + 2 * hkv) * d;
    CUtensorMap tm = make_tmap_bf16_2d(qkv, (uint64_t)width, (uint64_t)s, (uint64_t)width, 64, 128);
    auto k = fatc::fwd_tc_kernel;
    static bool attr = false;
    if (!attr) {
        SPT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, fatc::SMEM_BYTES));
        attr = true;
    }
    dim3 grid((unsigned)(s / 256), (unsigned)hq);
    k<<<grid, fatc::THREADS, fatc::SMEM_BYTES, st>>>(tm, s, hq, hkv, seg, scale * fatc::LOG2E, (bf16*)o, lse);
    count_launch("attn_fwd_tc");
    SPT_CUDA(cudaGetLastError());
    return true;
}

// Deterministic tcgen05 backward (d = 128, s % 256 == 0).  Dv = rowsum(dO * O) must be precomputed.
bool attn_bwd_tc(const void* qkv, const void* dout, const float* lse2, const float* Dv, int64_t s, int hq, int hkv,
                 int d, const int32_t* seg, float scale, void* dqkv, cudaStream_t st) {
    if (d != fatc::D || s % 256 != 0) return false;
    const int64_t width = (int64_t)(hq + 2 * hkv) * d;
    CUtensorMap t128 = make_tmap_bf16_2d(qkv, (uint64_t)width, (uint64_t)s, (uint64_t)width, 64, 128);
    CUtensorMap t64 = make_tmap_bf16_2d(qkv, (uint64_t)width, (uint64_t)s, (uint64_t)width, 64, 64);
    CUtensorMap do128 = make_tmap_bf16_2d(dout, (uint64_t)hq * d, (uint64_t)s, (uint64_t)hq * d, 64, 128);
    CUtensorMap do64 = make_tmap_bf16_2d(dout, (uint64_t)hq * d, (uint64_t)s, (uint64_t)hq * d, 64, 64);
    static bool attr = false;
    if (!attr) {
        SPT_CUDA(cudaFuncSetAttribute(fatc::dq_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, fatc::dq::SMEM));
        SPT_CUDA(cudaFuncSetAttribute(fatc::dkdv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fatc::dkv::SMEM));
        attr = true;
    }
    fatc::dkdv_tc_kernel<<<dim3((unsigned)(s / 128), (unsigned)hkv), fatc::THREADS, fatc::dkv::SMEM, st>>>(
        t128, t64, do64, s, hq, hkv, seg, lse2, Dv, scale, (bf16*)dqkv);
    count_launch("attn_dkdv_tc");
    SPT_CUDA(cudaGetLastError());
    fatc::dq_tc_kernel<<<dim3((unsigned)(s / 128), (unsigned)hq), fatc::THREADS, fatc::dq::SMEM, st>>>(
        t128, t64, do128, s, hq, hkv, seg, lse2, Dv, scale, (bf16*)dqkv);
    count_launch("attn_dq_tc");
    SPT_CUDA(cudaGetLastError());
    return true;
}

}  // namespace spt
