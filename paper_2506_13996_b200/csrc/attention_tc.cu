// tcgen05 / TMEM / TMA flash attention for head_dim 128 (K3 forward, K4 backward), Blackwell-native.
//
// All kernels: 10 warps — 8 elementwise/softmax warps (thread = one TMEM lane = one matrix row),
// warp 8 = MMA issuer (one lane) + TMEM owner, warp 9 = TMA producer.  Scores are computed by
// tcgen05.mma into TMEM, read with tcgen05.ld, masked lazily (causal / block-causal runs,
// SPEC.md:243-251), and the probabilities go back either into TMEM (forward: P aliases the consumed
// score columns and is the A operand of the PV MMA) or into swizzled smem (backward).  Online softmax
// uses a lazy rescale: O is only rescaled in TMEM when the running max grows by > 2^8.
#include <algorithm>
#include <string>
#include <type_traits>

#include "common.h"
#include "launch.h"
#include "sm100.cuh"

namespace spt {
namespace fatc {

constexpr int D = 128;
constexpr int BQ = 128;   // rows per query tile
constexpr int THREADS = 320;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;
constexpr float RESCALE_THRESHOLD = 8.f;  // log2 units
// packed sequences: a tile pair whose first sample started at least this many keys before its end runs on
// the 128-key forward, the rest on the 64-key forward (short samples straddle 128-key blocks)
constexpr int64_t FWD_LONG_KEYS = 4096;

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 2^x on the FMA pipe (Cody-Waite split + degree-3 fit of 2^f on [-1/2, 1/2], max rel err 1.5e-4, far
// below the bf16 rounding of P).  The forward softmax runs a fraction of its exponentials through this so
// the MUFU pipe (16 ex2/clk/SM, exactly the rate a 128x64 score tile needs at full tensor throughput) stops
// being the co-bottleneck.  Inputs below -126 (masked -inf) return exactly 0 like ex2.approx.ftz.
__device__ __forceinline__ float ex2_poly(float x) {
    const float xc = fmaxf(x, -127.f);
    const float t = xc + 12582912.f;  // 1.5 * 2^23: round(xc) lands in the low mantissa bits of t
    const float rf = t - 12582912.f;
    const float f = xc - rf;
    const float p = fmaf(fmaf(fmaf(0.05508868f, f, 0.24260405f), f, 0.69327624f), f, 0.99992894f);
    const float y = __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
    return x < -126.f ? 0.f : y;
}

// 2^x for a PAIR on the FMA pipe with packed f32x2 arithmetic (FADD2 / FFMA2: half the instructions of two
// ex2_poly calls): the same Cody-Waite split and degree-3 fit, exponent inserted by an integer add.  Inputs are
// clamped to >= -126 so the inserted exponent never underflows into the sign (the result there is ~1e-38, not
// exactly 0: callers use it only on unmasked score blocks, where masked -inf never occurs).
__device__ __forceinline__ void ex2_poly2(float x0, float x1, float& y0, float& y1) {
    const uint64_t big = f2pack(12582912.f, 12582912.f);  // 1.5 * 2^23
    const uint64_t xc = f2pack(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
    const uint64_t t = fadd2(xc, big);
    const uint64_t f = fsub2(xc, fsub2(t, big));
    uint64_t p = ffma2(f2pack(0.05508868f, 0.05508868f), f, f2pack(0.24260405f, 0.24260405f));
    p = ffma2(p, f, f2pack(0.69327624f, 0.69327624f));
    p = ffma2(p, f, f2pack(0.99992894f, 0.99992894f));
    float p0, p1, t0, t1;
    f2unpack(p, p0, p1);
    f2unpack(t, t0, t1);
    y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
    y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

#ifndef SPT_DQ_TMEM_DEFAULT
#define SPT_DQ_TMEM_DEFAULT 1
#endif
#ifndef SPT_DQ_MC_DEFAULT
#define SPT_DQ_MC_DEFAULT 0
#endif
#ifndef SPT_ATTN_BWD_DEFAULT
#define SPT_ATTN_BWD_DEFAULT 0
#endif
#ifndef SPT_DKDV_MC_DEFAULT
#define SPT_DKDV_MC_DEFAULT 1
#endif
#ifndef SPT_FWD_ORDER
#define SPT_FWD_ORDER 0
#endif
#ifdef SPT_DQ_PROF
__device__ unsigned long long g_dq_prof[8];  // [0] MMA wait kv, [1] MMA wait ds_full, [2] elem wait s_full,
                                             // [3] elem busy, [4] MMA total, [5] CTAs, [6] iterations
#define DQP_T0() const long long _t0 = clock64()
#define DQP_ADD(i) atomicAdd(&g_dq_prof[i], (unsigned long long)(clock64() - _t0))
#else
#define DQP_T0()
#define DQP_ADD(i)
#endif
#ifndef SPT_DQ_POLY_EVERY
#define SPT_DQ_POLY_EVERY 0
#endif
#ifndef SPT_FWD_POLY_EVERY
#define SPT_FWD_POLY_EVERY 0  // N > 0: every N-th exponential pair goes through ex2_poly (measured slower: the
                              // forward softmax is issue-bound, not MUFU-bound, on B200)
#endif

// Grid-order remap for the Q-outer kernels (grid = (q head, row block), row blocks longest first).
// CTAs are dispatched in order of groups of `kvg` kv heads (slowest), then row block, then the q heads of
// the group.  kvg >= hkv: q heads fastest — one wave streams the K/V of every kv head.  kvg = 1: kv-major —
// consecutive waves share one kv head's K/V, which then stays in L2 instead of being re-read from HBM by
// every wave, at the price of more CTAs reading the same lines at once.
__device__ __forceinline__ void grid_head_row(int kvg, int hq, int hkv, int& h, int& yb) {
    if (kvg >= hkv) {
        h = blockIdx.x;
        yb = blockIdx.y;
        return;
    }
    const int hg = kvg * (hq / hkv);  // q heads per full group; the last group may be partial
    const int L = blockIdx.x + blockIdx.y * gridDim.x;
    const int per = hg * gridDim.y;
    const int g = L / per, rem = L - g * per;
    const int hgl = min(hg, hq - g * hg);
    yb = rem / hgl;
    h = g * hg + (rem - yb * hgl);
}

// 2^x0, 2^x1 with one ex2.approx.f16x2 (inputs rounded to f16: |x| <= 2^-11 relative, results f16-accurate,
// 2^-24 flush; the forward uses x <= RESCALE_THRESHOLD, so no overflow), widened back to fp32.
__device__ __forceinline__ void ex2_f16x2(float x0, float x1, float& p0, float& p1) {
    uint32_t h, e;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x1), "f"(x0));
    asm("ex2.approx.f16x2 %0, %1;" : "=r"(e) : "r"(h));
    asm("{\n\t.reg .f16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\tcvt.f32.f16 %0, lo;\n\tcvt.f32.f16 %1, hi;\n\t}"
        : "=f"(p0), "=f"(p1)
        : "r"(e));
}

__device__ __forceinline__ void lds128(uint32_t addr, float& a, float& b, float& c, float& d) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "r"(addr));
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

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

// Backward kernels: 16 elementwise warps (4 per TMEM lane quarter, 16 of the 64 block columns each),
// warp 16 = MMA issuer / TMEM owner, warp 17 = TMA producer.
constexpr int BW_NEW = 16;
constexpr int BW_THREADS = (BW_NEW + 2) * 32;
constexpr int BW_MMA = BW_NEW, BW_TMA = BW_NEW + 1;

// Generic SW128 descriptors for tiles made of 128 B-wide column regions `region` bytes apart.
// The start-address field is the low 14 bits (16-byte units); smem offsets < 256 KiB never carry out,
// so a K step is a plain add on a loop-invariant base descriptor (keeps the single MMA-issuing thread
// at ~1 uniform op per tcgen05.mma — the N=64 score MMAs only last ~32 tensor cycles each).
__device__ __forceinline__ uint64_t kdesc_r(uint32_t tile, int kk, uint32_t region) {
    return make_sdesc_sw128(tile, 16, 1024) + (uint64_t)(((kk >> 2) * region + (kk & 3) * 32) >> 4);
}
__device__ __forceinline__ uint64_t mndesc_r(uint32_t tile, int kk, uint32_t region) {
    return make_sdesc_sw128(tile, region, 1024) + (uint64_t)((kk * 2048) >> 4);
}

// ------------------------------------------------------------------ forward
// CTA = (pair of consecutive 128-row query tiles, q head).  64-key blocks.  TMEM (512 columns):
//   tile t: S_t[0] | S_t[1] (64 columns each, double-buffered) | O_t (128)  at t*256.
// P_t (bf16) is written into the consumed S_t[b] columns and fed to the PV MMA from TMEM.
// MMA order per key block j: PV0(j) PV1(j) S0(j+2) S1(j+2): the score MMAs for block j+2 run while
// the softmax of block j+1 executes, so softmax and tensor core overlap within a tile too.
namespace fw {
constexpr int BKB = 64;
constexpr int Q_BYTES = BQ * D * 2;    // 32 KiB per tile
constexpr int KV_BYTES = BKB * D * 2;  // 16 KiB per K or V block (two 8 KiB regions)
constexpr int NSL = 10;
constexpr int OFF_Q = 0, OFF_KV = 2 * Q_BYTES;
constexpr int OFF_BAR = OFF_KV + NSL * KV_BYTES;
constexpr int SMEM = OFF_BAR + 512 + 1024;
}  // namespace fw

__global__ void __launch_bounds__(THREADS, 1)
    fwd_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tkv, int64_t s, int hq,
                  int hkv, const int32_t* __restrict__ seg, float scale_log2, bf16* __restrict__ o,
                  float* __restrict__ lse, int kvg, int filter) {
    using namespace fw;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* q_full = bar;
    uint64_t* kv_full = bar + 1;
    uint64_t* kv_empty = kv_full + NSL;
    uint64_t* s_full = kv_empty + NSL;  // [t*2 + b]
    uint64_t* p_full = s_full + 4;      // [t*2 + b]  per buffer: the softmax may run 2 blocks ahead
    uint64_t* pv_done = p_full + 4;     // [t]
    uint64_t* o_done = pv_done + 2;     // [t]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

    const int warp = warp_id(), lane = lane_id();
    const int npairs = (int)((s + 2 * BQ - 1) / (2 * BQ));  // s % 256 == 128: the last pair holds one tile
    // grid = (q head, query-tile pair): heads vary fastest so one wave of CTAs streams the K/V of every kv
    // head at once instead of 148 CTAs hammering the same K/V lines (L2-slice hot spot); longest rows first
    int h, yb;
    grid_head_row(kvg, hq, hkv, h, yb);
    const int pair = npairs - 1 - yb;
    const int kvh = h / (hq / hkv);
    const int64_t q0 = (int64_t)pair * 2 * BQ;
    const bool has1 = q0 + BQ < s;  // second query tile present
    const int jb0 = seg ? (int)(seg[q0] / BKB) : 0, jb1 = (seg && has1) ? (int)(seg[q0 + BQ] / BKB) : 0;
    const int je0 = (int)((q0 + BQ - 1) / BKB), je1 = has1 ? (int)((q0 + 2 * BQ - 1) / BKB) : -1;
    const int jlo = jb0, jhi = has1 ? je1 : je0;
    if (filter) {  // packed hybrid: this launch handles only the long (1) or short (2) tile pairs
        const bool longp = q0 + 2 * BQ - (seg ? seg[q0] : 0) >= FWD_LONG_KEYS;
        if ((filter == 1) != longp) return;  // whole CTA, before any barrier / TMEM allocation
    }  // jb0 <= jb1 (starts are monotone), je0 < je1

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < NSL; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 4; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 128);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&pv_done[t], 1);
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
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // provably warp-uniform: descriptor math stays in uniform registers
    const uint32_t sbase = smem_u32(smem);

    if (warp == 9) {
        if (lane == 0) {
            tma_prefetch_desc(&tq);
            tma_prefetch_desc(&tkv);
            mbar_arrive_expect_tx(q_full, 2 * Q_BYTES);
            for (int t = 0; t < 2; ++t)
                for (int r = 0; r < 2; ++r)
                    tma_load_2d(&tq, q_full, smem + OFF_Q + t * Q_BYTES + r * 16384, h * D + 64 * r,
                                (int)(q0 + t * BQ));
            const int nload = 2 * (jhi - jlo + 1);
            for (int li = 0; li < nload; ++li) {
                const int j = jlo + li / 2, w = li & 1;
                const int slot = li % NSL;
                mbar_wait(&kv_empty[slot], ((li / NSL) & 1) ^ 1);
                mbar_arrive_expect_tx(&kv_full[slot], KV_BYTES);
                const int col = (hq + (w ? hkv : 0) + kvh) * D;
                for (int r = 0; r < 2; ++r)
                    tma_load_2d(&tkv, &kv_full[slot], smem + OFF_KV + slot * KV_BYTES + r * 8192, col + 64 * r, j * BKB);
            }
        }
    } else if (warp == 8) {
        {  // whole warp, converged; elect.sync inside the MMA/commit wrappers picks the issuing lane
            constexpr uint32_t idesc_s = make_idesc_bf16(BQ, BKB, false, false);
            constexpr uint32_t idesc_o = make_idesc_bf16(BQ, D, false, true);
            mbar_wait(q_full, 0);
            const int jb[2] = {jb0, jb1}, je[2] = {je0, je1};
            int pv_count[2] = {0, 0};
            auto uses = [&](int t, int j) { return j >= jb[t] && j <= je[t]; };
            auto slot = [&](int j, int w) { return (2 * (j - jlo) + w) % NSL; };
            auto phase = [&](int j, int w) { return (uint32_t)(((2 * (j - jlo) + w) / NSL) & 1); };
            auto issue_s = [&](int t, int j) {
                mbar_wait(&kv_full[slot(j, 0)], phase(j, 0));
                tc_fence_after();
                const int b = (j - jb[t]) & 1;
                const uint32_t qa = sbase + OFF_Q + t * Q_BYTES;
                const uint32_t kb = sbase + OFF_KV + slot(j, 0) * KV_BYTES;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    mma_bf16_ss_w(tmem + t * 256 + b * 64, kdesc_r(qa, kk, 16384), kdesc_r(kb, kk, 8192), idesc_s, kk > 0);
                mma_commit_w(&s_full[t * 2 + b]);
            };
            auto issue_pv = [&](int t, int j) {
#ifdef SPT_WATCHDOG
                {
                    long long sp = 0;
                    while (!mbar_try_wait(smem_u32(&p_full[t * 2 + ((j - jb[t]) & 1)]), ((j - jb[t]) >> 1) & 1)) {
                        if (++sp == (1ll << 23)) {
                            volatile int* dbg = reinterpret_cast<volatile int*>(tmem_slot + 4);
                            printf("[fwd dbg] blk (%d,%d) waiting p_full[%d] j=%d; progress t0=(%d,%d) t1=(%d,%d)\n",
                                   blockIdx.x, blockIdx.y, t, j, dbg[0], dbg[1], dbg[2], dbg[3]);
                        }
                    }
                }
#endif
                mbar_wait(&p_full[t * 2 + ((j - jb[t]) & 1)], ((j - jb[t]) >> 1) & 1);
                mbar_wait(&kv_full[slot(j, 1)], phase(j, 1));
                tc_fence_after();
                const int b = (j - jb[t]) & 1;
                const uint32_t vb = sbase + OFF_KV + slot(j, 1) * KV_BYTES;
#pragma unroll
                for (int kk = 0; kk < BKB / 16; ++kk)
                    mma_bf16_ts_w(tmem + t * 256 + 128, tmem + t * 256 + b * 64 + kk * 8, mndesc_r(vb, kk, 8192), idesc_o,
                                (pv_count[t] > 0 || kk > 0));
                mma_commit_w(&pv_done[t]);
                ++pv_count[t];
            };
            // prologue: score MMAs for the first two blocks of each tile
            for (int j = jlo; j <= min(jlo + 1, jhi); ++j) {
                if (uses(0, j)) issue_s(0, j);
                if (uses(1, j)) issue_s(1, j);
                mma_commit_w(&kv_empty[slot(j, 0)]);  // K_j consumed by both tiles' S MMAs
            }
#if SPT_FWD_ORDER == 1
            // per tile: PV_t(j) then S_t(j+2) right away, so tile 0's next scores do not wait for tile 1's softmax
            for (int j = jlo; j <= jhi; ++j) {
                const bool more = j + 2 <= jhi;
                if (uses(0, j)) issue_pv(0, j);
                if (more && uses(0, j + 2)) issue_s(0, j + 2);
                if (uses(1, j)) issue_pv(1, j);
                mma_commit_w(&kv_empty[slot(j, 1)]);  // V_j consumed
                if (more) {
                    if (uses(1, j + 2)) issue_s(1, j + 2);
                    mma_commit_w(&kv_empty[slot(j + 2, 0)]);  // K_{j+2} consumed by both tiles
                }
            }
#else
            for (int j = jlo; j <= jhi; ++j) {
                if (uses(0, j)) issue_pv(0, j);
                if (uses(1, j)) issue_pv(1, j);
                mma_commit_w(&kv_empty[slot(j, 1)]);  // V_j consumed
                if (j + 2 <= jhi) {
                    if (uses(0, j + 2)) issue_s(0, j + 2);
                    if (uses(1, j + 2)) issue_s(1, j + 2);
                    mma_commit_w(&kv_empty[slot(j + 2, 0)]);
                }
            }
#endif
            mma_commit_w(&o_done[0]);
            mma_commit_w(&o_done[1]);
        }
    } else {
        // ---------------- softmax warpgroups (thread = query row)
        const int t = warp >> 2;
        const int sub = warp & 3;
        const int r = sub * 32 + lane;
        const int64_t q = q0 + t * BQ + r;
        const bool row_ok = q < s;  // false only for the absent second tile of a half pair
        const int start = (seg && row_ok) ? seg[q] : 0;
        const uint32_t lane_off = (uint32_t)(sub * 32) << 16;
        const uint32_t t_tm = tmem + lane_off + t * 256;
        const uint32_t o_tm = t_tm + 128;
        const int jb_t = t ? jb1 : jb0, je_t = t ? je1 : je0;
        float m_use = -INFINITY, l = 0.f;  // running max in log2 units (scaled)
        for (int j = jb_t; j <= je_t; ++j) {
            const int n = j - jb_t, b = n & 1;
            const uint32_t s_tm = t_tm + b * 64;
#ifdef SPT_WATCHDOG
            volatile int* dbg = reinterpret_cast<volatile int*>(tmem_slot + 4);
            if (r == 0) { dbg[2 * t] = j; dbg[2 * t + 1] = 1; }
#endif
            mbar_wait(&s_full[t * 2 + b], (n >> 1) & 1);
#ifdef SPT_WATCHDOG
            if (r == 0) dbg[2 * t + 1] = 2;
#endif
            tc_fence_after();
            const int64_t k0 = (int64_t)j * BKB;
            // warp-uniform: causal diagonal, or (packed) some row of this warp starts its sample inside the block
            const bool need_mask = (k0 + BKB - 1 > q0 + t * BQ) || (seg != nullptr && __any_sync(0xffffffffu, start > k0));
            uint32_t v[2][32];
            tmem_ld32(s_tm, v[0]);
            tmem_ld32(s_tm + 32, v[1]);
            tmem_ld_wait();
            // row max over the 64 columns: 8 independent partial maxima (short dependency chains; the two
            // softmax warps per SMSP cannot hide a 64-long serial FMNMX chain)
            float mp[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) mp[u] = -INFINITY;
            if (need_mask) {
                const int hi = (int)(q - k0), lo_ = start - (int)k0;  // keep columns lo_ <= i <= hi
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int col = c * 32 + i;
                        if (col > hi || col < lo_) v[c][i] = __float_as_uint(-INFINITY);
                    }
            }
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int i = 0; i < 32; i += 2)
                    mp[(c * 32 + i) >> 1 & 7] =
                        fmax3(mp[(c * 32 + i) >> 1 & 7], __uint_as_float(v[c][i]), __uint_as_float(v[c][i + 1]));
            const float mraw = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])),
                                     fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
            const float mx = mraw * scale_log2;
            // lazy rescale (warp-uniform: tcgen05.ld/st are warp-collective); needs PV_t(j-1) complete
            const bool grow = mx > m_use + RESCALE_THRESHOLD;
            const bool resc = grow && m_use != -INFINITY && n > 0;
            const float alpha = resc ? ex2(m_use - mx) : 1.f;
            if (__any_sync(0xffffffffu, resc)) {
                mbar_wait(&pv_done[t], (n - 1) & 1);
                tc_fence_after();
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    uint32_t ov[32];
                    tmem_ld32(o_tm + c * 32, ov);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
                    tmem_st32(o_tm + c * 32, ov);
                }
            }
            l *= alpha;
            if (grow) m_use = mx;
            const float nbase = m_use == -INFINITY ? 0.f : -m_use;
            uint32_t pw[32];
            const uint64_t sc2 = f2pack(scale_log2, scale_log2), nb2 = f2pack(nbase, nbase);
            uint64_t rs2[4];  // 4 independent packed row-sum accumulators (short FADD2 chains)
#pragma unroll
            for (int u = 0; u < 4; ++u) rs2[u] = f2pack(0.f, 0.f);
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const int c0 = 2 * k;
                const uint64_t x2 = ffma2(f2pack(__uint_as_float(v[c0 >> 5][c0 & 31]), __uint_as_float(v[c0 >> 5][(c0 + 1) & 31])),
                                          sc2, nb2);
                float x0, x1;
                f2unpack(x2, x0, x1);
                const bool poly = SPT_FWD_POLY_EVERY > 0 && (k % (SPT_FWD_POLY_EVERY > 0 ? SPT_FWD_POLY_EVERY : 1)) ==
                                                                (SPT_FWD_POLY_EVERY > 0 ? SPT_FWD_POLY_EVERY - 1 : 0);
                const float p0 = poly ? ex2_poly(x0) : ex2(x0);
                const float p1 = poly ? ex2_poly(x1) : ex2(x1);
                rs2[k & 3] = fadd2(rs2[k & 3], f2pack(p0, p1));
                pw[k] = pack_bf16x2(p0, p1);
            }
            float rs0, rs1;
            f2unpack(fadd2(fadd2(rs2[0], rs2[1]), fadd2(rs2[2], rs2[3])), rs0, rs1);
            const float rs = rs0 + rs1;
            l += rs;
#ifdef SPT_WATCHDOG
            if (r == 0) dbg[2 * t + 1] = 3;
#endif
            tmem_st32(s_tm, pw);  // packed P over the consumed S columns [0, 32)
            tmem_st_wait();
#ifdef SPT_WATCHDOG
            if (r == 0) dbg[2 * t + 1] = 4;
#endif
            tc_fence_before();
            mbar_arrive(&p_full[t * 2 + b]);
        }
        // epilogue: O_t / l -> global, lse
        mbar_wait(&o_done[t], 0);
        tc_fence_after();
        if (t == 1 && !has1) goto fwd_done;  // warp-uniform: the whole tile is absent
        {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        bf16* orow = o + (q * hq + h) * D;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t ov[32];
            tmem_ld32(o_tm + c * 32, ov);
            tmem_ld_wait();
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint4 w;
                w.x = pack_bf16x2(__uint_as_float(ov[8 * k + 0]) * inv, __uint_as_float(ov[8 * k + 1]) * inv);
                w.y = pack_bf16x2(__uint_as_float(ov[8 * k + 2]) * inv, __uint_as_float(ov[8 * k + 3]) * inv);
                w.z = pack_bf16x2(__uint_as_float(ov[8 * k + 4]) * inv, __uint_as_float(ov[8 * k + 5]) * inv);
                w.w = pack_bf16x2(__uint_as_float(ov[8 * k + 6]) * inv, __uint_as_float(ov[8 * k + 7]) * inv);
                dst[k] = w;
            }
        }
        lse[(int64_t)h * s + q] = l > 0.f ? (m_use + __log2f(l)) * LN2 : -INFINITY;
        }
    fwd_done:;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        __syncwarp();  // role branches diverged lane 0; dealloc is warp-collective (.sync.aligned)
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// Forward with 128-key blocks (fwd_tc128_kernel): same CTA / TMEM shape as fwd_tc_kernel (two 128-row query
// tiles, 256 TMEM columns each), but each tile's 128 S columns hold ONE 128-key score block instead of two
// double-buffered 64-key blocks.  The score MMA is then M=128 N=128 — full tensor rate with both operands in
// smem (64 of 64 cycles), where the N=64 form takes 48 of 32 (tools/micro/mma_rate.cu) — and per-block
// barrier / rescale overheads halve.  The price is a single S buffer per tile: S_t(j+1) is issued right after
// PV_t(j) (which consumes P_t(j) from the same columns), so the two tiles ping-pong: one tile's softmax runs
// under the other tile's MMAs.  MMA order per block j: PV0(j) S0(j+1) PV1(j) S1(j+1).
namespace fw2 {
constexpr int BKB = 128;
#ifndef SPT_FWD2_NPART
#define SPT_FWD2_NPART 4
#endif
constexpr int NPART = SPT_FWD2_NPART;  // P hand-off parts per block (PV MMAs start per part)
constexpr int Q_BYTES = BQ * D * 2;    // 32 KiB per tile
constexpr int KV_BYTES = BKB * D * 2;  // 32 KiB per K or V block (two 16 KiB regions)
#ifndef SPT_FWD2_NSL
#define SPT_FWD2_NSL 4
#endif
constexpr int NSL = SPT_FWD2_NSL;  // K/V ring slots (5 is the most that fits next to the two Q tiles)
// 12 warps = 3 warpgroups: two softmax warpgroups (one per query tile) and one for the MMA issuer (warp 8), the
// TMA producer (warp 9) and two idle warps.  ptxas sizes registers per warpgroup multiple (the old 10-warp launch
// was capped at 65536 / 384 = 168 and spilled the softmax loop state); setmaxnreg moves them where they are used.
constexpr int THREADS = 384;
constexpr int REG_SOFTMAX = 216, REG_PRODUCER = 64;  // 2 * 128 * 216 + 128 * 64 <= 168 * 384
static_assert(2 * 128 * REG_SOFTMAX + 128 * REG_PRODUCER <= 168 * THREADS, "register budget");
constexpr int OFF_Q = 0, OFF_KV = 2 * Q_BYTES;
constexpr int OFF_BAR = OFF_KV + NSL * KV_BYTES;
constexpr int SMEM = OFF_BAR + 512 + 1024;
}  // namespace fw2

// POLY > 0: every POLY-th exponential pair goes through ex2_poly on the FMA pipe (MUFU relief: with 128-key
// blocks the exponentials of both tiles need the whole MUFU throughput at full tensor rate).
// DH: head dim (128, 64 or 32).  Shared memory and TMEM keep the d=128 layout; a d < 128 tile fills DP = max(DH, 64)
// columns of it (one 64-column TMA box: for d = 32 the box also brings the next head's 32 columns, or TMA's zero
// fill past the last head).  The score MMA contracts over DH only; the PV MMA runs N = DP, and output columns
// >= DH (the neighbour's V) are never stored.
template <int POLY, int DH>
__global__ void __launch_bounds__(fw2::THREADS, 1)
    fwd_tc128_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tkv, int64_t s, int hq,
                     int hkv, const int32_t* __restrict__ seg, float scale_log2, bf16* __restrict__ o,
                     float* __restrict__ lse, int kvg, int filter) {
    using namespace fw2;
    constexpr int DP = DH < 64 ? 64 : DH, NR = DP / 64;
    constexpr int QB = BQ * DP * 2, KVB = BKB * DP * 2;  // bytes one tile / block load brings
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* q_full = bar;
    uint64_t* kv_full = bar + 1;
    uint64_t* kv_empty = kv_full + NSL;
    uint64_t* s_full = kv_empty + NSL;  // [t]
    uint64_t* p_full = s_full + 2;      // [t * NPART + part]: P for keys [part, part + 1) * 128 / NPART written
    uint64_t* pv_done = p_full + 2 * NPART;  // [t]
    uint64_t* o_done = pv_done + 2;     // [t]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

    const int warp = warp_id(), lane = lane_id();
    const int npairs = (int)((s + 2 * BQ - 1) / (2 * BQ));
    int h, yb;
    grid_head_row(kvg, hq, hkv, h, yb);
    const int pair = npairs - 1 - yb;
    const int kvh = h / (hq / hkv);
    const int64_t q0 = (int64_t)pair * 2 * BQ;
    const bool has1 = q0 + BQ < s;
    const int jb0 = seg ? (int)(seg[q0] / BKB) : 0, jb1 = (seg && has1) ? (int)(seg[q0 + BQ] / BKB) : 0;
    const int je0 = (int)((q0 + BQ - 1) / BKB), je1 = has1 ? (int)((q0 + 2 * BQ - 1) / BKB) : -1;
    const int jlo = jb0, jhi = has1 ? je1 : je0;
    if (filter) {  // packed hybrid: this launch handles only the long (1) or short (2) tile pairs
        const bool longp = q0 + 2 * BQ - (seg ? seg[q0] : 0) >= FWD_LONG_KEYS;
        if ((filter == 1) != longp) return;  // whole CTA, before any barrier / TMEM allocation
    }

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < NSL; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&s_full[t], 1);
            for (int part = 0; part < NPART; ++part) mbar_init(&p_full[NPART * t + part], 128);
            mbar_init(&pv_done[t], 1);
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
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
    const uint32_t sbase = smem_u32(smem);
    // setmaxnreg inside each role branch, so every role's code is dominated by its own register limit
    if (warp == 9) {
        reg_dealloc<REG_PRODUCER>();
        if (lane == 0) {
            tma_prefetch_desc(&tq);
            tma_prefetch_desc(&tkv);
            mbar_arrive_expect_tx(q_full, 2 * QB);
            for (int t = 0; t < 2; ++t)
                for (int r = 0; r < NR; ++r)
                    tma_load_2d(&tq, q_full, smem + OFF_Q + t * Q_BYTES + r * 16384, h * DH + 64 * r,
                                (int)(q0 + t * BQ));
            const int nload = 2 * (jhi - jlo + 1);
            for (int li = 0; li < nload; ++li) {
                const int j = jlo + li / 2, w = li & 1;
                const int slot = li % NSL;
                mbar_wait(&kv_empty[slot], ((li / NSL) & 1) ^ 1);
                mbar_arrive_expect_tx(&kv_full[slot], KVB);
                const int col = (hq + (w ? hkv : 0) + kvh) * DH;
                for (int r = 0; r < NR; ++r)
                    tma_load_2d(&tkv, &kv_full[slot], smem + OFF_KV + slot * KV_BYTES + r * 16384, col + 64 * r,
                                j * BKB);
            }
        }
    } else if (warp == 8) {
        reg_dealloc<REG_PRODUCER>();
        {
            constexpr uint32_t idesc_s = make_idesc_bf16(BQ, BKB, false, false);
            constexpr uint32_t idesc_o = make_idesc_bf16(BQ, DP, false, true);
            mbar_wait(q_full, 0);
            const int jb[2] = {jb0, jb1}, je[2] = {je0, je1};
            int pv_count[2] = {0, 0};
            auto uses = [&](int t, int j) { return j >= jb[t] && j <= je[t]; };
            auto slot = [&](int j, int w) { return (2 * (j - jlo) + w) % NSL; };
            auto phase = [&](int j, int w) { return (uint32_t)(((2 * (j - jlo) + w) / NSL) & 1); };
            auto issue_s = [&](int t, int j) {
                mbar_wait(&kv_full[slot(j, 0)], phase(j, 0));
                tc_fence_after();
                const uint32_t qa = sbase + OFF_Q + t * Q_BYTES;
                const uint32_t kb = sbase + OFF_KV + slot(j, 0) * KV_BYTES;
#pragma unroll
                for (int kk = 0; kk < DH / 16; ++kk)
                    mma_bf16_ss_w(tmem + t * 256, kdesc_r(qa, kk, 16384), kdesc_r(kb, kk, 16384), idesc_s, kk > 0);
                mma_commit_w(&s_full[t]);
            };
            auto issue_pv = [&](int t, int j) {  // in two halves: the first starts while the softmax finishes
                mbar_wait(&kv_full[slot(j, 1)], phase(j, 1));
                const uint32_t vb = sbase + OFF_KV + slot(j, 1) * KV_BYTES;
#pragma unroll
                for (int part = 0; part < NPART; ++part) {
                    mbar_wait(&p_full[NPART * t + part], (j - jb[t]) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int kq = 0; kq < BKB / 16 / NPART; ++kq) {
                        const int kk = part * (BKB / 16 / NPART) + kq;
                        mma_bf16_ts_w(tmem + t * 256 + 128, tmem + t * 256 + kk * 8, mndesc_r(vb, kk, 16384), idesc_o,
                                      (pv_count[t] > 0 || kk > 0));
                    }
                }
                mma_commit_w(&pv_done[t]);
                ++pv_count[t];
            };
            if (uses(0, jlo)) issue_s(0, jlo);
            if (uses(1, jlo)) issue_s(1, jlo);
            mma_commit_w(&kv_empty[slot(jlo, 0)]);
            for (int j = jlo; j <= jhi; ++j) {
                const bool more = j + 1 <= jhi;
                if (uses(0, j)) issue_pv(0, j);
                if (more && uses(0, j + 1)) issue_s(0, j + 1);
                if (uses(1, j)) issue_pv(1, j);
                mma_commit_w(&kv_empty[slot(j, 1)]);  // V_j consumed
                if (more) {
                    if (uses(1, j + 1)) issue_s(1, j + 1);
                    mma_commit_w(&kv_empty[slot(j + 1, 0)]);  // K_{j+1} consumed by both tiles
                }
            }
            mma_commit_w(&o_done[0]);
            mma_commit_w(&o_done[1]);
        }
    } else if (warp < 8) {
        reg_alloc<REG_SOFTMAX>();
        // ---------------- softmax warpgroups (thread = query row), 128 columns per block in 4 chunks of 32
        const int t = warp >> 2;
        const int sub = warp & 3;
        const int r = sub * 32 + lane;
        const int64_t q = q0 + t * BQ + r;
        const bool row_ok = q < s;
        const int start = (seg && row_ok) ? seg[q] : 0;
        const uint32_t lane_off = (uint32_t)(sub * 32) << 16;
        const uint32_t t_tm = tmem + lane_off + t * 256;
        const uint32_t o_tm = t_tm + 128;
        const int jb_t = t ? jb1 : jb0, je_t = t ? je1 : je0;
        float m_use = -INFINITY, l = 0.f;
        for (int j = jb_t; j <= je_t; ++j) {
            const int n = j - jb_t;
            mbar_wait(&s_full[t], n & 1);
            tc_fence_after();
            const int64_t k0 = (int64_t)j * BKB;
            const bool need_mask = (k0 + BKB - 1 > q0 + t * BQ) || (seg != nullptr && __any_sync(0xffffffffu, start > k0));
            uint32_t v[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(t_tm + c * 32, v[c]);
            tmem_ld_wait();
            float mp[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) mp[u] = -INFINITY;
            if (need_mask) {
                const int hi = (int)(q - k0), lo_ = start - (int)k0;
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int col = c * 32 + i;
                        if (col > hi || col < lo_) v[c][i] = __float_as_uint(-INFINITY);
                    }
            }
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int i = 0; i < 32; i += 2)
                    mp[(c * 32 + i) >> 1 & 7] =
                        fmax3(mp[(c * 32 + i) >> 1 & 7], __uint_as_float(v[c][i]), __uint_as_float(v[c][i + 1]));
            const float mraw = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])),
                                     fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
            const float mx = mraw * scale_log2;
            const bool grow = mx > m_use + RESCALE_THRESHOLD;
            const bool resc = grow && m_use != -INFINITY && n > 0;
            const float alpha = resc ? ex2(m_use - mx) : 1.f;
            if (__any_sync(0xffffffffu, resc)) {  // needs PV_t(j-1) complete
                mbar_wait(&pv_done[t], (n - 1) & 1);
                tc_fence_after();
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    uint32_t ov[32];
                    tmem_ld32(o_tm + c * 32, ov);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
                    tmem_st32(o_tm + c * 32, ov);
                }
            }
            l *= alpha;
            if (grow) m_use = mx;
            const float nbase = m_use == -INFINITY ? 0.f : -m_use;
            const uint64_t sc2 = f2pack(scale_log2, scale_log2), nb2 = f2pack(nbase, nbase);
            uint64_t rs2[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) rs2[u] = f2pack(0.f, 0.f);
            // P for chunk c (32 keys) -> 16 packed columns at [16c, 16c+16): the chunk's S columns [32c, 32c+32)
            // were already read into registers, and chunk c's P never lands on a chunk not yet read
            // POLY > 1: on unmasked blocks every POLY-th exponential pair runs on the FMA pipe (ex2_poly2), so
            // the MUFU pipe — exactly saturated by two 128x128 tiles at full tensor rate — is no longer the
            // co-bottleneck; masked blocks stay on MUFU (masked entries exactly 0).
            auto exps = [&](auto use_poly) {
                constexpr bool UP = decltype(use_poly)::value;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t pw[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const uint64_t x2 = ffma2(f2pack(__uint_as_float(v[c][2 * k]), __uint_as_float(v[c][2 * k + 1])), sc2, nb2);
                        float x0, x1;
                        f2unpack(x2, x0, x1);
                        float p0, p1;
                        if constexpr (POLY == 1) {  // two exponentials per MUFU op in f16 (P is bf16 anyway)
                            ex2_f16x2(x0, x1, p0, p1);
                        } else if constexpr (UP) {
                            if ((c * 16 + k) % POLY == POLY - 1) ex2_poly2(x0, x1, p0, p1);
                            else {
                                p0 = ex2(x0);
                                p1 = ex2(x1);
                            }
                        } else {
                            p0 = ex2(x0);
                            p1 = ex2(x1);
                        }
                        rs2[k & 3] = fadd2(rs2[k & 3], f2pack(p0, p1));
                        pw[k] = pack_bf16x2(p0, p1);
                    }
                    tmem_st16(t_tm + c * 16, pw);
                    if (c < 3 && (c + 1) % (4 / NPART) == 0) {  // this part of P done: its PV MMAs can start
                        tmem_st_wait();
                        tc_fence_before();
                        mbar_arrive(&p_full[NPART * t + (c + 1) / (4 / NPART) - 1]);
                    }
                }
            };
            if (POLY > 1 && !need_mask) exps(std::true_type{});
            else exps(std::false_type{});
            float rs0, rs1;
            f2unpack(fadd2(fadd2(rs2[0], rs2[1]), fadd2(rs2[2], rs2[3])), rs0, rs1);
            l += rs0 + rs1;
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&p_full[NPART * t + NPART - 1]);
        }
        mbar_wait(&o_done[t], 0);
        tc_fence_after();
        if (t == 1 && !has1) goto fwd2_done;
        {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        bf16* orow = o + (q * hq + h) * DH;
#pragma unroll 1
        for (int c = 0; c < DH / 32; ++c) {
            uint32_t ov[32];
            tmem_ld32(o_tm + c * 32, ov);
            tmem_ld_wait();
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint4 w;
                w.x = pack_bf16x2(__uint_as_float(ov[8 * k + 0]) * inv, __uint_as_float(ov[8 * k + 1]) * inv);
                w.y = pack_bf16x2(__uint_as_float(ov[8 * k + 2]) * inv, __uint_as_float(ov[8 * k + 3]) * inv);
                w.z = pack_bf16x2(__uint_as_float(ov[8 * k + 4]) * inv, __uint_as_float(ov[8 * k + 5]) * inv);
                w.w = pack_bf16x2(__uint_as_float(ov[8 * k + 6]) * inv, __uint_as_float(ov[8 * k + 7]) * inv);
                dst[k] = w;
            }
        }
        lse[(int64_t)h * s + q] = l > 0.f ? (m_use + __log2f(l)) * LN2 : -INFINITY;
        }
    fwd2_done:;
    } else {
        reg_dealloc<REG_PRODUCER>();  // warps 10, 11: no role
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

namespace fwt {  // forward with Q resident in TMEM (fwd_tmem_kernel)
constexpr int BKB = 64;
constexpr int KV_BYTES = BKB * D * 2;  // 16 KiB per K or V block (two 8 KiB regions)
constexpr int NSL = 13;
constexpr int OFF_KV = 0;
constexpr int OFF_BAR = OFF_KV + NSL * KV_BYTES;
constexpr int SMEM = OFF_BAR + 512 + 1024;
}  // namespace fwt

// Forward with Q resident in TMEM: per tile one S buffer (64 cols) + Q (64 cols, bf16 pairs) + O (128 cols).
// S = Q K^T becomes a ts-form MMA that reads only its 2 KiB B operand (K) from smem: with both operands in
// smem an M=128 N=64 K=16 MMA is smem-bandwidth bound (48 cycles for 32 of math, tools/micro/mma_rate.cu).
__global__ void __launch_bounds__(THREADS, 1)
    fwd_tmem_kernel(const __grid_constant__ CUtensorMap tkv, const bf16* __restrict__ qkv_in, int64_t s, int hq,
                  int hkv, const int32_t* __restrict__ seg, float scale_log2, bf16* __restrict__ o,
                  float* __restrict__ lse) {
    using namespace fwt;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* q_full = bar;  // here: Q tiles written into TMEM by the softmax warps (256 arrivals)
    uint64_t* kv_full = bar + 1;
    uint64_t* kv_empty = kv_full + NSL;
    uint64_t* s_full = kv_empty + NSL;  // [t*2 + b]
    uint64_t* p_full = s_full + 4;      // [t*2 + b]  per buffer: the softmax may run 2 blocks ahead
    uint64_t* pv_done = p_full + 4;     // [t]
    uint64_t* o_done = pv_done + 2;     // [t]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

    const int warp = warp_id(), lane = lane_id();
    const int npairs = (int)((s + 2 * BQ - 1) / (2 * BQ));  // s % 256 == 128: the last pair holds one tile
    // grid = (q head, query-tile pair): heads vary fastest so one wave of CTAs streams the K/V of every kv
    // head at once instead of 148 CTAs hammering the same K/V lines (L2-slice hot spot); longest rows first
    const int pair = npairs - 1 - (int)blockIdx.y;
    const int h = blockIdx.x;
    const int kvh = h / (hq / hkv);
    const int64_t q0 = (int64_t)pair * 2 * BQ;
    const bool has1 = q0 + BQ < s;  // second query tile present
    const int jb0 = seg ? (int)(seg[q0] / BKB) : 0, jb1 = (seg && has1) ? (int)(seg[q0 + BQ] / BKB) : 0;
    const int je0 = (int)((q0 + BQ - 1) / BKB), je1 = has1 ? (int)((q0 + 2 * BQ - 1) / BKB) : -1;
    const int jlo = jb0, jhi = has1 ? je1 : je0;  // jb0 <= jb1 (starts are monotone), je0 < je1

    if (threadIdx.x == 0) {
        mbar_init(q_full, 256);
        for (int i = 0; i < NSL; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 4; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 128);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&pv_done[t], 1);
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
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // provably warp-uniform: descriptor math stays in uniform registers
    const uint32_t sbase = smem_u32(smem);

    if (warp == 9) {
        if (lane == 0) {
            tma_prefetch_desc(&tkv);
            const int nload = 2 * (jhi - jlo + 1);
            for (int li = 0; li < nload; ++li) {
                const int j = jlo + li / 2, w = li & 1;
                const int slot = li % NSL;
                mbar_wait(&kv_empty[slot], ((li / NSL) & 1) ^ 1);
                mbar_arrive_expect_tx(&kv_full[slot], KV_BYTES);
                const int col = (hq + (w ? hkv : 0) + kvh) * D;
                for (int r = 0; r < 2; ++r)
                    tma_load_2d(&tkv, &kv_full[slot], smem + OFF_KV + slot * KV_BYTES + r * 8192, col + 64 * r, j * BKB);
            }
        }
    } else if (warp == 8) {
        {  // whole warp, converged; elect.sync inside the MMA/commit wrappers picks the issuing lane
            constexpr uint32_t idesc_s = make_idesc_bf16(BQ, BKB, false, false);
            constexpr uint32_t idesc_o = make_idesc_bf16(BQ, D, false, true);
            mbar_wait(q_full, 0);  // Q tiles resident in TMEM
            tc_fence_after();
            const int jb[2] = {jb0, jb1}, je[2] = {je0, je1};
            int pv_count[2] = {0, 0};
            auto uses = [&](int t, int j) { return j >= jb[t] && j <= je[t]; };
            auto slot = [&](int j, int w) { return (2 * (j - jlo) + w) % NSL; };
            auto phase = [&](int j, int w) { return (uint32_t)(((2 * (j - jlo) + w) / NSL) & 1); };
            // S_t(j) = Q_t K_j^T with Q_t from TMEM (ts form: only K is read from smem)
            auto issue_s = [&](int t, int j) {
                mbar_wait(&kv_full[slot(j, 0)], phase(j, 0));
                tc_fence_after();
                const uint32_t kb = sbase + OFF_KV + slot(j, 0) * KV_BYTES;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    mma_bf16_ts_w(tmem + t * 256, tmem + t * 256 + 64 + kk * 8, kdesc_r(kb, kk, 8192), idesc_s, kk > 0);
                mma_commit_w(&s_full[t * 2]);
            };
            auto issue_pv = [&](int t, int j) {
                mbar_wait(&p_full[t * 2], (j - jb[t]) & 1);
                mbar_wait(&kv_full[slot(j, 1)], phase(j, 1));
                tc_fence_after();
                const uint32_t vb = sbase + OFF_KV + slot(j, 1) * KV_BYTES;
#pragma unroll
                for (int kk = 0; kk < BKB / 16; ++kk)
                    mma_bf16_ts_w(tmem + t * 256 + 128, tmem + t * 256 + kk * 8, mndesc_r(vb, kk, 8192), idesc_o,
                                  (pv_count[t] > 0 || kk > 0));
                mma_commit_w(&pv_done[t]);
                ++pv_count[t];
            };
            // one S buffer per tile: S_t(j+1) overwrites P_t(j) right after PV_t(j) (in-order tensor pipe);
            // the two tiles ping-pong so one tile's softmax overlaps the other tile's MMAs
            if (uses(0, jlo)) issue_s(0, jlo);
            if (uses(1, jlo)) issue_s(1, jlo);
            mma_commit_w(&kv_empty[slot(jlo, 0)]);
            for (int j = jlo; j <= jhi; ++j) {
                const bool more = j + 1 <= jhi;
                if (uses(0, j)) issue_pv(0, j);
                if (more && uses(0, j + 1)) issue_s(0, j + 1);
                if (uses(1, j)) issue_pv(1, j);
                mma_commit_w(&kv_empty[slot(j, 1)]);  // V_j consumed
                if (more) {
                    if (uses(1, j + 1)) issue_s(1, j + 1);
                    mma_commit_w(&kv_empty[slot(j + 1, 0)]);  // K_{j+1} consumed by both tiles
                }
            }
            mma_commit_w(&o_done[0]);
            mma_commit_w(&o_done[1]);
        }
    } else {
        // ---------------- softmax warpgroups (thread = query row)
        const int t = warp >> 2;
        const int sub = warp & 3;
        const int r = sub * 32 + lane;
        const int64_t q = q0 + t * BQ + r;
        const bool row_ok = q < s;  // false only for the absent second tile of a half pair
        const int start = (seg && row_ok) ? seg[q] : 0;
        const uint32_t lane_off = (uint32_t)(sub * 32) << 16;
        const uint32_t t_tm = tmem + lane_off + t * 256;
        const uint32_t o_tm = t_tm + 128;
        {  // this thread's Q row (q head h) -> TMEM columns [t*256 + 64, +64) as bf16 pairs (A operand of S)
            const uint4* qs = reinterpret_cast<const uint4*>(qkv_in + (row_ok ? q : 0) * (int64_t)(hq + 2 * hkv) * D +
                                                             (int64_t)h * D);
            uint32_t qv[32];
#pragma unroll
            for (int half = 0; half < 2; ++half) {
#pragma unroll
                for (int k4 = 0; k4 < 8; ++k4) {
                    const uint4 a4 = __ldg(qs + half * 8 + k4);
                    qv[4 * k4] = a4.x; qv[4 * k4 + 1] = a4.y; qv[4 * k4 + 2] = a4.z; qv[4 * k4 + 3] = a4.w;
                }
                tmem_st32(t_tm + 64 + half * 32, qv);
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(q_full);
        }
        const int jb_t = t ? jb1 : jb0, je_t = t ? je1 : je0;
        float m_use = -INFINITY, l = 0.f;  // running max in log2 units (scaled)
        for (int j = jb_t; j <= je_t; ++j) {
            const int n = j - jb_t, b = 0;
            const uint32_t s_tm = t_tm + b * 64;
#ifdef SPT_WATCHDOG
            volatile int* dbg = reinterpret_cast<volatile int*>(tmem_slot + 4);
            if (r == 0) { dbg[2 * t] = j; dbg[2 * t + 1] = 1; }
#endif
            mbar_wait(&s_full[t * 2], n & 1);
#ifdef SPT_WATCHDOG
            if (r == 0) dbg[2 * t + 1] = 2;
#endif
            tc_fence_after();
            const int64_t k0 = (int64_t)j * BKB;
            // warp-uniform: causal diagonal, or (packed) some row of this warp starts its sample inside the block
            const bool need_mask = (k0 + BKB - 1 > q0 + t * BQ) || (seg != nullptr && __any_sync(0xffffffffu, start > k0));
            uint32_t v[2][32];
            tmem_ld32(s_tm, v[0]);
            tmem_ld32(s_tm + 32, v[1]);
            tmem_ld_wait();
            // row max over the 64 columns: 8 independent partial maxima (short dependency chains; the two
            // softmax warps per SMSP cannot hide a 64-long serial FMNMX chain)
            float mp[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) mp[u] = -INFINITY;
            if (need_mask) {
                const int hi = (int)(q - k0), lo_ = start - (int)k0;  // keep columns lo_ <= i <= hi
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int col = c * 32 + i;
                        if (col > hi || col < lo_) v[c][i] = __float_as_uint(-INFINITY);
                        mp[col & 7] = fmaxf(mp[col & 7], __uint_as_float(v[c][i]));
                    }
            } else {
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int i = 0; i < 32; i += 2)
                        mp[(c * 32 + i) >> 1 & 7] =
                            fmaxf(mp[(c * 32 + i) >> 1 & 7], fmaxf(__uint_as_float(v[c][i]), __uint_as_float(v[c][i + 1])));
            }
            const float mraw = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])),
                                     fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
            const float mx = mraw * scale_log2;
            // lazy rescale (warp-uniform: tcgen05.ld/st are warp-collective); needs PV_t(j-1) complete
            const bool grow = mx > m_use + RESCALE_THRESHOLD;
            const bool resc = grow && m_use != -INFINITY && n > 0;
            const float alpha = resc ? ex2(m_use - mx) : 1.f;
            if (__any_sync(0xffffffffu, resc)) {
                mbar_wait(&pv_done[t], (n - 1) & 1);
                tc_fence_after();
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    uint32_t ov[32];
                    tmem_ld32(o_tm + c * 32, ov);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
                    tmem_st32(o_tm + c * 32, ov);
                }
            }
            l *= alpha;
            if (grow) m_use = mx;
            const float nbase = m_use == -INFINITY ? 0.f : -m_use;
            uint32_t pw[32];
            const uint64_t sc2 = f2pack(scale_log2, scale_log2), nb2 = f2pack(nbase, nbase);
            uint64_t rs2[4];  // 4 independent packed row-sum accumulators (short FADD2 chains)
#pragma unroll
            for (int u = 0; u < 4; ++u) rs2[u] = f2pack(0.f, 0.f);
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const int c0 = 2 * k;
                const uint64_t x2 = ffma2(f2pack(__uint_as_float(v[c0 >> 5][c0 & 31]), __uint_as_float(v[c0 >> 5][(c0 + 1) & 31])),
                                          sc2, nb2);
                float x0, x1;
                f2unpack(x2, x0, x1);
                const bool poly = SPT_FWD_POLY_EVERY > 0 && (k % (SPT_FWD_POLY_EVERY > 0 ? SPT_FWD_POLY_EVERY : 1)) ==
                                                                (SPT_FWD_POLY_EVERY > 0 ? SPT_FWD_POLY_EVERY - 1 : 0);
                const float p0 = poly ? ex2_poly(x0) : ex2(x0);
                const float p1 = poly ? ex2_poly(x1) : ex2(x1);
                rs2[k & 3] = fadd2(rs2[k & 3], f2pack(p0, p1));
                pw[k] = pack_bf16x2(p0, p1);
            }
            float rs0, rs1;
            f2unpack(fadd2(fadd2(rs2[0], rs2[1]), fadd2(rs2[2], rs2[3])), rs0, rs1);
            const float rs = rs0 + rs1;
            l += rs;
#ifdef SPT_WATCHDOG
            if (r == 0) dbg[2 * t + 1] = 3;
#endif
            tmem_st32(s_tm, pw);  // packed P over the consumed S columns [0, 32)
            tmem_st_wait();
#ifdef SPT_WATCHDOG
            if (r == 0) dbg[2 * t + 1] = 4;
#endif
            tc_fence_before();
            mbar_arrive(&p_full[t * 2]);
        }
        // epilogue: O_t / l -> global, lse
        mbar_wait(&o_done[t], 0);
        tc_fence_after();
        if (t == 1 && !has1) goto fwd_done;  // warp-uniform: the whole tile is absent
        {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        bf16* orow = o + (q * hq + h) * D;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t ov[32];
            tmem_ld32(o_tm + c * 32, ov);
            tmem_ld_wait();
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint4 w;
                w.x = pack_bf16x2(__uint_as_float(ov[8 * k + 0]) * inv, __uint_as_float(ov[8 * k + 1]) * inv);
                w.y = pack_bf16x2(__uint_as_float(ov[8 * k + 2]) * inv, __uint_as_float(ov[8 * k + 3]) * inv);
                w.z = pack_bf16x2(__uint_as_float(ov[8 * k + 4]) * inv, __uint_as_float(ov[8 * k + 5]) * inv);
                w.w = pack_bf16x2(__uint_as_float(ov[8 * k + 6]) * inv, __uint_as_float(ov[8 * k + 7]) * inv);
                dst[k] = w;
            }
        }
        lse[(int64_t)h * s + q] = l > 0.f ? (m_use + __log2f(l)) * LN2 : -INFINITY;
        }
    fwd_done:;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        __syncwarp();  // role branches diverged lane 0; dealloc is warp-collective (.sync.aligned)
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ===================================================================================== backward

// ------------------------------------------------------------------ dQ pass
// CTA = (128-row q tile, q head).  Per 64-key block j (double-buffered in TMEM):
//   S_j = Q K_j^T, dP_j = dO V_j^T -> dS_j = P (dP - D) (bf16, smem, double-buffered) -> dQ += dS_j K_j.
// 8 elementwise warps (2 per TMEM lane quarter, each owning 32 of the 64 key columns), 6-slot K/V ring.
namespace dq {
constexpr int BKB = 64;
constexpr int Q_BYTES = 128 * D * 2;        // 32 KiB
constexpr int KV_BYTES = BKB * D * 2;       // 16 KiB (two 8 KiB regions)
#ifndef SPT_DQ_NSL
#define SPT_DQ_NSL 10
#endif
constexpr int NSL = SPT_DQ_NSL;  // K/V ring slots (16 KiB each): 5 blocks of K+V in flight
constexpr int NB = 3;          // S/dP TMEM buffers (128 columns each): the MMA runs NB-1 blocks ahead
constexpr int DQ_COL = 384;    // dQ accumulator columns [384, 512)
constexpr int OFF_Q = 0, OFF_DO = Q_BYTES, OFF_KV = 2 * Q_BYTES;  // dS lives in TMEM (A operand of dQ)
constexpr int OFF_BAR = OFF_KV + NSL * KV_BYTES;
constexpr int SMEM = OFF_BAR + 256 + 1024;
}  // namespace dq

// MC: q heads (2m, 2m+1) of the same kv head and q tile form a cluster; their K/V streams are identical, so
// rank 0 multicasts the K blocks and rank 1 the V blocks into both CTAs (half the L2->SM bytes per CTA);
// a K/V slot is released by both CTAs' MMAs (multicast commit, count 2).
template <bool MC>
__global__ void __launch_bounds__(BW_THREADS, 1)
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
    uint64_t* s_full = kv_empty + NSL;  // [NB]
    uint64_t* ds_full = s_full + NB;     // [NB]
    uint64_t* dq_done = ds_full + NB;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_done + 1);
    const int warp = warp_id(), lane = lane_id();
    const int nqb = (int)(s / 128);
    const int qb = nqb - 1 - (int)blockIdx.y;  // longest rows first; heads vary fastest (see fwd_tc_kernel)
    const int h = blockIdx.x;
    const int kvh = h / (hq / hkv);
    const int64_t q0 = (int64_t)qb * 128;
    const int jb = seg ? (int)(seg[q0] / BKB) : 0;
    const int je = (int)((q0 + 127) / BKB);
    const int nblk = je - jb + 1;
    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < NSL; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], MC ? 2 : 1);
        }
        for (int t = 0; t < NB; ++t) {
            mbar_init(&s_full[t], 1);
            mbar_init(&ds_full[t], BW_NEW * 32);
        }
        mbar_init(dq_done, 1);
        fence_barrier_init();
    }
    if (warp == BW_MMA) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    if (MC) cluster_sync();  // both CTAs' barriers initialised before any multicast load / remote arrive
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // provably warp-uniform: descriptor math stays in uniform registers
    const uint32_t sbase = smem_u32(smem);
    const uint32_t crank = MC ? cluster_ctarank() : 0;
    if (warp == BW_TMA) {
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
#ifdef SPT_EXP_HALF_KV  // experiment (wrong results): half the K/V bytes, to test for L2->SM bandwidth limits
                mbar_arrive_expect_tx(&kv_full[slot], KV_BYTES / 2);
                const int col = (hq + (w ? hkv : 0) + kvh) * D;
                tma_load_2d(&tkv, &kv_full[slot], smem + OFF_KV + slot * KV_BYTES, col, j * BKB);
#else
                mbar_arrive_expect_tx(&kv_full[slot], KV_BYTES);
                const int col = (hq + (w ? hkv : 0) + kvh) * D;
                if constexpr (MC) {
                    if ((uint32_t)w == crank)  // rank 0: K blocks, rank 1: V blocks, each into both CTAs
                        for (int r = 0; r < 2; ++r)
                            tma_load_2d_mc(&tkv, &kv_full[slot], smem + OFF_KV + slot * KV_BYTES + r * 8192,
                                           col + 64 * r, j * BKB, 0x3);
                } else {
                    for (int r = 0; r < 2; ++r)
                        tma_load_2d(&tkv, &kv_full[slot], smem + OFF_KV + slot * KV_BYTES + r * 8192, col + 64 * r,
                                    j * BKB);
                }
#endif
            }
        }
    } else if (warp == BW_MMA) {
        {  // whole warp, converged; elect.sync inside the MMA/commit wrappers picks the issuing lane
            constexpr uint32_t id_s = make_idesc_bf16(128, BKB, false, false);
            constexpr uint32_t id_q = make_idesc_bf16(128, D, false, true);
            mbar_wait(q_full, 0);
            const uint32_t qa = sbase + OFF_Q, da = sbase + OFF_DO;
            auto issue_sdp = [&](int it) {
                const int ks = (2 * it) % NSL, vs = (2 * it + 1) % NSL;
                {
                    DQP_T0();
                    mbar_wait(&kv_full[ks], ((2 * it) / NSL) & 1);
                    mbar_wait(&kv_full[vs], ((2 * it + 1) / NSL) & 1);
                    if (lane == 0) DQP_ADD(0);
                }
                tc_fence_after();
                const uint32_t kb = sbase + OFF_KV + ks * KV_BYTES, vb = sbase + OFF_KV + vs * KV_BYTES;
                const uint32_t d_s = tmem + (it % NB) * 128;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    mma_bf16_ss_w(d_s, kdesc_r(qa, kk, 16384), kdesc_r(kb, kk, 8192), id_s, kk > 0);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    mma_bf16_ss_w(d_s + 64, kdesc_r(da, kk, 16384), kdesc_r(vb, kk, 8192), id_s, kk > 0);
                mma_commit_w(&s_full[it % NB]);
                if constexpr (MC) mma_commit_mc_w(&kv_empty[vs], 0x3);  // V_j only feeds dP
                else mma_commit_w(&kv_empty[vs]);
            };
            auto issue_dq = [&](int it) {
                {
                    DQP_T0();
                    mbar_wait(&ds_full[it % NB], (it / NB) & 1);
                    if (lane == 0) DQP_ADD(1);
                }
                tc_fence_after();
                const int ks = (2 * it) % NSL;
                const uint32_t kb = sbase + OFF_KV + ks * KV_BYTES;
                // A = dS in TMEM: keys [16g, 16g+16) packed in S columns [16g, 16g+8) of buffer it%NB
#pragma unroll
                for (int kk = 0; kk < BKB / 16; ++kk)
                    mma_bf16_ts_w(tmem + DQ_COL, tmem + (it % NB) * 128 + kk * 16, mndesc_r(kb, kk, 8192), id_q,
                                  (it > 0 || kk > 0));
                if constexpr (MC) mma_commit_mc_w(&kv_empty[ks], 0x3);
                else mma_commit_w(&kv_empty[ks]);
            };
#ifdef SPT_DQ_PROF
            const long long _tm0 = clock64();
#endif
            for (int it = 0; it < min(NB, nblk); ++it) issue_sdp(it);
            for (int it = 0; it < nblk; ++it) {
                issue_dq(it);
                if (it + NB < nblk) issue_sdp(it + NB);
            }
            mma_commit_w(dq_done);
#ifdef SPT_DQ_PROF
            if (lane == 0) {
                atomicAdd(&g_dq_prof[4], (unsigned long long)(clock64() - _tm0));
                atomicAdd(&g_dq_prof[5], 1ull);
                atomicAdd(&g_dq_prof[6], (unsigned long long)nblk);
            }
#endif
        }
    } else {
        const int sub = warp & 3, grp = warp >> 2;  // lanes [32 sub, +32), keys [16 grp, +16) of each block
        const int r = sub * 32 + lane;
        const int64_t q = q0 + r;
        const int q32 = (int)q, q0i = (int)q0;  // s < 2^31 (attn_bwd_tc checks)
        const int start = seg ? seg[q] : 0;
        const float nlse2 = -lse2v[(int64_t)h * s + q];  // -(lse * log2 e), precomputed
        const float Dq = Dv[(int64_t)h * s + q];
        const float sl2 = scale * LOG2E;
        const uint32_t lo = (uint32_t)(sub * 32) << 16;
        for (int it = 0; it < nblk; ++it) {
            const int b = it % NB;
            {
                DQP_T0();
                mbar_wait(&s_full[b], (it / NB) & 1);
                if (threadIdx.x == 0) DQP_ADD(2);
            }
            tc_fence_after();
#ifdef SPT_EXP_NO_ELEM
            tc_fence_before();
            mbar_arrive(&ds_full[b]);
            continue;
#endif
            uint32_t sv[16], dv[16];
            tmem_ld16(tmem + lo + b * 128 + grp * 16, sv);
            tmem_ld16(tmem + lo + b * 128 + 64 + grp * 16, dv);
            tmem_ld_wait();
            const int k0 = (jb + it) * BKB + grp * 16;
            uint32_t w[8];
            // Two straight-line bodies (the branch is warp-uniform): the unmasked blocks carry no per-element
            // compare/select work at all; masked blocks compare the column index against int32 limits.
            auto body = [&](auto mask_c) {
                constexpr bool MASK = decltype(mask_c)::value;
                const int hi = q32 - k0, lo_ = start - k0;  // keep columns lo_ <= i <= hi
                const uint64_t sl2x = f2pack(sl2, sl2), nlx = f2pack(nlse2, nlse2), dqx = f2pack(Dq, Dq);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    float x0, x1;
                    f2unpack(ffma2(f2pack(__uint_as_float(sv[2 * k]), __uint_as_float(sv[2 * k + 1])), sl2x, nlx), x0, x1);
                    // part of the exponentials on the FMA pipe: this pass is MUFU-queue-bound, not issue-bound
                    const bool poly = SPT_DQ_POLY_EVERY > 0 && (k % (SPT_DQ_POLY_EVERY > 0 ? SPT_DQ_POLY_EVERY : 1)) ==
                                                                     (SPT_DQ_POLY_EVERY > 0 ? SPT_DQ_POLY_EVERY - 1 : 0);
                    float p0 = poly ? ex2_poly(x0) : ex2(x0), p1 = poly ? ex2_poly(x1) : ex2(x1);
                    if constexpr (MASK) {
                        p0 = (2 * k > hi || 2 * k < lo_) ? 0.f : p0;
                        p1 = (2 * k + 1 > hi || 2 * k + 1 < lo_) ? 0.f : p1;
                    }
                    const uint64_t ds = fmul2(f2pack(p0, p1),
                                              fsub2(f2pack(__uint_as_float(dv[2 * k]), __uint_as_float(dv[2 * k + 1])), dqx));
                    float d0, d1;
                    f2unpack(ds, d0, d1);
                    w[k] = pack_bf16x2(d0, d1);
                }
            };
            if (k0 + 15 > q0i || (seg != nullptr && __any_sync(0xffffffffu, start > k0))) body(std::true_type{});
            else body(std::false_type{});
            tmem_st8(tmem + lo + b * 128 + grp * 16, w);  // over this warp's consumed S columns
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&ds_full[b]);
        }
        mbar_wait(dq_done, 0);
        tc_fence_after();
        bf16* dst = dqkv + (q * (hq + 2 * hkv) + h) * D + grp * 32;
        {
            uint32_t v[32];
            tmem_ld32(tmem + lo + DQ_COL + grp * 32, v);
            tmem_ld_wait();
            uint4* d4 = reinterpret_cast<uint4*>(dst);
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
    if (MC) cluster_sync();  // the peer's multicast loads / remote arrives target this CTA until it is done
    if (warp == BW_MMA) {
        __syncwarp();  // role branches diverged lane 0; dealloc is warp-collective (.sync.aligned)
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ dQ pass, Q / dO resident in TMEM
// Same schedule as dq_tc_kernel, but the S = Q K^T and dP = dO V^T MMAs take their A operand (Q, dO) from
// TMEM ("ts" form) instead of shared memory.  A tcgen05.mma M=128 N=64 K=16 with both operands in smem reads
// 4 KiB (A) + 2 KiB (B) of smem at 128 B/clk = 48 cycles for 32 cycles of math (tools/micro/mma_rate.cu:
// N=64 runs at 67% of peak, N>=128 at 100%); with A in TMEM only the 2 KiB B operand is read from smem.
// TMEM: S/dP double buffer [0, 256) | dQ [256, 384) | Q [384, 448) | dO [448, 512) (bf16 pairs per column).
namespace dqt {
constexpr int BKB = 64;
constexpr int KV_BYTES = BKB * D * 2;  // 16 KiB (two 8 KiB regions)
constexpr int NSL = 12;                // K/V ring slots: 6 blocks of K+V in flight (Q/dO no longer in smem)
constexpr int NB = 2;
constexpr int DQ_COL = 256, QT_COL = 384, DOT_COL = 448;
constexpr int OFF_KV = 0;
constexpr int OFF_BAR = OFF_KV + NSL * KV_BYTES;
constexpr int SMEM = OFF_BAR + 256 + 1024;
}  // namespace dqt

// DH = 64 / 32: DP = 64 columns of the d=128 layout (see fwd_tc128_kernel); dQ runs N = DP, columns >= DH unused.
template <int DH>
__global__ void __launch_bounds__(BW_THREADS, 1)
    dq_tmem_kernel(const __grid_constant__ CUtensorMap tkv, const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                   int64_t s, int hq, int hkv, const int32_t* __restrict__ seg, const float* __restrict__ lse2v,
                   const float* __restrict__ Dv, float scale, bf16* __restrict__ dqkv, int kvg) {
    using namespace dqt;
    constexpr int DP = DH < 64 ? 64 : DH, NR = DP / 64;
    constexpr int KVB = BKB * DP * 2;  // bytes one K or V block load brings
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* qt_ready = bar;
    uint64_t* kv_full = bar + 1;
    uint64_t* kv_empty = kv_full + NSL;
    uint64_t* s_full = kv_empty + NSL;  // [NB]
    uint64_t* ds_full = s_full + NB;    // [NB]
    uint64_t* dq_done = ds_full + NB;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_done + 1);
    const int warp = warp_id(), lane = lane_id();
    const int nqb = (int)(s / 128);
    int h, yb;
    grid_head_row(kvg, hq, hkv, h, yb);
    const int qb = nqb - 1 - yb;  // longest rows first
    const int kvh = h / (hq / hkv);
    const int64_t q0 = (int64_t)qb * 128;
    const int jb = seg ? (int)(seg[q0] / BKB) : 0;
    const int je = (int)((q0 + 127) / BKB);
    const int nblk = je - jb + 1;
    if (threadIdx.x == 0) {
        mbar_init(qt_ready, BW_NEW * 32);
        for (int i = 0; i < NSL; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int t = 0; t < NB; ++t) {
            mbar_init(&s_full[t], 1);
            mbar_init(&ds_full[t], BW_NEW * 32);
        }
        mbar_init(dq_done, 1);
        fence_barrier_init();
    }
    if (warp == BW_MMA) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
    const uint32_t sbase = smem_u32(smem);
    if (warp == BW_TMA) {
        if (lane == 0) {
            tma_prefetch_desc(&tkv);
            for (int li = 0; li < 2 * nblk; ++li) {  // K_j, V_j, K_j+1, ...
                const int j = jb + li / 2, w = li & 1;
                const int slot = li % NSL;
                mbar_wait(&kv_empty[slot], ((li / NSL) & 1) ^ 1);
                mbar_arrive_expect_tx(&kv_full[slot], KVB);
                const int col = (hq + (w ? hkv : 0) + kvh) * DH;
                for (int r = 0; r < NR; ++r)
                    tma_load_2d(&tkv, &kv_full[slot], smem + OFF_KV + slot * KV_BYTES + r * 8192, col + 64 * r,
                                j * BKB);
            }
        }
    } else if (warp == BW_MMA) {
        constexpr uint32_t id_s = make_idesc_bf16(128, BKB, false, false);
        constexpr uint32_t id_q = make_idesc_bf16(128, DP, false, true);
        mbar_wait(qt_ready, 0);
        tc_fence_after();
        auto issue_sdp = [&](int it) {
            const int ks = (2 * it) % NSL, vs = (2 * it + 1) % NSL;
            mbar_wait(&kv_full[ks], ((2 * it) / NSL) & 1);
            mbar_wait(&kv_full[vs], ((2 * it + 1) / NSL) & 1);
            tc_fence_after();
            const uint32_t kb = sbase + OFF_KV + ks * KV_BYTES, vb = sbase + OFF_KV + vs * KV_BYTES;
            const uint32_t d_s = tmem + (it & 1) * 128;
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk)  // S = Q K^T, Q from TMEM: d chunk kk = 8 packed columns
                mma_bf16_ts_w(d_s, tmem + QT_COL + kk * 8, kdesc_r(kb, kk, 8192), id_s, kk > 0);
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk)  // dP = dO V^T
                mma_bf16_ts_w(d_s + 64, tmem + DOT_COL + kk * 8, kdesc_r(vb, kk, 8192), id_s, kk > 0);
            mma_commit_w(&s_full[it & 1]);
            mma_commit_w(&kv_empty[vs]);  // V_j only feeds dP
        };
        auto issue_dq = [&](int it) {
            mbar_wait(&ds_full[it & 1], (it >> 1) & 1);
            tc_fence_after();
            const int ks = (2 * it) % NSL;
            const uint32_t kb = sbase + OFF_KV + ks * KV_BYTES;
            // A = dS in TMEM: keys [16g, 16g+16) packed in S columns [16g, 16g+8) of buffer it&1
#pragma unroll
            for (int kk = 0; kk < BKB / 16; ++kk)
                mma_bf16_ts_w(tmem + DQ_COL, tmem + (it & 1) * 128 + kk * 16, mndesc_r(kb, kk, 8192), id_q,
                              (it > 0 || kk > 0));
            mma_commit_w(&kv_empty[ks]);
        };
        for (int it = 0; it < min(NB, nblk); ++it) issue_sdp(it);
        for (int it = 0; it < nblk; ++it) {
            issue_dq(it);
            if (it + NB < nblk) issue_sdp(it + NB);
        }
        mma_commit_w(dq_done);
    } else {
        const int sub = warp & 3, grp = warp >> 2;  // lanes [32 sub, +32), keys [16 grp, +16) of each block
        const int r = sub * 32 + lane;
        const int64_t q = q0 + r;
        const int q32 = (int)q, q0i = (int)q0;
        const uint32_t lo = (uint32_t)(sub * 32) << 16;
        {  // Q and dO rows -> TMEM (this warp: d elements [32 grp, 32 grp + 32) = packed columns [16 grp, +16))
            if (32 * grp < DH) {
                const int64_t width = (int64_t)(hq + 2 * hkv) * DH;
                const uint4* qs = reinterpret_cast<const uint4*>(qkv + q * width + (int64_t)h * DH + 32 * grp);
                const uint4* ds = reinterpret_cast<const uint4*>(dout + (q * hq + h) * DH + 32 * grp);
                uint32_t qv[16], dv[16];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint4 a = __ldg(qs + k), b = __ldg(ds + k);
                    qv[4 * k] = a.x; qv[4 * k + 1] = a.y; qv[4 * k + 2] = a.z; qv[4 * k + 3] = a.w;
                    dv[4 * k] = b.x; dv[4 * k + 1] = b.y; dv[4 * k + 2] = b.z; dv[4 * k + 3] = b.w;
                }
                tmem_st16(tmem + lo + QT_COL + grp * 16, qv);
                tmem_st16(tmem + lo + DOT_COL + grp * 16, dv);
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(qt_ready);
        }
        const int start = seg ? seg[q] : 0;
        const float nlse2 = -lse2v[(int64_t)h * s + q];
        const float Dq = Dv[(int64_t)h * s + q];
        const float sl2 = scale * LOG2E;
        for (int it = 0; it < nblk; ++it) {
            const int b = it & 1;
            mbar_wait(&s_full[b], (it >> 1) & 1);
            tc_fence_after();
            uint32_t sv[16], dv[16];
            tmem_ld16(tmem + lo + b * 128 + grp * 16, sv);
            tmem_ld16(tmem + lo + b * 128 + 64 + grp * 16, dv);
            tmem_ld_wait();
            const int k0 = (jb + it) * BKB + grp * 16;
            uint32_t w[8];
            auto body = [&](auto mask_c) {
                constexpr bool MASK = decltype(mask_c)::value;
                const int hi = q32 - k0, lo_ = start - k0;
                const uint64_t sl2x = f2pack(sl2, sl2), nlx = f2pack(nlse2, nlse2), dqx = f2pack(Dq, Dq);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    float x0, x1;
                    f2unpack(ffma2(f2pack(__uint_as_float(sv[2 * k]), __uint_as_float(sv[2 * k + 1])), sl2x, nlx), x0, x1);
                    float p0 = ex2(x0), p1 = ex2(x1);
                    if constexpr (MASK) {
                        p0 = (2 * k > hi || 2 * k < lo_) ? 0.f : p0;
                        p1 = (2 * k + 1 > hi || 2 * k + 1 < lo_) ? 0.f : p1;
                    }
                    const uint64_t d2 = fmul2(f2pack(p0, p1),
                                              fsub2(f2pack(__uint_as_float(dv[2 * k]), __uint_as_float(dv[2 * k + 1])), dqx));
                    float d0, d1;
                    f2unpack(d2, d0, d1);
                    w[k] = pack_bf16x2(d0, d1);
                }
            };
            if (k0 + 15 > q0i || (seg != nullptr && __any_sync(0xffffffffu, start > k0))) body(std::true_type{});
            else body(std::false_type{});
            tmem_st8(tmem + lo + b * 128 + grp * 16, w);  // over this warp's consumed S columns
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&ds_full[b]);
        }
        mbar_wait(dq_done, 0);
        tc_fence_after();
        if (32 * grp >= DH) goto dq_done_label;
        {
        bf16* dst = dqkv + (q * (hq + 2 * hkv) + h) * DH + grp * 32;
        uint32_t v[32];
        tmem_ld32(tmem + lo + DQ_COL + grp * 32, v);
        tmem_ld_wait();
        uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint4 o;
            o.x = pack_bf16x2(__uint_as_float(v[8 * k + 0]) * scale, __uint_as_float(v[8 * k + 1]) * scale);
            o.y = pack_bf16x2(__uint_as_float(v[8 * k + 2]) * scale, __uint_as_float(v[8 * k + 3]) * scale);
            o.z = pack_bf16x2(__uint_as_float(v[8 * k + 4]) * scale, __uint_as_float(v[8 * k + 5]) * scale);
            o.w = pack_bf16x2(__uint_as_float(v[8 * k + 6]) * scale, __uint_as_float(v[8 * k + 7]) * scale);
            d4[k] = o;
        }
        }
    dq_done_label:;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == BW_MMA) {
        __syncwarp();
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
constexpr int NQS = 4;                                              // Q/dO ring stages
constexpr int OFF_K = 0, OFF_V = KB_BYTES, OFF_QS = 2 * KB_BYTES;  // NQS stages x (Q, dO)
constexpr int OFF_LD = OFF_QS + NQS * 2 * QS_BYTES;                 // NQS x (lse*log2e[64], D[64]) fp32
constexpr int OFF_BAR = OFF_LD + NQS * 512;                         // P^T / dS^T live in TMEM
constexpr int SMEM = OFF_BAR + 256 + 1024;
}  // namespace dkv

// MC: CTAs (2m, 2m+1) form a cluster and stream ONE shared Q/dO sequence (the pair's union of visible q
// blocks, starting at the even CTA's first block — the odd CTA's extra blocks are fully masked), each CTA
// multicasting half of every stage into both CTAs' smem: half the L2->SM bytes per CTA.  Stage release needs
// both CTAs' MMAs (multicast commit onto qs_empty, count 2).
// KT: the K block lives in TMEM (written once by the elementwise warps) and S^T = K Q^T reads only its B
// operand from smem: M=128 N=64 MMAs run at the full tensor rate from TMEM but at 2/3 of it with both
// operands in smem (tools/micro/mma_pair_rate.cu).  The 64 columns come from single-buffering S^T:
// TMEM = S^T (64) | dP^T[2] (64 each) | K (64) | dV (128) | dK (128).  The elementwise warps release S^T
// (s_free) right after loading it and write P^T / dS^T into the consumed dP^T buffer, so S^T(it+1) and
// dP^T(it+1) run while the elementwise phase of it computes.
// DH = 64 / 32: the d=128 layout with DP = max(DH, 64) columns filled (see fwd_tc128_kernel); S^T / dP^T contract
// over DH, dV / dK run N = DP and their columns >= DH are never stored.
template <bool MC, bool KT, int DH>
__global__ void __launch_bounds__(BW_THREADS, 1)
    dkdv_tc_kernel(const __grid_constant__ CUtensorMap tkv, const __grid_constant__ CUtensorMap tq,
                   const __grid_constant__ CUtensorMap tdo, int64_t s, int hq, int hkv, const int32_t* __restrict__ seg,
                   const float* __restrict__ lse2v, const float* __restrict__ Dv, float scale, bf16* __restrict__ dqkv,
                   const bf16* __restrict__ qkv) {
    using namespace dkv;
    constexpr int DP = DH < 64 ? 64 : DH, NR = DP / 64;
    constexpr int KBB = 128 * DP * 2, QSB = BQB * DP * 2;  // bytes one K/V block / Q or dO tile load brings
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* kv_full = bar;
    uint64_t* qs_full = bar + 1;          // [NQS]
    uint64_t* qs_empty = qs_full + NQS;   // [NQS]
    uint64_t* s_full = qs_empty + NQS;    // [2]
    uint64_t* pd_full = s_full + 2;       // [2]
    uint64_t* acc_done = pd_full + 2;
    uint64_t* s_free = acc_done + 1;      // KT: the single S^T buffer has been read
    uint64_t* k_ready = s_free + 1;       // KT: K block written to TMEM
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(k_ready + 1);
    constexpr uint32_t DP_COL = 64, K_COL = 192;  // KT layout: S^T at 0, dP^T[b] at 64 + 64 b
    const int warp = warp_id(), lane = lane_id();
    const int nkb = (int)(s / 128);
    const int kb = (int)blockIdx.x;  // small kb = most work: launched first
    const int kvh = blockIdx.y;
    const int grp = hq / hkv;
    const int64_t k0 = (int64_t)kb * 128;
    (void)nkb;
    const uint32_t crank = MC ? cluster_ctarank() : 0;
    // visible q range: q >= k0 and (block-causal) start[q] <= k0 + 127 (MC: the pair's union)
    const int qb_first = (int)(((MC ? (k0 & ~int64_t(255)) : k0)) / BQB);
    int qb_last = (int)((s - 1) / BQB);
    if (seg) {
        const int64_t klast = (MC ? (k0 | 128) : k0) + 127;  // the odd CTA's last key
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
            mbar_init(&qs_empty[i], MC ? 2 : 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&pd_full[i], BW_NEW * 32);
        }
        mbar_init(acc_done, 1);
        mbar_init(s_free, BW_NEW * 32);
        mbar_init(k_ready, BW_NEW * 32);
        fence_barrier_init();
    }
    if (warp == BW_MMA) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    if (MC) cluster_sync();  // both CTAs' barriers initialised before any multicast load / remote arrive
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // provably warp-uniform: descriptor math stays in uniform registers
    const uint32_t sbase = smem_u32(smem);
    if (warp == BW_TMA) {
        if (lane == 0) {
            mbar_arrive_expect_tx(kv_full, (KT ? 1 : 2) * KBB);
            for (int r = 0; r < NR; ++r) {
                if (!KT) tma_load_2d(&tkv, kv_full, smem + OFF_K + r * 16384, (hq + kvh) * DH + 64 * r, (int)k0);
                tma_load_2d(&tkv, kv_full, smem + OFF_V + r * 16384, (hq + hkv + kvh) * DH + 64 * r, (int)k0);
            }
            int hh = kvh * grp, qblk = 0;
            for (int it = 0; it < total; ++it) {
                const int st = it % NQS;
                mbar_wait(&qs_empty[st], ((it / NQS) & 1) ^ 1);
                mbar_arrive_expect_tx(&qs_full[st], 2 * QSB + 512);
                const int qq = (qb_first + qblk) * BQB;
                const int hcur = hh;
                if (++qblk == nqb) { qblk = 0; ++hh; }
                uint8_t* base = smem + OFF_QS + st * 2 * QS_BYTES;
                if constexpr (MC) {  // rank 0 brings Q + lse, rank 1 brings dO + D, into both CTAs
                    if (crank == 0) {
                        for (int r = 0; r < NR; ++r)
                            tma_load_2d_mc(&tq, &qs_full[st], base + r * 8192, hcur * DH + 64 * r, qq, 0x3);
                        bulk_load_mc(smem + OFF_LD + st * 512, lse2v + (int64_t)hcur * s + qq, 256, &qs_full[st], 0x3);
                    } else {
                        for (int r = 0; r < NR; ++r)
                            tma_load_2d_mc(&tdo, &qs_full[st], base + QS_BYTES + r * 8192, hcur * DH + 64 * r, qq, 0x3);
                        bulk_load_mc(smem + OFF_LD + st * 512 + 256, Dv + (int64_t)hcur * s + qq, 256, &qs_full[st], 0x3);
                    }
                } else {
                    for (int r = 0; r < NR; ++r) {
                        tma_load_2d(&tq, &qs_full[st], base + r * 8192, hcur * DH + 64 * r, qq);
                        tma_load_2d(&tdo, &qs_full[st], base + QS_BYTES + r * 8192, hcur * DH + 64 * r, qq);
                    }
                    // per-column softmax statistics of this q block (lse*log2e, D) for the elementwise warps
                    bulk_load(smem + OFF_LD + st * 512, lse2v + (int64_t)hcur * s + qq, 256, &qs_full[st]);
                    bulk_load(smem + OFF_LD + st * 512 + 256, Dv + (int64_t)hcur * s + qq, 256, &qs_full[st]);
                }
            }
        }
    } else if (warp == BW_MMA) {
        {  // whole warp, converged; elect.sync inside the MMA/commit wrappers picks the issuing lane
            constexpr uint32_t id_s = make_idesc_bf16(128, BQB, false, false);
            constexpr uint32_t id_a = make_idesc_bf16(128, DP, false, true);
            mbar_wait(kv_full, 0);
            if (KT) mbar_wait(k_ready, 0);
            const uint32_t ka = sbase + OFF_K, va = sbase + OFF_V;
            auto issue_sdp_kt = [&](int it) {  // KT: S^T (A = K from TMEM) into the single S^T buffer, dP^T[it&1]
                const int st = it % NQS;
                mbar_wait(&qs_full[st], (it / NQS) & 1);
                if (it > 0) mbar_wait(s_free, (it - 1) & 1);
                tc_fence_after();
                const uint32_t qb_ = sbase + OFF_QS + st * 2 * QS_BYTES, dob = qb_ + QS_BYTES;
#pragma unroll
                for (int kk = 0; kk < DH / 16; ++kk)
                    mma_bf16_ts_w(tmem, tmem + K_COL + kk * 8, kdesc_r(qb_, kk, 8192), id_s, kk > 0);
#pragma unroll
                for (int kk = 0; kk < DH / 16; ++kk)
                    mma_bf16_ss_w(tmem + DP_COL + (it & 1) * 64, kdesc_r(va, kk, 16384), kdesc_r(dob, kk, 8192), id_s,
                                  kk > 0);
                mma_commit_w(&s_full[it & 1]);
            };
            auto issue_sdp = [&](int it) {
                const int st = it % NQS;
                mbar_wait(&qs_full[st], (it / NQS) & 1);
                tc_fence_after();
                const uint32_t qb_ = sbase + OFF_QS + st * 2 * QS_BYTES, dob = qb_ + QS_BYTES;
                const uint32_t d_s = tmem + (it & 1) * 128;
#pragma unroll
                for (int kk = 0; kk < DH / 16; ++kk)
                    mma_bf16_ss_w(d_s, kdesc_r(ka, kk, 16384), kdesc_r(qb_, kk, 8192), id_s, kk > 0);
#pragma unroll
                for (int kk = 0; kk < DH / 16; ++kk)
                    mma_bf16_ss_w(d_s + 64, kdesc_r(va, kk, 16384), kdesc_r(dob, kk, 8192), id_s, kk > 0);
                mma_commit_w(&s_full[it & 1]);
            };
            auto issue_acc = [&](int it, auto&& before) {
                const int b = it & 1, st = it % NQS;
                mbar_wait(&pd_full[b], (it >> 1) & 1);
                tc_fence_after();
                before();
                const uint32_t qb_ = sbase + OFF_QS + st * 2 * QS_BYTES, dob = qb_ + QS_BYTES;
                const uint32_t sb = KT ? tmem + DP_COL + b * 64 : tmem + b * 128;
                // A operands from TMEM: column group g packed P^T for q [16g, 16g+16) into S^T columns
                // [16g, 16g+8) and dS^T into [16g+8, 16g+16) of buffer b
#pragma unroll
                for (int kk = 0; kk < BQB / 16; ++kk)
                    mma_bf16_ts_w(tmem + 256, sb + kk * 16, mndesc_r(dob, kk, 8192), id_a, (it > 0 || kk > 0));
#pragma unroll
                for (int kk = 0; kk < BQB / 16; ++kk)
                    mma_bf16_ts_w(tmem + 384, sb + kk * 16 + 8, mndesc_r(qb_, kk, 8192), id_a,
                                  (it > 0 || kk > 0));
                if constexpr (MC) mma_commit_mc_w(&qs_empty[st], 0x3);  // the stage is free in both CTAs
                else mma_commit_w(&qs_empty[st]);
            };
            if constexpr (KT) {
                // order: S/dP(0) | per it: [wait s_free(it)] S/dP(it+1) [wait pd_full(it)] acc(it)
                if (total > 0) issue_sdp_kt(0);
                for (int it = 0; it < total; ++it) {
                    if (it + 1 < total) issue_sdp_kt(it + 1);
                    issue_acc(it, [] {});
                }
            } else {
                if (total > 0) issue_sdp(0);
                if (total > 1) issue_sdp(1);
                for (int it = 0; it < total; ++it) {
                    issue_acc(it, [] {});
                    if (it + 2 < total) issue_sdp(it + 2);
                }
            }
            mma_commit_w(acc_done);
        }
    } else {
        // elementwise: warp w: TMEM lanes (w&3)*32.., q columns [16g, 16g+16) with g = w>>2
        const int sub = warp & 3, grp = warp >> 2;
        const int r = sub * 32 + lane;  // key row
        const int64_t key = k0 + r;
        const int key32 = (int)key;  // s < 2^31 (attn_bwd_tc checks)
        const uint32_t lo = (uint32_t)(sub * 32) << 16;
        const float sl2 = scale * LOG2E;
        if constexpr (KT) {  // K row `key` -> TMEM (this warp: d elements [32 grp, +32) = packed columns [16 grp, +16))
            if (32 * grp < DH) {
                const int64_t width = (int64_t)(hq + 2 * hkv) * DH;
                const uint4* ks = reinterpret_cast<const uint4*>(qkv + key * width + (int64_t)(hq + kvh) * DH + 32 * grp);
                uint32_t kv[16];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint4 a = __ldg(ks + k);
                    kv[4 * k] = a.x; kv[4 * k + 1] = a.y; kv[4 * k + 2] = a.z; kv[4 * k + 3] = a.w;
                }
                tmem_st16(tmem + lo + K_COL + grp * 16, kv);
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(k_ready);
        }

        int qblk = 0;  // iteration it = (q head it / nqb, q block qb_first + it % nqb), kept incrementally
        for (int it = 0; it < total; ++it) {
            const int b = it & 1;
            const int qq = (qb_first + qblk) * BQB + grp * 16;
            if (++qblk == nqb) qblk = 0;
            mbar_wait(&s_full[b], (it >> 1) & 1);
            tc_fence_after();
#ifdef SPT_EXP_NO_ELEM
            tc_fence_before();
            if (KT) mbar_arrive(s_free);
            mbar_arrive(&pd_full[b]);
            continue;
#endif
            uint32_t sv[16], dv[16];
            // P^T / dS^T go back into the consumed S^T columns (KT: into the consumed dP^T buffer)
            const uint32_t sbuf = KT ? tmem + lo : tmem + lo + b * 128;
            const uint32_t dpbuf = KT ? tmem + lo + DP_COL + b * 64 : sbuf + 64;
            const uint32_t pbuf = KT ? dpbuf : sbuf;
            tmem_ld16(sbuf + grp * 16, sv);
            tmem_ld16(dpbuf + grp * 16, dv);
            tmem_ld_wait();
            if constexpr (KT) {
                tc_fence_before();
                mbar_arrive(s_free);
            }
            // the stage's statistics landed with Q/dO (s_full(it) follows the MMA's qs_full wait) and the
            // stage is not recycled before acc(it) completes, which needs this warp's arrival
            const uint32_t lsm = sbase + OFF_LD + (it % NQS) * 512 + grp * 64;
            uint32_t pw[8], sw[8];
            // warp-uniform choice between a straight-line unmasked body and the masked one (int32 limits)
            auto body = [&](auto mask_c) {
                constexpr bool MASK = decltype(mask_c)::value;
                const int lo_ = key32 - qq;  // causal: keep columns i >= key - qq
                const uint64_t sl2x = f2pack(sl2, sl2);
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    float lv[8], dd[8];
                    lds128(lsm + 32 * k, lv[0], lv[1], lv[2], lv[3]);
                    lds128(lsm + 32 * k + 16, lv[4], lv[5], lv[6], lv[7]);
                    lds128(lsm + 256 + 32 * k, dd[0], dd[1], dd[2], dd[3]);
                    lds128(lsm + 256 + 32 * k + 16, dd[4], dd[5], dd[6], dd[7]);
#pragma unroll
                    for (int e = 0; e < 8; e += 2) {
                        const int i = 8 * k + e;
                        float x0, x1;
                        f2unpack(ffma2(f2pack(__uint_as_float(sv[i]), __uint_as_float(sv[i + 1])), sl2x,
                                       f2pack(-lv[e], -lv[e + 1])),
                                 x0, x1);
                        float p0 = ex2(x0), p1 = ex2(x1);
                        if constexpr (MASK) {
                            if (i < lo_ || (seg && key32 < seg[qq + i])) p0 = 0.f;
                            if (i + 1 < lo_ || (seg && key32 < seg[qq + i + 1])) p1 = 0.f;
                        }
                        const uint64_t ds = fmul2(f2pack(p0, p1), fsub2(f2pack(__uint_as_float(dv[i]), __uint_as_float(dv[i + 1])),
                                                                        f2pack(dd[e], dd[e + 1])));
                        float s0, s1;
                        f2unpack(ds, s0, s1);
                        pw[4 * k + e / 2] = pack_bf16x2(p0, p1);
                        sw[4 * k + e / 2] = pack_bf16x2(s0, s1);
                    }
                }
            };
            // packed: the 16 queries' sample starts are nondecreasing, so seg[qq + 15] bounds them all; the
            // warp's smallest key is key32 - lane
            if (qq < key32 - r + 127 || (seg != nullptr && seg[qq + 15] > key32 - lane)) body(std::true_type{});
            else body(std::false_type{});
            tmem_st8(pbuf + grp * 16, pw);
            tmem_st8(pbuf + grp * 16 + 8, sw);
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&pd_full[b]);
        }
        // epilogue: column groups 0,1 write dV, 2,3 write dK (scaled); 64 columns each
        mbar_wait(acc_done, 0);
        tc_fence_after();
        const int64_t rs = (int64_t)(hq + 2 * hkv) * DH;
        const bool isk = grp >= 2;
        const int c0 = (grp & 1) * 64;
        bf16* dst = dqkv + key * rs + (int64_t)(isk ? (hq + kvh) : (hq + hkv + kvh)) * DH + c0;
        const float mul = isk ? scale : 1.f;
        const uint32_t acc_tm = tmem + lo + (isk ? 384 : 256) + c0;
        if (c0 >= DH) {
        } else if (total == 0) {
            uint4* d4 = reinterpret_cast<uint4*>(dst);
            for (int k = 0; k < (DH < 64 ? DH : 64) / 8; ++k) d4[k] = make_uint4(0, 0, 0, 0);
        } else {
#pragma unroll 1
            for (int c = 0; c < (DH < 64 ? DH : 64) / 32; ++c) {
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
    if (MC) cluster_sync();  // the peer's multicast loads / remote arrives target this CTA until it is done
    if (warp == BW_MMA) {
        __syncwarp();  // role branches diverged lane 0; dealloc is warp-collective (.sync.aligned)
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ dK / dV pass, CTA pair (cta_group::2)
// Same iteration space as dkdv_tc_kernel<true> (cluster (2m, 2m+1) over 256 keys, one shared Q/dO sequence),
// but every MMA is a 2-SM tcgen05.mma issued by the leader: M = 256 keys (each CTA's K / V block and TMEM
// hold its own 128), B split across the pair.  The score MMAs (S^T = K Q^T, dP^T = V dO^T, N = 64 queries)
// take queries [32c, 32c+32) of the block from CTA c, so each SM reads 4 KiB (A) + 1 KiB (B) of smem per
// K=16 step instead of 4 + 2 KiB: the smem-read cap of those MMAs rises from 32/48 to 32/40 of the tensor
// rate.  The accumulating MMAs (dV += P^T dO, dK += dS^T Q, N = d = 128) take head-dim columns
// [64c, 64c+64) from CTA c.  A stage therefore holds, per CTA and per tensor (Q, dO), its 32-query half
// (both 64-column regions) for the score MMAs and its 64-column region (all 64 queries) for the
// accumulating ones: 16 KiB, as before.  P^T / dS^T stay in each CTA's TMEM (A operand of the 2-SM MMA).
namespace dkp {
constexpr int BQB = 64;
constexpr int KB_BYTES = 128 * D * 2;                  // K or V block, 32 KiB
constexpr int STG = 32768;                             // QS(8K) DS(8K) QA(8K) DA(8K)
constexpr int ST_QS = 0, ST_DS = 8192, ST_QA = 16384, ST_DA = 24576;
constexpr int NQS = 4;
constexpr int OFF_K = 0, OFF_V = KB_BYTES, OFF_QS = 2 * KB_BYTES;
constexpr int OFF_LD = OFF_QS + NQS * STG;             // NQS x (lse*log2e[64], D[64]) fp32, per CTA
constexpr int OFF_BAR = OFF_LD + NQS * 512;
constexpr int SMEM = OFF_BAR + 256 + 1024;
}  // namespace dkp

__global__ void __launch_bounds__(BW_THREADS, 1)
    dkdv_pair_kernel(const __grid_constant__ CUtensorMap tkv, const __grid_constant__ CUtensorMap tq32,
                     const __grid_constant__ CUtensorMap tdo32, const __grid_constant__ CUtensorMap tq64,
                     const __grid_constant__ CUtensorMap tdo64, int64_t s, int hq, int hkv,
                     const int32_t* __restrict__ seg, const float* __restrict__ lse2v, const float* __restrict__ Dv,
                     float scale, bf16* __restrict__ dqkv) {
    using namespace dkp;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* kv_full = bar;              // leader's copy counts both CTAs' bytes
    uint64_t* qs_full = bar + 1;          // [NQS] leader's copy counts both CTAs' bytes
    uint64_t* qs_empty = qs_full + NQS;   // [NQS] multicast commit from the leader
    uint64_t* ld_full = qs_empty + NQS;   // [NQS] local statistics
    uint64_t* s_full = ld_full + NQS;     // [2] multicast commit
    uint64_t* pd_full = s_full + 2;       // [2] leader's copy: one arrival per elementwise warp of both CTAs
    uint64_t* acc_done = pd_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);
    const int warp = warp_id(), lane = lane_id();
    const int kb = (int)blockIdx.x;
    const int kvh = blockIdx.y;
    const int grp = hq / hkv;
    const int64_t k0 = (int64_t)kb * 128;
    const uint32_t crank = cluster_ctarank();
    const int qb_first = (int)((k0 & ~int64_t(255)) / BQB);
    int qb_last = (int)((s - 1) / BQB);
    if (seg) {
        const int64_t klast = (k0 | 128) + 127;  // the odd CTA's last key
        int64_t lo = k0 & ~int64_t(255), hi = s - 1;
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
            mbar_init(&ld_full[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&pd_full[i], 2 * BW_NEW);
        }
        mbar_init(acc_done, 1);
        fence_barrier_init();
    }
    if (warp == BW_MMA) {
        tmem_alloc_pair(tmem_slot, 512);
        tmem_relinquish_pair();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
    const uint32_t sbase = smem_u32(smem);
    if (warp == BW_TMA) {
        if (lane == 0) {
            if (crank == 0) mbar_arrive_expect_tx(kv_full, 4 * KB_BYTES);
            for (int r = 0; r < 2; ++r) {
                tma_load_2d_pair(&tkv, kv_full, smem + OFF_K + r * 16384, (hq + kvh) * D + 64 * r, (int)k0);
                tma_load_2d_pair(&tkv, kv_full, smem + OFF_V + r * 16384, (hq + hkv + kvh) * D + 64 * r, (int)k0);
            }
            int hh = kvh * grp, qblk = 0;
            for (int it = 0; it < total; ++it) {
                const int st = it % NQS;
                mbar_wait(&qs_empty[st], ((it / NQS) & 1) ^ 1);
                if (crank == 0) mbar_arrive_expect_tx(&qs_full[st], 2 * STG);
                mbar_arrive_expect_tx(&ld_full[st], 512);
                const int qq = (qb_first + qblk) * BQB;
                const int hcur = hh;
                if (++qblk == nqb) { qblk = 0; ++hh; }
                uint8_t* base = smem + OFF_QS + st * STG;
                for (int r = 0; r < 2; ++r) {
                    tma_load_2d_pair(&tq32, &qs_full[st], base + ST_QS + r * 4096, hcur * D + 64 * r, qq + 32 * (int)crank);
                    tma_load_2d_pair(&tdo32, &qs_full[st], base + ST_DS + r * 4096, hcur * D + 64 * r, qq + 32 * (int)crank);
                }
                tma_load_2d_pair(&tq64, &qs_full[st], base + ST_QA, hcur * D + 64 * (int)crank, qq);
                tma_load_2d_pair(&tdo64, &qs_full[st], base + ST_DA, hcur * D + 64 * (int)crank, qq);
                bulk_load(smem + OFF_LD + st * 512, lse2v + (int64_t)hcur * s + qq, 256, &ld_full[st]);
                bulk_load(smem + OFF_LD + st * 512 + 256, Dv + (int64_t)hcur * s + qq, 256, &ld_full[st]);
            }
        }
    } else if (warp == BW_MMA) {
        if (crank == 0) {  // whole warp, converged; elect.sync inside the wrappers picks the issuing lane
            constexpr uint32_t id_s = make_idesc_bf16(256, BQB, false, false);
            constexpr uint32_t id_a = make_idesc_bf16(256, D, false, true);
            mbar_wait(kv_full, 0);
            const uint32_t ka = sbase + OFF_K, va = sbase + OFF_V;
            auto issue_sdp = [&](int it) {
                const int st = it % NQS;
                mbar_wait(&qs_full[st], (it / NQS) & 1);
                tc_fence_after();
                const uint32_t b_ = sbase + OFF_QS + st * STG;
                const uint32_t d_s = tmem + (it & 1) * 128;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    mma_bf16_ss_pair_w(d_s, kdesc_r(ka, kk, 16384), kdesc_r(b_ + ST_QS, kk, 4096), id_s, kk > 0);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    mma_bf16_ss_pair_w(d_s + 64, kdesc_r(va, kk, 16384), kdesc_r(b_ + ST_DS, kk, 4096), id_s, kk > 0);
                mma_commit_pair_w(&s_full[it & 1], 0x3);
            };
            auto issue_acc = [&](int it) {
                const int b = it & 1, st = it % NQS;
                mbar_wait(&pd_full[b], (it >> 1) & 1);
                tc_fence_after();
                const uint32_t b_ = sbase + OFF_QS + st * STG;
#pragma unroll
                for (int kk = 0; kk < BQB / 16; ++kk)
                    mma_bf16_ts_pair_w(tmem + 256, tmem + b * 128 + kk * 16, mndesc_r(b_ + ST_DA, kk, 8192), id_a,
                                       (it > 0 || kk > 0));
#pragma unroll
                for (int kk = 0; kk < BQB / 16; ++kk)
                    mma_bf16_ts_pair_w(tmem + 384, tmem + b * 128 + kk * 16 + 8, mndesc_r(b_ + ST_QA, kk, 8192), id_a,
                                       (it > 0 || kk > 0));
                mma_commit_pair_w(&qs_empty[st], 0x3);
            };
            if (total > 0) issue_sdp(0);
            if (total > 1) issue_sdp(1);
            for (int it = 0; it < total; ++it) {
                issue_acc(it);
                if (it + 2 < total) issue_sdp(it + 2);
            }
            mma_commit_pair_w(acc_done, 0x3);
        }
    } else {
        // elementwise (both CTAs, own 128 keys): warp w: TMEM lanes (w&3)*32.., q columns [16g, 16g+16), g = w>>2
        const int sub = warp & 3, grp = warp >> 2;
        const int r = sub * 32 + lane;
        const int64_t key = k0 + r;
        const int key32 = (int)key;
        const uint32_t lo = (uint32_t)(sub * 32) << 16;
        const float sl2 = scale * LOG2E;
        const uint32_t pd_leader0 = mapa_shared(smem_u32(&pd_full[0]), 0);
        const uint32_t pd_leader1 = mapa_shared(smem_u32(&pd_full[1]), 0);
        int qblk = 0;
        for (int it = 0; it < total; ++it) {
            const int b = it & 1;
            const int qq = (qb_first + qblk) * BQB + grp * 16;
            if (++qblk == nqb) qblk = 0;
            mbar_wait(&s_full[b], (it >> 1) & 1);
            mbar_wait(&ld_full[it % NQS], (it / NQS) & 1);
            tc_fence_after();
            uint32_t sv[16], dv[16];
            tmem_ld16(tmem + lo + b * 128 + grp * 16, sv);
            tmem_ld16(tmem + lo + b * 128 + 64 + grp * 16, dv);
            tmem_ld_wait();
            const uint32_t lsm = sbase + OFF_LD + (it % NQS) * 512 + grp * 64;
            uint32_t pw[8], sw[8];
            auto body = [&](auto mask_c) {
                constexpr bool MASK = decltype(mask_c)::value;
                const int lo_ = key32 - qq;
                const uint64_t sl2x = f2pack(sl2, sl2);
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    float lv[8], dd[8];
                    lds128(lsm + 32 * k, lv[0], lv[1], lv[2], lv[3]);
                    lds128(lsm + 32 * k + 16, lv[4], lv[5], lv[6], lv[7]);
                    lds128(lsm + 256 + 32 * k, dd[0], dd[1], dd[2], dd[3]);
                    lds128(lsm + 256 + 32 * k + 16, dd[4], dd[5], dd[6], dd[7]);
#pragma unroll
                    for (int e = 0; e < 8; e += 2) {
                        const int i = 8 * k + e;
                        float x0, x1;
                        f2unpack(ffma2(f2pack(__uint_as_float(sv[i]), __uint_as_float(sv[i + 1])), sl2x,
                                       f2pack(-lv[e], -lv[e + 1])),
                                 x0, x1);
                        float p0 = ex2(x0), p1 = ex2(x1);
                        if constexpr (MASK) {
                            if (i < lo_ || (seg && key32 < seg[qq + i])) p0 = 0.f;
                            if (i + 1 < lo_ || (seg && key32 < seg[qq + i + 1])) p1 = 0.f;
                        }
                        const uint64_t ds = fmul2(f2pack(p0, p1), fsub2(f2pack(__uint_as_float(dv[i]), __uint_as_float(dv[i + 1])),
                                                                        f2pack(dd[e], dd[e + 1])));
                        float s0, s1;
                        f2unpack(ds, s0, s1);
                        pw[4 * k + e / 2] = pack_bf16x2(p0, p1);
                        sw[4 * k + e / 2] = pack_bf16x2(s0, s1);
                    }
                }
            };
            // packed: the 16 queries' sample starts are nondecreasing, so seg[qq + 15] bounds them all; the
            // warp's smallest key is key32 - lane
            if (qq < key32 - r + 127 || (seg != nullptr && seg[qq + 15] > key32 - lane)) body(std::true_type{});
            else body(std::false_type{});
            tmem_st8(tmem + lo + b * 128 + grp * 16, pw);
            tmem_st8(tmem + lo + b * 128 + grp * 16 + 8, sw);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(b ? pd_leader1 : pd_leader0);
        }
        mbar_wait(acc_done, 0);
        tc_fence_after();
        const int64_t rs = (int64_t)(hq + 2 * hkv) * D;
        const bool isk = grp >= 2;
        const int c0 = (grp & 1) * 64;
        bf16* dst = dqkv + key * rs + (int64_t)(isk ? (hq + kvh) : (hq + hkv + kvh)) * D + c0;
        const float mul = isk ? scale : 1.f;
        const uint32_t acc_tm = tmem + lo + (isk ? 384 : 256) + c0;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
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
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // the leader's MMAs read this CTA's smem / TMEM and its commits target this CTA
    if (warp == BW_MMA) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc_pair(tmem, 512);
    }
}

// ------------------------------------------------------------------ fused dK / dV / dQ pass
// One KV-outer pass computes all three gradients (5 matmuls per tile instead of the 7 of the two-pass
// scheme): on top of the dK/dV pass above, each iteration also forms dQ^T_partial = K^T dS^T (M = d,
// N = 64 queries, K = 128 keys) into the consumed dP^T columns of its TMEM buffer, with dS^T staged in
// swizzled smem as the MN-major B operand.  Four drain warps read dQ^T_partial out of TMEM, transpose it
// through smem into [q][d] rows and add it into an fp32 dQ accumulator in global memory with bulk
// reductions (cp.reduce.async.bulk .add.f32).
//
// Determinism: the contributions to a (q head, 64-query block) are added in a FIXED order —
// descending key block, i.e. the diagonal block first — enforced by a per-(head, q block) counter: key
// block kb adds only after the (j/2 - kb) key blocks above it have published theirs (acquire / release
// at gpu scope).  CTAs are launched in descending key-block order, so every CTA kb waits only on CTA
// kb + 1, which was launched earlier (no deadlock); and since CTA kb + 1 reaches any (head, q block) at
// least two iterations before CTA kb does, the waits are normally already satisfied.  Publication of an
// iteration is deferred by one iteration (bulk-group completion is waited one group behind), which keeps
// the drain warps off the L2 round-trip latency.
namespace dkvq {
constexpr int BQB = 64;
constexpr int KB_BYTES = 128 * D * 2;                                // K or V block, 32 KiB
constexpr int QS_BYTES = BQB * D * 2;                                // Q or dO tile, 16 KiB
constexpr int NQS = 3;                                               // Q/dO ring stages
constexpr int DS_BYTES = 128 * BQB * 2;                              // dS^T [128 keys][64 q] bf16, 16 KiB
constexpr int STG_BYTES = 32 * D * 4;                                // dQ staging half: 32 rows x 512 B
constexpr int OFF_K = 0, OFF_V = KB_BYTES, OFF_QS = 2 * KB_BYTES;    // NQS stages x (Q, dO)
constexpr int OFF_DS = OFF_QS + NQS * 2 * QS_BYTES;
constexpr int OFF_STG = OFF_DS + DS_BYTES;                           // 2 staging halves
constexpr int OFF_LD = OFF_STG + 2 * STG_BYTES;                      // NQS x (lse*log2e[64], D[64]) fp32
constexpr int OFF_BAR = OFF_LD + NQS * 512;
constexpr int SMEM = OFF_BAR + 256 + 1024;
constexpr int NDRAIN = 4;                                            // drain warps
constexpr int THREADS = (BW_NEW + 2 + NDRAIN) * 32;
constexpr int W_DRAIN0 = BW_NEW + 2;
static_assert(SMEM <= 232448, "dkvq smem");
}  // namespace dkvq

__device__ __forceinline__ void bulk_reduce_add_f32(float* g, uint32_t saddr, uint32_t bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(g), "r"(saddr),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_gpu_add(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void drain_bar() { asm volatile("bar.sync 1, %0;" ::"n"(dkvq::NDRAIN * 32) : "memory"); }

__global__ void __launch_bounds__(dkvq::THREADS, 1)
    dkdvq_tc_kernel(const __grid_constant__ CUtensorMap tkv, const __grid_constant__ CUtensorMap tq,
                    const __grid_constant__ CUtensorMap tdo, int64_t s, int hq, int hkv, const int32_t* __restrict__ seg,
                    const float* __restrict__ lse2v, const float* __restrict__ Dv, float scale, bf16* __restrict__ dqkv,
                    const __grid_constant__ CUtensorMap tdq, int* __restrict__ dq_cnt) {
    using namespace dkvq;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* kv_full = bar;
    uint64_t* qs_full = bar + 1;          // [NQS]
    uint64_t* qs_empty = qs_full + NQS;   // [NQS]
    uint64_t* s_full = qs_empty + NQS;    // [2]
    uint64_t* pd_full = s_full + 2;       // [2]
    uint64_t* dq_full = pd_full + 2;      // [2]
    uint64_t* dq_drained = dq_full + 2;   // [2]
    uint64_t* ds_free = dq_drained + 2;   // dS^T smem consumed by the dQ MMA
    uint64_t* acc_done = ds_free + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);
    const int warp = warp_id(), lane = lane_id();
    const int nkb = (int)(s / 128);
    const int kb = nkb - 1 - (int)blockIdx.y;  // DESCENDING key blocks (dQ ordering, see above)
    const int kvh = blockIdx.x;
    const int grp = hq / hkv;
    const int64_t k0 = (int64_t)kb * 128;
    const int nqb_all = (int)(s / BQB);
    const int qb_first = (int)(k0 / BQB);
    int qb_last = nqb_all - 1;
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
            mbar_init(&pd_full[i], BW_NEW * 32);
            mbar_init(&dq_full[i], 1);
            mbar_init(&dq_drained[i], NDRAIN * 32);
        }
        mbar_init(ds_free, 1);
        mbar_init(acc_done, 1);
        fence_barrier_init();
    }
    if (warp == BW_MMA) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
    const uint32_t sbase = smem_u32(smem);
    if (warp == BW_TMA) {
        if (lane == 0) {
            mbar_arrive_expect_tx(kv_full, 2 * KB_BYTES);
            for (int r = 0; r < 2; ++r) {
                tma_load_2d(&tkv, kv_full, smem + OFF_K + r * 16384, (hq + kvh) * D + 64 * r, (int)k0);
                tma_load_2d(&tkv, kv_full, smem + OFF_V + r * 16384, (hq + hkv + kvh) * D + 64 * r, (int)k0);
            }
            int hh = kvh * grp, qblk = 0;
            for (int it = 0; it < total; ++it) {
                const int st = it % NQS;
                mbar_wait(&qs_empty[st], ((it / NQS) & 1) ^ 1);
                mbar_arrive_expect_tx(&qs_full[st], 2 * QS_BYTES + 512);
                const int qq = (qb_first + qblk) * BQB;
                const int hcur = hh;
                if (++qblk == nqb) { qblk = 0; ++hh; }
                uint8_t* base = smem + OFF_QS + st * 2 * QS_BYTES;
                for (int r = 0; r < 2; ++r) {
                    tma_load_2d(&tq, &qs_full[st], base + r * 8192, hcur * D + 64 * r, qq);
                    tma_load_2d(&tdo, &qs_full[st], base + QS_BYTES + r * 8192, hcur * D + 64 * r, qq);
                }
                bulk_load(smem + OFF_LD + st * 512, lse2v + (int64_t)hcur * s + qq, 256, &qs_full[st]);
                bulk_load(smem + OFF_LD + st * 512 + 256, Dv + (int64_t)hcur * s + qq, 256, &qs_full[st]);
            }
        }
    } else if (warp == BW_MMA) {
        constexpr uint32_t id_s = make_idesc_bf16(128, BQB, false, false);
        constexpr uint32_t id_a = make_idesc_bf16(128, D, false, true);
        constexpr uint32_t id_q = make_idesc_bf16(128, BQB, true, true);  // dQ^T = K^T dS^T: both MN-major
        mbar_wait(kv_full, 0);
        const uint32_t ka = sbase + OFF_K, va = sbase + OFF_V, dsa = sbase + OFF_DS;
        auto issue_sdp = [&](int it) {
            const int st = it % NQS;
            mbar_wait(&qs_full[st], (it / NQS) & 1);
            tc_fence_after();
            const uint32_t qb_ = sbase + OFF_QS + st * 2 * QS_BYTES, dob = qb_ + QS_BYTES;
            const uint32_t d_s = tmem + (it & 1) * 128;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
                mma_bf16_ss_w(d_s, kdesc_r(ka, kk, 16384), kdesc_r(qb_, kk, 8192), id_s, kk > 0);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
                mma_bf16_ss_w(d_s + 64, kdesc_r(va, kk, 16384), kdesc_r(dob, kk, 8192), id_s, kk > 0);
            mma_commit_w(&s_full[it & 1]);
        };
        auto issue_acc = [&](int it) {
            const int b = it & 1, st = it % NQS;
            mbar_wait(&pd_full[b], (it >> 1) & 1);
            tc_fence_after();
            const uint32_t qb_ = sbase + OFF_QS + st * 2 * QS_BYTES, dob = qb_ + QS_BYTES;
            // dQ^T_partial[d][q] = sum_key K[key][d] dS^T[key][q] -> the dP^T columns of buffer b.  Issued
            // first so the drain warps read it out of TMEM while dV / dK execute (no bubble before the
            // next score MMAs into this buffer)
#pragma unroll
            for (int kk = 0; kk < 128 / 16; ++kk)
                mma_bf16_ss_w(tmem + b * 128 + 64, mndesc_r(ka, kk, 16384), mndesc_r(dsa, kk, 16384), id_q, kk > 0);
            mma_commit_w(&dq_full[b]);
            mma_commit_w(ds_free);
#pragma unroll
            for (int kk = 0; kk < BQB / 16; ++kk)
                mma_bf16_ts_w(tmem + 256, tmem + b * 128 + kk * 16, mndesc_r(dob, kk, 8192), id_a, (it > 0 || kk > 0));
#pragma unroll
            for (int kk = 0; kk < BQB / 16; ++kk)
                mma_bf16_ts_w(tmem + 384, tmem + b * 128 + kk * 16 + 8, mndesc_r(qb_, kk, 8192), id_a,
                              (it > 0 || kk > 0));
            mma_commit_w(&qs_empty[st]);
        };
        if (total > 0) issue_sdp(0);
        if (total > 1) issue_sdp(1);
        for (int it = 0; it < total; ++it) {
            issue_acc(it);
            if (it + 2 < total) {
                mbar_wait(&dq_drained[it & 1], (it >> 1) & 1);  // buffer's dQ^T read out of TMEM
                tc_fence_after();
                issue_sdp(it + 2);
            }
        }
        mma_commit_w(acc_done);
    } else if (warp >= W_DRAIN0) {
        // ---- drain: dQ^T_partial (TMEM lane = d) -> smem rows [q][d] -> ordered bulk add into dq_acc
        const int dw = warp & 3;  // TMEM lane quarter this warp may access (warp id mod 4)
        const int d = dw * 32 + lane;
        const uint32_t lo = (uint32_t)(dw * 32) << 16;
        const bool leader = threadIdx.x == W_DRAIN0 * 32;
        int hh = kvh * grp, qblk = 0;
        int prev_cnt_idx = -1;
        for (int it = 0; it < total; ++it) {
            const int b = it & 1;
            const int jq = qb_first + qblk;
            const int hcur = hh;
            if (++qblk == nqb) { qblk = 0; ++hh; }
            mbar_wait(&dq_full[b], (it >> 1) & 1);
            tc_fence_after();
            uint32_t v[64];
            tmem_ld32(tmem + lo + b * 128 + 64, *reinterpret_cast<uint32_t(*)[32]>(v));
            tmem_ld32(tmem + lo + b * 128 + 96, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&dq_drained[b]);
            const int cnt_idx = hcur * nqb_all + jq;
#ifdef SPT_EXP_NO_DQRED
            continue;  // experiment: drain TMEM only (no global dQ accumulation)
#endif
            for (int hf = 0; hf < 2; ++hf) {
                if (leader) bulk_wait_read<1>();  // this half's previous bulk group finished reading smem
                drain_bar();
                const uint32_t stg = sbase + OFF_STG + hf * STG_BYTES;
#pragma unroll
                for (int r = 0; r < 32; ++r)
                    asm volatile("st.shared.f32 [%0], %1;" ::"r"(stg + r * 512 + d * 4), "f"(__uint_as_float(v[hf * 32 + r]))
                                 : "memory");
                fence_proxy_async();
                drain_bar();
                if (leader) {
#ifndef SPT_EXP_NO_DQORDER
                    if (hf == 0) {
#else
                    if (false) {  // experiment: unordered (non-deterministic) accumulation
#endif
                        const int need = (jq >> 1) - kb;  // key blocks above this one, all added first
                        if (ld_acquire_gpu(dq_cnt + cnt_idx) < need) {
                            const long long t0 = clock64();
                            while (ld_acquire_gpu(dq_cnt + cnt_idx) < need) {
                                // ordering bug or lost CTA: fail loudly instead of hanging the device (~20 s)
                                if (clock64() - t0 > (1ll << 35)) {
                                    printf("[spt] dQ ordering wait timed out: kb %d head %d qblock %d need %d\n", kb,
                                           hcur, jq, need);
                                    __trap();
                                }
                            }
                        }
                    }
                    // one TMA tensor reduction: box {d 128, head 1, q 32} of dq_acc[q][head][d] += staging
                    asm volatile(
                        "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                            &tdq),
                        "r"(0), "r"(hcur), "r"(jq * BQB + hf * 32), "r"(stg)
                        : "memory");
                    bulk_commit();
                }
            }
            if (leader) {
                // publish the PREVIOUS iteration: its two bulk groups are complete once at most the two
                // groups of this iteration remain in flight
#ifdef SPT_EXP_NO_DQWAIT
                if (false) {  // experiment: never wait for reduction completion inside the loop
#else
                if (prev_cnt_idx >= 0) {
#endif
                    bulk_wait<2>();
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    red_release_gpu_add(dq_cnt + prev_cnt_idx, 1);
                }
                prev_cnt_idx = cnt_idx;
            }
        }
        if (leader && prev_cnt_idx >= 0) {
            bulk_wait<0>();
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            red_release_gpu_add(dq_cnt + prev_cnt_idx, 1);
        }
    } else {
        // elementwise: warp w: TMEM lanes (w&3)*32.., q columns [16g, 16g+16) with g = w>>2
        const int sub = warp & 3, grp4 = warp >> 2;
        const int r = sub * 32 + lane;  // key row
        const int64_t key = k0 + r;
        const int key32 = (int)key;
        const uint32_t lo = (uint32_t)(sub * 32) << 16;
        const float sl2 = scale * LOG2E;
        // dS^T smem row r: MN-major SW128 (64 q per 128 B row, 8-row atoms of 1 KiB); 16-byte chunks
        // 2*grp4 and 2*grp4+1 of this row, XOR-swizzled by (r & 7)
        const uint32_t ds_row = sbase + OFF_DS + (r >> 3) * 1024 + (r & 7) * 128;
        const uint32_t ds_c0 = ds_row + ((((uint32_t)(2 * grp4)) ^ (r & 7)) << 4);
        const uint32_t ds_c1 = ds_row + ((((uint32_t)(2 * grp4 + 1)) ^ (r & 7)) << 4);
        int qblk = 0;
        for (int it = 0; it < total; ++it) {
            const int b = it & 1;
            const int qq = (qb_first + qblk) * BQB + grp4 * 16;
            if (++qblk == nqb) qblk = 0;
            mbar_wait(&s_full[b], (it >> 1) & 1);
            tc_fence_after();
            uint32_t sv[16], dv[16];
            tmem_ld16(tmem + lo + b * 128 + grp4 * 16, sv);
            tmem_ld16(tmem + lo + b * 128 + 64 + grp4 * 16, dv);
            tmem_ld_wait();
            const uint32_t lsm = sbase + OFF_LD + (it % NQS) * 512 + grp4 * 64;
            uint32_t pw[8], sw[8];
            auto body = [&](auto mask_c) {
                constexpr bool MASK = decltype(mask_c)::value;
                const int lo_ = key32 - qq;
                const uint64_t sl2x = f2pack(sl2, sl2);
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    float lv[8], dd[8];
                    lds128(lsm + 32 * k, lv[0], lv[1], lv[2], lv[3]);
                    lds128(lsm + 32 * k + 16, lv[4], lv[5], lv[6], lv[7]);
                    lds128(lsm + 256 + 32 * k, dd[0], dd[1], dd[2], dd[3]);
                    lds128(lsm + 256 + 32 * k + 16, dd[4], dd[5], dd[6], dd[7]);
#pragma unroll
                    for (int e = 0; e < 8; e += 2) {
                        const int i = 8 * k + e;
                        float x0, x1;
                        f2unpack(ffma2(f2pack(__uint_as_float(sv[i]), __uint_as_float(sv[i + 1])), sl2x,
                                       f2pack(-lv[e], -lv[e + 1])),
                                 x0, x1);
                        float p0 = ex2(x0), p1 = ex2(x1);
                        if constexpr (MASK) {
                            if (i < lo_ || (seg && key32 < seg[qq + i])) p0 = 0.f;
                            if (i + 1 < lo_ || (seg && key32 < seg[qq + i + 1])) p1 = 0.f;
                        }
                        const uint64_t ds = fmul2(f2pack(p0, p1), fsub2(f2pack(__uint_as_float(dv[i]), __uint_as_float(dv[i + 1])),
                                                                        f2pack(dd[e], dd[e + 1])));
                        float s0, s1;
                        f2unpack(ds, s0, s1);
                        pw[4 * k + e / 2] = pack_bf16x2(p0, p1);
                        sw[4 * k + e / 2] = pack_bf16x2(s0, s1);
                    }
                }
            };
            // packed: the 16 queries' sample starts are nondecreasing, so seg[qq + 15] bounds them all; the
            // warp's smallest key is key32 - lane
            if (qq < key32 - r + 127 || (seg != nullptr && seg[qq + 15] > key32 - lane)) body(std::true_type{});
            else body(std::false_type{});
            tmem_st8(tmem + lo + b * 128 + grp4 * 16, pw);
            tmem_st8(tmem + lo + b * 128 + grp4 * 16 + 8, sw);
            // dS^T -> smem (B operand of the dQ MMA) once the previous iteration's dQ MMA has read it
            if (it > 0) mbar_wait(ds_free, (it - 1) & 1);
            sts128(ds_c0, sw[0], sw[1], sw[2], sw[3]);
            sts128(ds_c1, sw[4], sw[5], sw[6], sw[7]);
            fence_proxy_async();
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&pd_full[b]);
        }
        // epilogue: column groups 0,1 write dV, 2,3 write dK (scaled); 64 columns each
        mbar_wait(acc_done, 0);
        tc_fence_after();
        const int64_t rs = (int64_t)(hq + 2 * hkv) * D;
        const bool isk = grp4 >= 2;
        const int c0 = (grp4 & 1) * 64;
        bf16* dst = dqkv + key * rs + (int64_t)(isk ? (hq + kvh) : (hq + hkv + kvh)) * D + c0;
        const float mul = isk ? scale : 1.f;
        const uint32_t acc_tm = tmem + lo + (isk ? 384 : 256) + c0;
        if (total == 0) {
            uint4* d4 = reinterpret_cast<uint4*>(dst);
            for (int k = 0; k < 8; ++k) d4[k] = make_uint4(0, 0, 0, 0);
        } else {
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
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
    if (warp == BW_MMA) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ fused dK / dV / dQ pass, clusters of 4
// The fused pass above computes 5 matmuls per tile pair instead of 7, but sends a 32 KiB fp32 dQ partial per
// (128-key, 64-query) tile pair through L2 reductions, which sustain only ~2.2 TB/s (69 GB at s = 32K).  Here
// four CTAs with CONSECUTIVE key blocks form a cluster and walk one shared (q head, q block) sequence in
// lockstep (the union of their visible q blocks; blocks below a CTA's own keys are fully masked): each CTA
// TMA-multicasts a quarter of every Q / dO stage into all four (a quarter of the L2->SM bytes per CTA), and
// the four dQ partials of an iteration are summed through distributed shared memory before ONE reduction per
// cluster reaches global memory — CTA c adds rows [16c, 16c + 16) of the 64-query block, summing the four
// partials in descending key-block order.  A quarter of the reduction bytes, so the pass stays tensor-bound.
//
// Determinism: within a cluster the order is fixed (key block 4cl+3 down to 4cl); across
// clusters the contributions to a (q head, q block) are added in descending cluster order, enforced by the
// per-(head, q block) counter as in dkdvq_tc_kernel (4 publications per cluster).  Clusters are launched in
// descending order, so a cluster only ever waits on clusters launched before it.  Plain causal attention only
// (packed sequences keep the two-pass scheme), s % 512 == 0.
namespace dkvq4 {
constexpr int BQB = 64;
constexpr int KB_BYTES = 128 * D * 2;                             // K or V block, 32 KiB
constexpr int QS_BYTES = BQB * D * 2;                             // Q or dO tile, 16 KiB (two 8 KiB regions)
constexpr int NQS = 3;                                            // Q/dO ring stages
constexpr int DS_BYTES = 128 * BQB * 2;                           // dS^T [128 keys][64 q] bf16, 16 KiB
constexpr int STG_BYTES = BQB * D * 4;                            // this CTA's dQ partial [64 q][128 d] fp32
constexpr int OUT_BYTES = 16 * D * 4;                             // reduced rows [16 q][128 d] fp32
constexpr int OFF_K = 0, OFF_V = KB_BYTES, OFF_QS = 2 * KB_BYTES;  // NQS stages x (Q, dO)
constexpr int OFF_DS = OFF_QS + NQS * 2 * QS_BYTES;
constexpr int OFF_STG = OFF_DS + DS_BYTES;
constexpr int OFF_OUT = OFF_STG + STG_BYTES;                      // 2 buffers
constexpr int OFF_LD = OFF_OUT + 2 * OUT_BYTES;                   // NQS x (lse*log2e[64], D[64]) fp32
constexpr int OFF_BAR = OFF_LD + NQS * 512;
constexpr int SMEM = OFF_BAR + 256 + 1024;
constexpr int NDRAIN = 4;
constexpr int THREADS = (BW_NEW + 2 + NDRAIN) * 32;
constexpr int W_DRAIN0 = BW_NEW + 2;
constexpr int CL = 4;  // cluster size (key blocks per cluster)
static_assert(SMEM <= 232448, "dkvq4 smem");
}  // namespace dkvq4

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}
__device__ __forceinline__ void drain4_bar() { asm volatile("bar.sync 1, %0;" ::"n"(dkvq4::NDRAIN * 32) : "memory"); }

__global__ void __launch_bounds__(dkvq4::THREADS, 1)
    dkdvq4_kernel(const __grid_constant__ CUtensorMap tkv, const __grid_constant__ CUtensorMap tq,
                  const __grid_constant__ CUtensorMap tdo, int64_t s, int hq, int hkv, const float* __restrict__ lse2v,
                  const float* __restrict__ Dv, float scale, bf16* __restrict__ dqkv,
                  const __grid_constant__ CUtensorMap tdq, int* __restrict__ dq_cnt, int dbg) {
    // dbg (experiments only, spt_tuning_set("attn_bwd4_dbg", bits)): 1 = no dQ reduction at all, 2 = no
    // cross-cluster ordering wait, 4 = sum only this CTA's own partial (no DSMEM loads), 8 = no in-cluster
    // staging handshakes, 16 = no global reduction (TMA)
    using namespace dkvq4;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* kv_full = bar;
    uint64_t* qs_full = bar + 1;          // [NQS]
    uint64_t* qs_empty = qs_full + NQS;   // [NQS] count 4: every CTA's MMAs are done with the stage
    uint64_t* s_full = qs_empty + NQS;    // [2]
    uint64_t* pd_full = s_full + 2;       // [2]
    uint64_t* dq_full = pd_full + 2;      // [2]
    uint64_t* dq_drained = dq_full + 2;   // [2]
    uint64_t* ds_free = dq_drained + 2;
    uint64_t* acc_done = ds_free + 1;
    uint64_t* stg_full = acc_done + 1;    // count 4: every CTA's dQ partial of the iteration is staged
    uint64_t* stg_free = stg_full + 1;    // count 4: every CTA has read this CTA's staged partial
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(stg_free + 1);
    const int warp = warp_id(), lane = lane_id();
    const int nkb = (int)(s / 128);
    const uint32_t crank = cluster_ctarank();
    const int cl = nkb / CL - 1 - (int)(blockIdx.y / CL);  // DESCENDING clusters (dQ ordering)
    const int kb = cl * CL + (int)crank;
    const int kvh = blockIdx.x;
    const int grp = hq / hkv;
    const int64_t k0 = (int64_t)kb * 128;
    const int nqb_all = (int)(s / BQB);
    const int qb_first = cl * CL * 128 / BQB;  // the cluster's lowest key block's first q block
    const int nqb = nqb_all - qb_first;
    const int total = nqb * grp;
    if (threadIdx.x == 0) {
        mbar_init(kv_full, 1);
        for (int i = 0; i < NQS; ++i) {
            mbar_init(&qs_full[i], 1);
            mbar_init(&qs_empty[i], CL);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&pd_full[i], BW_NEW * 32);
            mbar_init(&dq_full[i], 1);
            mbar_init(&dq_drained[i], NDRAIN * 32);
        }
        mbar_init(ds_free, 1);
        mbar_init(acc_done, 1);
        mbar_init(stg_full, CL);
        mbar_init(stg_free, CL);
        fence_barrier_init();
    }
    if (warp == BW_MMA) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    cluster_sync();  // every CTA's barriers initialised before any multicast load / remote arrive
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
    const uint32_t sbase = smem_u32(smem);
    if (warp == BW_TMA) {
        if (lane == 0) {
            mbar_arrive_expect_tx(kv_full, 2 * KB_BYTES);
            for (int r = 0; r < 2; ++r) {
                tma_load_2d(&tkv, kv_full, smem + OFF_K + r * 16384, (hq + kvh) * D + 64 * r, (int)k0);
                tma_load_2d(&tkv, kv_full, smem + OFF_V + r * 16384, (hq + hkv + kvh) * D + 64 * r, (int)k0);
            }
            int hh = kvh * grp, qblk = 0;
            for (int it = 0; it < total; ++it) {
                const int st = it % NQS;
                mbar_wait(&qs_empty[st], ((it / NQS) & 1) ^ 1);  // all four CTAs released the stage
                mbar_arrive_expect_tx(&qs_full[st], 2 * QS_BYTES + 512);
                const int qq = (qb_first + qblk) * BQB;
                const int hcur = hh;
                if (++qblk == nqb) { qblk = 0; ++hh; }
                uint8_t* base = smem + OFF_QS + st * 2 * QS_BYTES;
                // this CTA's quarter of the stage, multicast into all four: Q / dO 64-column regions, lse / D
                const int r = (int)(crank & 1);
                if (crank < 2) {
                    tma_load_2d_mc(&tq, &qs_full[st], base + r * 8192, hcur * D + 64 * r, qq, 0xF);
                    if (crank == 0)
                        bulk_load_mc(smem + OFF_LD + st * 512, lse2v + (int64_t)hcur * s + qq, 256, &qs_full[st], 0xF);
                } else {
                    tma_load_2d_mc(&tdo, &qs_full[st], base + QS_BYTES + r * 8192, hcur * D + 64 * r, qq, 0xF);
                    if (crank == 2)
                        bulk_load_mc(smem + OFF_LD + st * 512 + 256, Dv + (int64_t)hcur * s + qq, 256, &qs_full[st],
                                     0xF);
                }
            }
        }
    } else if (warp == BW_MMA) {
        constexpr uint32_t id_s = make_idesc_bf16(128, BQB, false, false);
        constexpr uint32_t id_a = make_idesc_bf16(128, D, false, true);
        constexpr uint32_t id_q = make_idesc_bf16(128, BQB, true, true);  // dQ^T = K^T dS^T: both MN-major
        mbar_wait(kv_full, 0);
        const uint32_t ka = sbase + OFF_K, va = sbase + OFF_V, dsa = sbase + OFF_DS;
        auto issue_sdp = [&](int it) {
            const int st = it % NQS;
            mbar_wait(&qs_full[st], (it / NQS) & 1);
            tc_fence_after();
            const uint32_t qb_ = sbase + OFF_QS + st * 2 * QS_BYTES, dob = qb_ + QS_BYTES;
            const uint32_t d_s = tmem + (it & 1) * 128;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
                mma_bf16_ss_w(d_s, kdesc_r(ka, kk, 16384), kdesc_r(qb_, kk, 8192), id_s, kk > 0);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
                mma_bf16_ss_w(d_s + 64, kdesc_r(va, kk, 16384), kdesc_r(dob, kk, 8192), id_s, kk > 0);
            mma_commit_w(&s_full[it & 1]);
        };
        auto issue_acc = [&](int it) {
            const int b = it & 1, st = it % NQS;
            mbar_wait(&pd_full[b], (it >> 1) & 1);
            tc_fence_after();
            const uint32_t qb_ = sbase + OFF_QS + st * 2 * QS_BYTES, dob = qb_ + QS_BYTES;
#pragma unroll
            for (int kk = 0; kk < 128 / 16; ++kk)
                mma_bf16_ss_w(tmem + b * 128 + 64, mndesc_r(ka, kk, 16384), mndesc_r(dsa, kk, 16384), id_q, kk > 0);
            mma_commit_w(&dq_full[b]);
            mma_commit_w(ds_free);
#pragma unroll
            for (int kk = 0; kk < BQB / 16; ++kk)
                mma_bf16_ts_w(tmem + 256, tmem + b * 128 + kk * 16, mndesc_r(dob, kk, 8192), id_a, (it > 0 || kk > 0));
#pragma unroll
            for (int kk = 0; kk < BQB / 16; ++kk)
                mma_bf16_ts_w(tmem + 384, tmem + b * 128 + kk * 16 + 8, mndesc_r(qb_, kk, 8192), id_a,
                              (it > 0 || kk > 0));
            mma_commit_mc_w(&qs_empty[st], 0xF);  // the stage is free once every CTA's MMAs have read it
        };
        if (total > 0) issue_sdp(0);
        if (total > 1) issue_sdp(1);
        for (int it = 0; it < total; ++it) {
            issue_acc(it);
            if (it + 2 < total) {
                mbar_wait(&dq_drained[it & 1], (it >> 1) & 1);
                tc_fence_after();
                issue_sdp(it + 2);
            }
        }
        mma_commit_w(acc_done);
    } else if (warp >= W_DRAIN0) {
        // ---- drain: dQ^T partial (TMEM lane = d) -> staging [q][d] -> cluster sum of rows [16c, 16c+16) ->
        // ordered bulk add into dq_acc
        const int dw = warp & 3;
        const int d = dw * 32 + lane;
        const uint32_t lo = (uint32_t)(dw * 32) << 16;
        const int t = threadIdx.x - W_DRAIN0 * 32;  // 0..127
        const bool leader = t == 0;
        const uint32_t stg = sbase + OFF_STG;
        uint32_t peer_stg[CL], peer_full[CL], peer_free[CL];
#pragma unroll
        for (int j = 0; j < CL; ++j) {
            peer_stg[j] = mapa_shared(stg, (uint32_t)j);
            peer_full[j] = mapa_shared(smem_u32(stg_full), (uint32_t)j);
            peer_free[j] = mapa_shared(smem_u32(stg_free), (uint32_t)j);
        }
        const int rrow = (int)crank * 16 + (t >> 3);  // the q row of the block this thread reduces
        const int rcol = (t & 7) * 16;                // its 16 d columns
        int hh = kvh * grp, qblk = 0;
        // publication of an iteration waits for its reduction to COMPLETE in L2 (~2 us); deferring it by
        // LAG iterations keeps that round trip off the loop (the next cluster down needs (head, q block) only
        // 8 iterations after this one produced it)
        constexpr int LAG = 6;
        int pend[LAG + 1];
        int npend = 0;
        for (int it = 0; it < total; ++it) {
            const int b = it & 1;
            const int jq = qb_first + qblk;
            const int hcur = hh;
            if (++qblk == nqb) { qblk = 0; ++hh; }
            mbar_wait(&dq_full[b], (it >> 1) & 1);
            tc_fence_after();
            uint32_t v[64];
            tmem_ld32(tmem + lo + b * 128 + 64, *reinterpret_cast<uint32_t(*)[32]>(v));
            tmem_ld32(tmem + lo + b * 128 + 96, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&dq_drained[b]);
            if (dbg & 1) continue;
            // the staging buffer is free once all four CTAs read the previous iteration's partial from it
            if (it > 0 && !(dbg & 8)) mbar_wait_cluster(stg_free, (it - 1) & 1);
#pragma unroll
            for (int q = 0; q < 64; ++q)
                asm volatile("st.shared.f32 [%0], %1;" ::"r"(stg + q * 512 + d * 4), "f"(__uint_as_float(v[q])) : "memory");
            drain4_bar();  // the leader's release.cluster arrive below is cumulative over these rows
            if (leader && !(dbg & 8)) {
#pragma unroll
                for (int j = 0; j < CL; ++j) mbar_arrive_cluster(peer_full[j]);  // release.cluster: rows visible
            }
            if (!(dbg & 8)) mbar_wait_cluster(stg_full, it & 1);  // all four partials staged
            // sum rows [16c, 16c+16) over the four CTAs, descending key block (fixed order)
            float4 acc[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                acc[k] = ld_dsmem_f4(peer_stg[(dbg & 4) ? crank : CL - 1] + rrow * 512 + (rcol + 4 * k) * 4);
#pragma unroll
            for (int j = CL - 2; j >= 0 && !(dbg & 4); --j) {
                float4 x[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) x[k] = ld_dsmem_f4(peer_stg[j] + rrow * 512 + (rcol + 4 * k) * 4);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    acc[k].x += x[k].x;
                    acc[k].y += x[k].y;
                    acc[k].z += x[k].z;
                    acc[k].w += x[k].w;
                }
            }
            drain4_bar();  // every thread of this CTA finished reading the four partials
            if (leader) {
                if (!(dbg & 8)) {
#pragma unroll
                    for (int j = 0; j < CL; ++j) mbar_arrive_cluster(peer_free[j]);
                }
                bulk_wait_read<1>();  // the reduction issued two iterations ago has read out[b]
            }
            drain4_bar();
            const uint32_t out = sbase + OFF_OUT + b * OUT_BYTES;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(out + (t >> 3) * 512 + (rcol + 4 * k) * 4),
                             "f"(acc[k].x), "f"(acc[k].y), "f"(acc[k].z), "f"(acc[k].w)
                             : "memory");
            fence_proxy_async();
            drain4_bar();
            const int cnt_idx = hcur * nqb_all + jq;
            if (leader) {
                const int need = CL * ((jq * BQB / 128) / CL - cl);  // publications of the clusters above
                if (!(dbg & 2) && ld_acquire_gpu(dq_cnt + cnt_idx) < need) {
                    const long long t0 = clock64();
                    while (ld_acquire_gpu(dq_cnt + cnt_idx) < need) {
                        if (clock64() - t0 > (1ll << 35)) {
                            printf("[spt] dQ4 ordering wait timed out: cluster %d rank %u head %d qblock %d need %d\n",
                                   cl, crank, hcur, jq, need);
                            __trap();
                        }
                    }
                }
                if (!(dbg & 16))
                    asm volatile(
                        "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                            &tdq),
                        "r"(0), "r"(hcur), "r"(jq * BQB + (int)crank * 16), "r"(out)
                        : "memory");
                bulk_commit();
                pend[npend++] = cnt_idx;
                if (dbg & 32) npend = 0;
                if (npend > LAG) {  // the oldest pending iteration's reduction is complete: publish it
                    bulk_wait<LAG>();
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    red_release_gpu_add(dq_cnt + pend[0], 1);
#pragma unroll
                    for (int i = 0; i < LAG; ++i) pend[i] = pend[i + 1];
                    --npend;
                }
            }
        }
        if (leader && npend > 0) {
            bulk_wait<0>();
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            for (int i = 0; i < npend; ++i) red_release_gpu_add(dq_cnt + pend[i], 1);
        }
    } else {
        // elementwise (as dkdvq_tc_kernel; queries below this CTA's keys come out fully masked)
        const int sub = warp & 3, grp4 = warp >> 2;
        const int r = sub * 32 + lane;
        const int64_t key = k0 + r;
        const int key32 = (int)key;
        const uint32_t lo = (uint32_t)(sub * 32) << 16;
        const float sl2 = scale * LOG2E;
        const uint32_t ds_row = sbase + OFF_DS + (r >> 3) * 1024 + (r & 7) * 128;
        const uint32_t ds_c0 = ds_row + ((((uint32_t)(2 * grp4)) ^ (r & 7)) << 4);
        const uint32_t ds_c1 = ds_row + ((((uint32_t)(2 * grp4 + 1)) ^ (r & 7)) << 4);
        int qblk = 0;
        for (int it = 0; it < total; ++it) {
            const int b = it & 1;
            const int qq = (qb_first + qblk) * BQB + grp4 * 16;
            if (++qblk == nqb) qblk = 0;
            mbar_wait(&s_full[b], (it >> 1) & 1);
            tc_fence_after();
            uint32_t sv[16], dv[16];
            tmem_ld16(tmem + lo + b * 128 + grp4 * 16, sv);
            tmem_ld16(tmem + lo + b * 128 + 64 + grp4 * 16, dv);
            tmem_ld_wait();
            const uint32_t lsm = sbase + OFF_LD + (it % NQS) * 512 + grp4 * 64;
            uint32_t pw[8], sw[8];
            auto body = [&](auto mask_c) {
                constexpr bool MASK = decltype(mask_c)::value;
                const int lo_ = key32 - qq;
                const uint64_t sl2x = f2pack(sl2, sl2);
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    float lv[8], dd[8];
                    lds128(lsm + 32 * k, lv[0], lv[1], lv[2], lv[3]);
                    lds128(lsm + 32 * k + 16, lv[4], lv[5], lv[6], lv[7]);
                    lds128(lsm + 256 + 32 * k, dd[0], dd[1], dd[2], dd[3]);
                    lds128(lsm + 256 + 32 * k + 16, dd[4], dd[5], dd[6], dd[7]);
#pragma unroll
                    for (int e = 0; e < 8; e += 2) {
                        const int i = 8 * k + e;
                        float x0, x1;
                        f2unpack(ffma2(f2pack(__uint_as_float(sv[i]), __uint_as_float(sv[i + 1])), sl2x,
                                       f2pack(-lv[e], -lv[e + 1])),
                                 x0, x1);
                        float p0 = ex2(x0), p1 = ex2(x1);
                        if constexpr (MASK) {
                            if (i < lo_) p0 = 0.f;
                            if (i + 1 < lo_) p1 = 0.f;
                        }
                        const uint64_t ds = fmul2(f2pack(p0, p1), fsub2(f2pack(__uint_as_float(dv[i]), __uint_as_float(dv[i + 1])),
                                                                        f2pack(dd[e], dd[e + 1])));
                        float s0, s1;
                        f2unpack(ds, s0, s1);
                        pw[4 * k + e / 2] = pack_bf16x2(p0, p1);
                        sw[4 * k + e / 2] = pack_bf16x2(s0, s1);
                    }
                }
            };
            if (qq < key32 - r + 127) body(std::true_type{});
            else body(std::false_type{});
            tmem_st8(tmem + lo + b * 128 + grp4 * 16, pw);
            tmem_st8(tmem + lo + b * 128 + grp4 * 16 + 8, sw);
            if (it > 0) mbar_wait(ds_free, (it - 1) & 1);
            sts128(ds_c0, sw[0], sw[1], sw[2], sw[3]);
            sts128(ds_c1, sw[4], sw[5], sw[6], sw[7]);
            fence_proxy_async();
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&pd_full[b]);
        }
        mbar_wait(acc_done, 0);
        tc_fence_after();
        const int64_t rs = (int64_t)(hq + 2 * hkv) * D;
        const bool isk = grp4 >= 2;
        const int c0 = (grp4 & 1) * 64;
        bf16* dst = dqkv + key * rs + (int64_t)(isk ? (hq + kvh) : (hq + hkv + kvh)) * D + c0;
        const float mul = isk ? scale : 1.f;
        const uint32_t acc_tm = tmem + lo + (isk ? 384 : 256) + c0;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
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
    tc_fence_before();
    cluster_sync();  // no CTA leaves while a peer may still read its staged partial or multicast into it
    if (warp == BW_MMA) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// dq (bf16, inside dqkv) = dq_acc * scale
__global__ void dq_convert_kernel(const float* __restrict__ acc, int64_t s, int hq, int hkv, float scale,
                                  bf16* __restrict__ dqkv) {
    const int64_t n8 = s * hq * (D / 8);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / (D / 8), c = (i % (D / 8)) * 8;  // row = q * hq + h
        const int64_t q = row / hq, h = row % hq;
        const float4 a = reinterpret_cast<const float4*>(acc + row * D + c)[0];
        const float4 b = reinterpret_cast<const float4*>(acc + row * D + c)[1];
        uint4 w;
        w.x = pack_bf16x2(a.x * scale, a.y * scale);
        w.y = pack_bf16x2(a.z * scale, a.w * scale);
        w.z = pack_bf16x2(b.x * scale, b.y * scale);
        w.w = pack_bf16x2(b.z * scale, b.w * scale);
        *reinterpret_cast<uint4*>(dqkv + (q * (hq + 2 * hkv) + h) * D + c) = w;
    }
}

}  // namespace fatc

// debug builds (SPT_DQ_PROF): accumulated wait cycles of the dQ pass, see g_dq_prof
extern "C" int spt_debug_dq_prof(unsigned long long* out, int reset) {
#ifdef SPT_DQ_PROF
    cudaMemcpyFromSymbol(out, fatc::g_dq_prof, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(fatc::g_dq_prof, z, sizeof(z));
    }
    return 1;
#else
    (void)out;
    (void)reset;
    return 0;
#endif
}

// SPT_ATTN_KV_GROUP (run time: spt_tuning_set("attn_kv_group", v)): kv heads per dispatch group of the
// Q-outer kernels' grid, see grid_head_row.  0 (default): heads fastest while K and V of all kv heads
// (s * hkv * d * 4 bytes) fit ~L2, kv-major (1) beyond — measured (profiles/r1z3_kv_major.txt): 32K x 8 kv
// heads (134 MB) is faster heads-fastest, 48K x 8 (201 MB) and beyond kv-major (forward -10% at 48K, -13% at
// 128K; dQ pass -1.4% / -2.7%).  With one kv head all orders coincide.
int g_attn_kv_group = [] {
    const char* e = getenv("SPT_ATTN_KV_GROUP");
    return e ? atoi(e) : 0;
}();
static int kv_group(int64_t s, int hkv, int d) {
    if (g_attn_kv_group > 0) return g_attn_kv_group;
    return (double)s * hkv * d * 4 > 160e6 ? 1 : hkv;
}

// SPT_ATTN_FWD_BK128 (run time: spt_tuning_set("attn_fwd_bk128", v)): forward with 128-key blocks
// (default 1, values below fwd_bk128; 0: the 64-key double-buffered kernel).  With the P hand-off split in halves it measured -3% at 32K x 32 heads, -3.4% at
// 128K x 4, -6% at the L8 rank shape (profiles/r1z3_fwd_bk128.txt).  -1: 128-key only for s * hq >= 2^21
// (the rule before the split hand-off).
// SPT_ATTN_FWD_HYBRID=0|1 (run time: spt_tuning_set("attn_fwd_hybrid", v)): packed sequences split per tile
// pair between the 128-key and the 64-key forward.  Opt-in: with the packed mask fast path both kernels
// measured within run-to-run noise on packed sequences (tools/packed_attn_bench.py, s=128K, mean sample
// 2K / 8K / 32K), so the single 64-key launch stays the default there.
int g_attn_fwd_hybrid = [] {
    const char* e = getenv("SPT_ATTN_FWD_HYBRID");
    return e ? atoi(e) : 0;
}();

int g_attn_fwd_bk128 = [] {
    const char* e = getenv("SPT_ATTN_FWD_BK128");
    return e ? atoi(e) : 1;
}();
// Packed sequences keep the 64-key kernel: with short samples most 128-key blocks straddle a sample start
// (s=128K, mean sample 2048: 6.57 vs 4.56 ms), while long samples gain only a few % (32768: 57.7 vs 61.3 ms).
// Values: 1 (default) 128-key with every 3rd exponential pair of an unmasked block on the FMA pipe (= 13) unless
// packed, 11 the same with every exponential on MUFU (the default before the 12-warp register split), 2 128-key
// always, 0 64-key, 4 / 8 128-key + FMA-pipe exp2, 3 128-key with f16x2 exponentials, 10 + n (n = 2, 3, 4, 6, 8):
// 128-key with every n-th exponential pair of an unmasked block on the FMA pipe (packed ex2_poly2),
// -1 128-key for s * hq >= 2^21.  Returns 0 (64-key) or the 128-key kernel's POLY selector.
// The FMA-pipe share became a win once the softmax stopped spilling (12 warps, setmaxnreg): every 3rd pair
// measured -2.2% at 32K x 32q/8kv, -9.7% at 128K x 4q/1kv, -2.7% at the L8 rank shape, -9.1% at 64K x 8q/2kv
// (profiles/r2d_fwd_regsplit.txt); every 2nd / 4th pair and MUFU-only were slower.
static int fwd_bk128(int64_t s, int hq, const int32_t* seg) {
    const int v = g_attn_fwd_bk128;
    if (v == 1) return seg != nullptr ? 0 : 13;
    if (v == 11) return seg != nullptr ? 0 : 11;
    if (v == 22) return 13;  // the default 128-key form also on packed sequences
    if (v == 2) return 1;
    if (v == -1) return (double)s * hq >= 2097152.0 ? 1 : 0;
    return v;
}

// SPT_ATTN_FWD_TMEM=0|1 (run time: spt_tuning_set("attn_fwd_tmem", v)): forward with Q resident in TMEM
int g_attn_fwd_tmem = [] {
    const char* e = getenv("SPT_ATTN_FWD_TMEM");
    return e ? (e[0] == '1' ? 1 : 0) : 0;
}();

bool attn_fwd_tc(const void* qkv, int64_t s, int hq, int hkv, int d, const int32_t* seg, float scale, void* o,
                 float* lse, cudaStream_t st) {
    if ((d != 128 && d != 64 && d != 32) || s % 128 != 0) return false;
    const int64_t width = (int64_t)(hq + 2 * hkv) * d;
    CUtensorMap tq = make_tmap_bf16_2d(qkv, (uint64_t)width, (uint64_t)s, (uint64_t)width, 64, 128);
    CUtensorMap tkv = make_tmap_bf16_2d(qkv, (uint64_t)width, (uint64_t)s, (uint64_t)width, 64, 64);
    static bool attr = false;
    if (!attr) {
        SPT_CUDA(cudaFuncSetAttribute(fatc::fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, fatc::fw::SMEM));
        for (auto k : {fatc::fwd_tc128_kernel<0, 128>, fatc::fwd_tc128_kernel<1, 128>, fatc::fwd_tc128_kernel<2, 128>,
                       fatc::fwd_tc128_kernel<3, 128>, fatc::fwd_tc128_kernel<4, 128>, fatc::fwd_tc128_kernel<6, 128>,
                       fatc::fwd_tc128_kernel<8, 128>, fatc::fwd_tc128_kernel<0, 64>, fatc::fwd_tc128_kernel<0, 32>})
            SPT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, fatc::fw2::SMEM));
        SPT_CUDA(cudaFuncSetAttribute(fatc::fwd_tmem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fatc::fwt::SMEM));
        attr = true;
    }
    dim3 grid((unsigned)hq, (unsigned)((s + 255) / 256));
    if (d != 128) {  // head dims 64 / 32: the 128-key kernel (plain causal and packed) on DP = 64 columns
        CUtensorMap tkv128 = make_tmap_bf16_2d(qkv, (uint64_t)width, (uint64_t)s, (uint64_t)width, 64, 128);
        auto k = d == 64 ? fatc::fwd_tc128_kernel<0, 64> : fatc::fwd_tc128_kernel<0, 32>;
        k<<<grid, fatc::fw2::THREADS, fatc::fw2::SMEM, st>>>(tq, tkv128, s, hq, hkv, seg, scale * fatc::LOG2E, (bf16*)o, lse,
                                                        kv_group(s, hkv, d), 0);
        count_launch("attn_fwd_tc");
        SPT_CUDA(cudaGetLastError());
        return true;
    }
    const int bk128 = fwd_bk128(s, hq, seg);
    if (bk128) {
        CUtensorMap tkv128 = make_tmap_bf16_2d(qkv, (uint64_t)width, (uint64_t)s, (uint64_t)width, 64, 128);
        auto k = bk128 == 4 || bk128 == 14 ? fatc::fwd_tc128_kernel<4, 128>
                 : bk128 == 8 || bk128 == 18 ? fatc::fwd_tc128_kernel<8, 128>
                 : bk128 == 12 ? fatc::fwd_tc128_kernel<2, 128>
                 : bk128 == 13 ? fatc::fwd_tc128_kernel<3, 128>
                 : bk128 == 16 ? fatc::fwd_tc128_kernel<6, 128>
                 : bk128 == 3 ? fatc::fwd_tc128_kernel<1, 128>
                              : fatc::fwd_tc128_kernel<0, 128>;  // 1, 2, 11: every exponential on MUFU
        k<<<grid, fatc::fw2::THREADS, fatc::fw2::SMEM, st>>>(tq, tkv128, s, hq, hkv, seg, scale * fatc::LOG2E, (bf16*)o, lse,
                                                        kv_group(s, hkv, d), 0);
    } else if (seg != nullptr && g_attn_fwd_bk128 == 1 && g_attn_fwd_hybrid) {
        // packed: long-sample tile pairs on the 128-key kernel, short ones on the 64-key kernel
        CUtensorMap tkv128 = make_tmap_bf16_2d(qkv, (uint64_t)width, (uint64_t)s, (uint64_t)width, 64, 128);
        fatc::fwd_tc128_kernel<3, 128><<<grid, fatc::fw2::THREADS, fatc::fw2::SMEM, st>>>(
            tq, tkv128, s, hq, hkv, seg, scale * fatc::LOG2E, (bf16*)o, lse, kv_group(s, hkv, d), 1);
        fatc::fwd_tc_kernel<<<grid, fatc::THREADS, fatc::fw::SMEM, st>>>(tq, tkv, s, hq, hkv, seg, scale * fatc::LOG2E,
                                                                          (bf16*)o, lse, kv_group(s, hkv, d), 2);
    } else if (g_attn_fwd_tmem)
        fatc::fwd_tmem_kernel<<<grid, fatc::THREADS, fatc::fwt::SMEM, st>>>(tkv, (const bf16*)qkv, s, hq, hkv, seg,
                                                                              scale * fatc::LOG2E, (bf16*)o, lse);
    else
        fatc::fwd_tc_kernel<<<grid, fatc::THREADS, fatc::fw::SMEM, st>>>(tq, tkv, s, hq, hkv, seg, scale * fatc::LOG2E,
                                                                          (bf16*)o, lse, kv_group(s, hkv, d), 0);
    count_launch("attn_fwd_tc");
    SPT_CUDA(cudaGetLastError());
    return true;
}

// Backward scheme.  Default: two passes (dK/dV KV-outer + dQ Q-outer, 7 matmuls per tile, no global
// accumulation).  SPT_ATTN_BWD=fused selects the single KV-outer pass with ordered fp32 dQ reductions
// (5 matmuls): its compute alone runs at 20.8 ms (1059 TF/s) at s=32K, but the 69 GB of fp32 dQ
// reductions it sends through L2 (32 KiB per 128x64 tile pair) make the pass take 52.5 ms against 24.0 ms
// for the two-pass scheme (profiles/README.md).  Experiments: unordered 47.3 ms; unordered and never
// waiting for reduction completion 31.9 ms, i.e. the reductions alone sustain only ~2.2 TB/s.  Kept for
// larger tiles (fewer reduction bytes per flop) / GPUs with faster L2 reductions.
// SPT_ATTN_BWD=fused4 (or spt_tuning_set("attn_bwd", 2)): the fused pass on clusters of four key blocks
// with the dQ partials summed through distributed shared memory first (dkdvq4_kernel; plain causal,
// s % 512 == 0; anything else takes the two-pass scheme).
int g_attn_bwd = [] {
    const char* e = getenv("SPT_ATTN_BWD");
    if (!e) return SPT_ATTN_BWD_DEFAULT;
    const std::string v(e);
    return v == "fused" ? 1 : v == "fused4" ? 2 : 0;
}();
static int bwd_mode() { return g_attn_bwd; }
int g_attn_bwd4_dbg = 0;  // dkdvq4_kernel experiment bits (wrong dQ when non-zero; timing only)

// SPT_ATTN_DKDV_MC=0|1: cluster-pair multicast of the dK/dV pass's Q/dO stream (default from measurement)
static bool dkdv_multicast() {
    static const bool v = [] {
        const char* e = getenv("SPT_ATTN_DKDV_MC");
        return e ? e[0] == '1' : SPT_DKDV_MC_DEFAULT != 0;
    }();
    return v;
}

// SPT_ATTN_DQ_TMEM=0|1: dQ pass with Q / dO resident in TMEM (default from measurement); also settable at run
// time through spt_tuning_set("attn_dq_tmem", v) for in-process A/B
int g_attn_dq_tmem = [] {
    const char* e = getenv("SPT_ATTN_DQ_TMEM");
    return e ? (e[0] == '1' ? 1 : 0) : (SPT_DQ_TMEM_DEFAULT != 0 ? 1 : 0);
}();
static bool dq_tmem() { return g_attn_dq_tmem != 0; }

// SPT_ATTN_DQ_MC=0|1: cluster-pair multicast of the dQ pass's K/V stream (head pairs of a GQA group)
static bool dq_multicast() {
    static const bool v = [] {
        const char* e = getenv("SPT_ATTN_DQ_MC");
        return e ? e[0] == '1' : SPT_DQ_MC_DEFAULT != 0;
    }();
    return v;
}

#ifndef SPT_DKDV_PAIR_DEFAULT
#define SPT_DKDV_PAIR_DEFAULT 0
#endif
// SPT_ATTN_DKDV_PAIR=0|1: dK/dV pass on CTA pairs with 2-SM MMAs (dkdv_pair_kernel); also settable at run time
// through spt_tuning_set("attn_dkdv_pair", v)
int g_attn_dkdv_pair = [] {
    const char* e = getenv("SPT_ATTN_DKDV_PAIR");
    return e ? (e[0] == '1' ? 1 : 0) : (SPT_DKDV_PAIR_DEFAULT != 0 ? 1 : 0);
}();

// SPT_ATTN_DKDV_KT=0|1|2: dK/dV pass with the K block resident in TMEM: off, on, or (2, default) on for
// plain causal attention and off for packed sequences, as measured (profiles/r1z3_dkdv_variants.txt);
// spt_tuning_set("attn_dkdv_kt", v)
int g_attn_dkdv_kt = [] {
    const char* e = getenv("SPT_ATTN_DKDV_KT");
    return e ? atoi(e) : 2;
}();

size_t attn_bwd_tc_workspace(int64_t s, int hq) {
    if (bwd_mode() == 0) return 0;
    return (size_t)s * hq * fatc::D * 4 + (size_t)hq * (s / 64) * 4 + 256;
}

// Deterministic tcgen05 backward (d = 128, s % 256 == 0).  Dv = rowsum(dO * O) must be precomputed.
// ws: attn_bwd_tc_workspace bytes (fp32 dQ accumulator + per-(head, q block) ordering counters).
bool attn_bwd_tc(const void* qkv, const void* dout, const float* lse2, const float* Dv, int64_t s, int hq, int hkv,
                 int d, const int32_t* seg, float scale, void* dqkv, void* ws, cudaStream_t st) {
    if ((d != 128 && d != 64 && d != 32) || s % 128 != 0 || s >= (int64_t(1) << 31) - 256) return false;
    const int64_t width = (int64_t)(hq + 2 * hkv) * d;
    CUtensorMap t128 = make_tmap_bf16_2d(qkv, (uint64_t)width, (uint64_t)s, (uint64_t)width, 64, 128);
    CUtensorMap t64 = make_tmap_bf16_2d(qkv, (uint64_t)width, (uint64_t)s, (uint64_t)width, 64, 64);
    CUtensorMap do128 = make_tmap_bf16_2d(dout, (uint64_t)hq * d, (uint64_t)s, (uint64_t)hq * d, 64, 128);
    CUtensorMap do64 = make_tmap_bf16_2d(dout, (uint64_t)hq * d, (uint64_t)s, (uint64_t)hq * d, 64, 64);
    static bool attr = false;
    if (!attr) {
        SPT_CUDA(cudaFuncSetAttribute(fatc::dq_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fatc::dq::SMEM));
        SPT_CUDA(cudaFuncSetAttribute(fatc::dq_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fatc::dq::SMEM));
        SPT_CUDA(cudaFuncSetAttribute(fatc::dq_tmem_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fatc::dqt::SMEM));
        SPT_CUDA(cudaFuncSetAttribute(fatc::dkdv_tc_kernel<false, false, 128>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, fatc::dkv::SMEM));
        SPT_CUDA(cudaFuncSetAttribute(fatc::dkdv_tc_kernel<true, false, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fatc::dkv::SMEM));
        SPT_CUDA(cudaFuncSetAttribute(fatc::dkdv_tc_kernel<false, true, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fatc::dkv::SMEM));
        SPT_CUDA(cudaFuncSetAttribute(fatc::dkdv_tc_kernel<true, true, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fatc::dkv::SMEM));
        SPT_CUDA(cudaFuncSetAttribute(fatc::dkdvq_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fatc::dkvq::SMEM));
        SPT_CUDA(cudaFuncSetAttribute(fatc::dkdv_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fatc::dkp::SMEM));
        SPT_CUDA(cudaFuncSetAttribute(fatc::dkdvq4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fatc::dkvq4::SMEM));
        for (auto k : {fatc::dkdv_tc_kernel<false, false, 64>, fatc::dkdv_tc_kernel<true, false, 64>,
                       fatc::dkdv_tc_kernel<false, true, 64>, fatc::dkdv_tc_kernel<true, true, 64>,
                       fatc::dkdv_tc_kernel<false, false, 32>, fatc::dkdv_tc_kernel<true, false, 32>,
                       fatc::dkdv_tc_kernel<false, true, 32>, fatc::dkdv_tc_kernel<true, true, 32>})
            SPT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, fatc::dkv::SMEM));
        SPT_CUDA(cudaFuncSetAttribute(fatc::dq_tmem_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fatc::dqt::SMEM));
        SPT_CUDA(cudaFuncSetAttribute(fatc::dq_tmem_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fatc::dqt::SMEM));
        attr = true;
    }
    if (d != 128) {  // head dims 64 / 32: the default two-pass scheme (dK/dV KV-outer + dQ with Q/dO in TMEM)
        const bool kt_ = g_attn_dkdv_kt == 1 || (g_attn_dkdv_kt == 2 && seg == nullptr);
        const bool mc = dkdv_multicast() && (s / 128) % 2 == 0;
        auto kern = d == 64 ? (mc ? (kt_ ? fatc::dkdv_tc_kernel<true, true, 64> : fatc::dkdv_tc_kernel<true, false, 64>)
                                  : (kt_ ? fatc::dkdv_tc_kernel<false, true, 64> : fatc::dkdv_tc_kernel<false, false, 64>))
                            : (mc ? (kt_ ? fatc::dkdv_tc_kernel<true, true, 32> : fatc::dkdv_tc_kernel<true, false, 32>)
                                  : (kt_ ? fatc::dkdv_tc_kernel<false, true, 32> : fatc::dkdv_tc_kernel<false, false, 32>));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(s / 128), (unsigned)hkv);
        cfg.blockDim = dim3(fatc::BW_THREADS);
        cfg.dynamicSmemBytes = fatc::dkv::SMEM;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = mc ? 2 : 1;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        SPT_CUDA(cudaLaunchKernelEx(&cfg, kern, t128, t64, do64, s, hq, hkv, seg, lse2, Dv, scale, (bf16*)dqkv,
                                    (const bf16*)qkv));
        count_launch("attn_dkdv_tc");
        SPT_CUDA(cudaGetLastError());
        auto kq = d == 64 ? fatc::dq_tmem_kernel<64> : fatc::dq_tmem_kernel<32>;
        kq<<<dim3((unsigned)hq, (unsigned)(s / 128)), fatc::BW_THREADS, fatc::dqt::SMEM, st>>>(
            t64, (const bf16*)qkv, (const bf16*)dout, s, hq, hkv, seg, lse2, Dv, scale, (bf16*)dqkv, kv_group(s, hkv, d));
        count_launch("attn_dq_tc");
        SPT_CUDA(cudaGetLastError());
        return true;
    }
    if (bwd_mode() == 2 && ws != nullptr && seg == nullptr && s % 512 == 0) {
        float* dq_acc = (float*)ws;
        int* cnt = (int*)(dq_acc + (size_t)s * hq * fatc::D);
        SPT_CUDA(cudaMemsetAsync(ws, 0, attn_bwd_tc_workspace(s, hq), st));
        CUtensorMap tdq = make_tmap_f32_3d(dq_acc, fatc::D, (uint64_t)hq, (uint64_t)s, (uint64_t)fatc::D * 4,
                                           (uint64_t)hq * fatc::D * 4, fatc::D, 1, 16);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)hkv, (unsigned)(s / 128));
        cfg.blockDim = dim3(fatc::dkvq4::THREADS);
        cfg.dynamicSmemBytes = fatc::dkvq4::SMEM;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1;
        at[0].val.clusterDim.y = fatc::dkvq4::CL;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        SPT_CUDA(cudaLaunchKernelEx(&cfg, fatc::dkdvq4_kernel, t128, t64, do64, s, hq, hkv, lse2, Dv, scale,
                                    (bf16*)dqkv, tdq, cnt, g_attn_bwd4_dbg));
        count_launch("attn_dkdvq4_tc");
        SPT_CUDA(cudaGetLastError());
        fatc::dq_convert_kernel<<<148 * 8, 256, 0, st>>>(dq_acc, s, hq, hkv, scale, (bf16*)dqkv);
        count_launch("attn_dq_convert");
        SPT_CUDA(cudaGetLastError());
        return true;
    }
    if (bwd_mode() == 1 && ws != nullptr && attn_bwd_tc_workspace(s, hq) > 0 && s % 256 == 0) {
        float* dq_acc = (float*)ws;
        int* cnt = (int*)(dq_acc + (size_t)s * hq * fatc::D);
        SPT_CUDA(cudaMemsetAsync(ws, 0, attn_bwd_tc_workspace(s, hq), st));
        CUtensorMap tdq = make_tmap_f32_3d(dq_acc, fatc::D, (uint64_t)hq, (uint64_t)s, (uint64_t)fatc::D * 4,
                                           (uint64_t)hq * fatc::D * 4, fatc::D, 1, 32);
        fatc::dkdvq_tc_kernel<<<dim3((unsigned)hkv, (unsigned)(s / 128)), fatc::dkvq::THREADS, fatc::dkvq::SMEM, st>>>(
            t128, t64, do64, s, hq, hkv, seg, lse2, Dv, scale, (bf16*)dqkv, tdq, cnt);
        count_launch("attn_dkdvq_tc");
        SPT_CUDA(cudaGetLastError());
        fatc::dq_convert_kernel<<<148 * 8, 256, 0, st>>>(dq_acc, s, hq, hkv, scale, (bf16*)dqkv);
        count_launch("attn_dq_convert");
        SPT_CUDA(cudaGetLastError());
        return true;
    }
    const bool kt = g_attn_dkdv_kt == 1 || (g_attn_dkdv_kt == 2 && seg == nullptr);
    if (g_attn_dkdv_pair != 0 && (s / 128) % 2 == 0) {  // 2-SM MMAs over key-block pairs
        CUtensorMap t32 = make_tmap_bf16_2d(qkv, (uint64_t)width, (uint64_t)s, (uint64_t)width, 64, 32);
        CUtensorMap do32 = make_tmap_bf16_2d(dout, (uint64_t)hq * d, (uint64_t)s, (uint64_t)hq * d, 64, 32);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(s / 128), (unsigned)hkv);
        cfg.blockDim = dim3(fatc::BW_THREADS);
        cfg.dynamicSmemBytes = fatc::dkp::SMEM;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        SPT_CUDA(cudaLaunchKernelEx(&cfg, fatc::dkdv_pair_kernel, t128, t32, do32, t64, do64, s, hq, hkv, seg, lse2, Dv,
                                    scale, (bf16*)dqkv));
    } else if (dkdv_multicast() && (s / 128) % 2 == 0) {  // CTA pairs along the key blocks share one Q/dO stream
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(s / 128), (unsigned)hkv);
        cfg.blockDim = dim3(fatc::BW_THREADS);
        cfg.dynamicSmemBytes = fatc::dkv::SMEM;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        SPT_CUDA(cudaLaunchKernelEx(&cfg, kt ? fatc::dkdv_tc_kernel<true, true, 128> : fatc::dkdv_tc_kernel<true, false, 128>,
                                    t128, t64, do64, s, hq, hkv, seg, lse2, Dv, scale, (bf16*)dqkv, (const bf16*)qkv));
    } else {
        auto kern = kt ? fatc::dkdv_tc_kernel<false, true, 128> : fatc::dkdv_tc_kernel<false, false, 128>;
        kern<<<dim3((unsigned)(s / 128), (unsigned)hkv), fatc::BW_THREADS, fatc::dkv::SMEM, st>>>(
            t128, t64, do64, s, hq, hkv, seg, lse2, Dv, scale, (bf16*)dqkv, (const bf16*)qkv);
    }
    count_launch("attn_dkdv_tc");
    SPT_CUDA(cudaGetLastError());
    if (dq_tmem()) {  // Q / dO resident in TMEM: S and dP MMAs read only their B operand from smem
        fatc::dq_tmem_kernel<128><<<dim3((unsigned)hq, (unsigned)(s / 128)), fatc::BW_THREADS, fatc::dqt::SMEM, st>>>(
            t64, (const bf16*)qkv, (const bf16*)dout, s, hq, hkv, seg, lse2, Dv, scale, (bf16*)dqkv,
            kv_group(s, hkv, d));
    } else if (dq_multicast() && (hq / hkv) % 2 == 0) {  // head pairs of one kv head share a multicast K/V stream
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)hq, (unsigned)(s / 128));
        cfg.blockDim = dim3(fatc::BW_THREADS);
        cfg.dynamicSmemBytes = fatc::dq::SMEM;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        SPT_CUDA(cudaLaunchKernelEx(&cfg, fatc::dq_tc_kernel<true>, t128, t64, do128, s, hq, hkv, seg, lse2, Dv, scale,
                                    (bf16*)dqkv));
    } else {
        fatc::dq_tc_kernel<false><<<dim3((unsigned)hq, (unsigned)(s / 128)), fatc::BW_THREADS, fatc::dq::SMEM, st>>>(
            t128, t64, do128, s, hq, hkv, seg, lse2, Dv, scale, (bf16*)dqkv);
    }
    count_launch("attn_dq_tc");
    SPT_CUDA(cudaGetLastError());
    return true;
}

}  // namespace spt
