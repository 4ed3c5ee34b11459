// Persistent warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[m, n] = sum_k A(m, k) * B(n, k)          bf16 x bf16 -> fp32 in TMEM -> fused epilogue
//
// A(m,k) is read from A[m*lda + k] (K-major) or A[k*lda + m] (MN-major); likewise B.  That covers
// the three shapes of a Linear layer: forward (X W^T: K,K), dgrad (dY W: K,MN) and wgrad
// (dY^T X: MN,MN), so every projection of the layer step, TiledMLP and the fused logits+loss run
// on this one kernel family.
//
// Roles (256 threads, 1 CTA/SM, grid = #SMs, static round-robin tile schedule):
//   warp 0      TMA producer (one elected lane), STAGES-deep smem ring, 128B swizzle
//   warp 1      MMA issuer (one lane): tcgen05.mma M=128, N=BN, K=16, accumulators in TMEM
//   warp 2      TMEM allocator (2*BN columns: double-buffered accumulator)
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> registers -> fused op -> global
// The epilogue of tile i overlaps the MMA main loop of tile i+1 (TMEM double buffer).
#pragma once

#include "sm100.cuh"

namespace spt {

enum EpiKind : int {
    EPI_BF16 = 0,        // C(bf16) = acc * alpha (+ R)
    EPI_F32 = 1,         // C(f32) = acc * alpha (+ C if accumulate)
    EPI_SWIGLU = 2,      // columns interleaved [g32|u32]...: C(bf16)[m, n/2] = silu(g) * u
    EPI_SWIGLU_BWD = 3,  // same interleave; aux = dA[m, n/2]; C = dGU (interleaved), C2 = A = silu(g)u
    EPI_F32_STATS = 4,   // C(f32) = acc, plus per-(row, BN-column tile) softmax stats (max, sum exp(x-max))
    EPI_EXP_STATS = 5,   // per (row, BN-column tile): m = max, C(bf16) = exp(acc - m), stats (m, sum exp(acc - m)),
                         // label_logit[row] = acc at column labels[row] when it falls in the tile (fp32, exact)
};

struct EpiParams {
    void* C = nullptr;
    int64_t ldc = 0;
    const bf16* R = nullptr;  // residual (EPI_BF16), optional
    int64_t ldr = 0;
    const bf16* aux = nullptr;  // dA for EPI_SWIGLU_BWD
    int64_t ldaux = 0;
    bf16* C2 = nullptr;  // activation output for EPI_SWIGLU_BWD
    int64_t ldc2 = 0;
    int accumulate = 0;  // EPI_F32: C += acc
    float alpha = 1.f;
    float* stats = nullptr;  // EPI_F32_STATS: [M][ld_stats] float2 (max, sumexp) per 256-column tile
    int64_t ld_stats = 0;
    const int64_t* labels = nullptr;  // EPI_EXP_STATS: per-row label (column index; anything else matches none)
    float* label_logit = nullptr;     // EPI_EXP_STATS: [M] fp32 logit of the row's label
    // Tile order and L2 hints (gemm() picks them per shape, see gemm.cu raster rule): raster 0 = groups of GROUP_M
    // row blocks sweeping all column blocks, 1 = column blocks fastest (the whole B stays in L2, every A panel is
    // read once), 2 = row blocks fastest (A stays, B panels read once), 3 = groups of group_m COLUMN blocks sweeping
    // all row blocks; hint_a / hint_b: TMA L2 policy of the
    // operand loads (0 none, 1 evict_first, 2 evict_last).
    int raster = 0;
    int group_m = 0;  // raster 0: row blocks per group (0: the kernel's default, 16)
    int hint_a = 0, hint_b = 0;
    int tstore = 1;  // fp32 epilogues: 0 per-thread stores, 1 smem transpose + coalesced stores, 2 TMA store /
                     // reduce-add (1-SM kernel, EPI_F32)
};

constexpr int GEMM_BM = 128;
// per epilogue warp: a 32 x 33 fp32 tile used to transpose TMEM rows into coalesced row segments
constexpr int EPI_TBUF_FLOATS = 32 * 33;
constexpr int EPI_TBUF_BYTES = 4 * EPI_TBUF_FLOATS * 4;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 256;

// fp32 epilogue through TMA: per epilogue warp two 32 x 32 fp32 staging tiles (128B-swizzled, 4 KiB each);
// the tile goes to global memory with cp.async.bulk.tensor (store) or cp.reduce.async.bulk.tensor .add
// (accumulate: the L2 does the read-modify-write, so the epilogue never waits on a load of C)
constexpr int EPI_STG_BYTES = 4 * 2 * 32 * 32 * 4;

template <int BN>
struct GemmCfg {
    static constexpr int STAGES = BN == 256 ? 4 : 6;
    static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;  // 16 KiB
    static constexpr int B_BYTES = BN * GEMM_BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = 2 * BN;
    // [stages][barriers: 1 KiB][epilogue staging / transpose tiles: 32 KiB, 1 KiB-aligned] + alignment slack
    static constexpr int OFF_EPI = STAGES * STAGE_BYTES + 1024;
    static constexpr int SMEM_BYTES = OFF_EPI + EPI_STG_BYTES + 1024;
    static_assert(EPI_STG_BYTES >= EPI_TBUF_BYTES, "transpose tiles alias the staging region");
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t smem, int32_t c0, int32_t c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
                 "r"(smem), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, uint32_t smem, int32_t c0, int32_t c1) {
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     map),
                 "r"(smem), "r"(c0), "r"(c1)
                 : "memory");
}

// One 32 x 32 fp32 block (lane = row, v[] = 32 consecutive columns) -> 128B-swizzled staging tile -> TMA.
__device__ __forceinline__ void epi_tma_block(const CUtensorMap* tmC, uint32_t stg, int64_t row0, int64_t col0,
                                              const float* v, float alpha, bool accumulate) {
    const int lane = lane_id();
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // this buffer's last use read
    __syncwarp();
    const uint32_t rowp = stg + lane * 128;
#pragma unroll
    for (int c = 0; c < 8; ++c)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(rowp + ((c ^ (lane & 7)) << 4)),
                     "f"(v[4 * c] * alpha), "f"(v[4 * c + 1] * alpha), "f"(v[4 * c + 2] * alpha),
                     "f"(v[4 * c + 3] * alpha)
                     : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
        if (accumulate) tma_reduce_add_2d(tmC, stg, (int32_t)col0, (int32_t)row0);
        else tma_store_2d(tmC, stg, (int32_t)col0, (int32_t)row0);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
}

__device__ __forceinline__ float silu_f(float g) { return g / (1.f + __expf(-g)); }

__device__ __forceinline__ void store_bf16x32(bf16* dst, const float* v) {
    uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint4 w;
        w.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
        w.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
        w.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
        w.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
        d[q] = w;
    }
}
__device__ __forceinline__ void load_bf16x32(const bf16* src, float* v) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint4 w = s[q];
        float2 a = unpack_bf16x2(w.x), b = unpack_bf16x2(w.y), c = unpack_bf16x2(w.z), d = unpack_bf16x2(w.w);
        v[8 * q + 0] = a.x; v[8 * q + 1] = a.y; v[8 * q + 2] = b.x; v[8 * q + 3] = b.y;
        v[8 * q + 4] = c.x; v[8 * q + 5] = c.y; v[8 * q + 6] = d.x; v[8 * q + 7] = d.y;
    }
}

// Coalesced store of a 32 x 32 block held one-row-per-lane (thread `lane` owns row row0+lane, 32 columns
// in v[]): transpose through the warp's smem tile so that each store instruction writes 32 consecutive
// columns of ONE row (128 B fp32 / 64 B bf16 per instruction instead of 32 scattered rows).
template <int KIND>
__device__ __forceinline__ void store_block_t(const EpiParams& ep, float* tb, int64_t row0, int64_t col0, int64_t M,
                                              const float* v) {
    const int lane = lane_id();
#pragma unroll
    for (int i = 0; i < 32; ++i) tb[lane * 33 + i] = v[i];
    __syncwarp();
    const int nrow = (M - row0) < 32 ? (int)(M - row0) : 32;
    if constexpr (KIND == EPI_BF16) {
        bf16* base = reinterpret_cast<bf16*>(ep.C) + row0 * ep.ldc + col0 + lane;
        if (ep.R != nullptr) {
            float res[32];  // all residual loads in flight before the stores
            const bf16* rb = ep.R + row0 * ep.ldr + col0 + lane;
#pragma unroll
            for (int rr = 0; rr < 32; ++rr) res[rr] = rr < nrow ? __bfloat162float(rb[rr * ep.ldr]) : 0.f;
#pragma unroll
            for (int rr = 0; rr < 32; ++rr)
                if (rr < nrow) base[rr * ep.ldc] = __float2bfloat16_rn(tb[rr * 33 + lane] * ep.alpha + res[rr]);
        } else {
#pragma unroll
            for (int rr = 0; rr < 32; ++rr)
                if (rr < nrow) base[rr * ep.ldc] = __float2bfloat16_rn(tb[rr * 33 + lane] * ep.alpha);
        }
    } else {
        float* base = reinterpret_cast<float*>(ep.C) + row0 * ep.ldc + col0 + lane;
        if (ep.accumulate) {
            float old[32];  // all 32 loads in flight before the read-modify-write stores
#pragma unroll
            for (int rr = 0; rr < 32; ++rr) old[rr] = rr < nrow ? base[rr * ep.ldc] : 0.f;
#pragma unroll
            for (int rr = 0; rr < 32; ++rr)
                if (rr < nrow) base[rr * ep.ldc] = tb[rr * 33 + lane] * ep.alpha + old[rr];
        } else {
#pragma unroll
            for (int rr = 0; rr < 32; ++rr)
                if (rr < nrow) base[rr * ep.ldc] = tb[rr * 33 + lane] * ep.alpha;
        }
    }
    __syncwarp();
}

// One 32-column chunk (or a g/u pair of chunks for the SwiGLU kinds) of one row.
template <int KIND>
__device__ __forceinline__ void epilogue_chunk(const EpiParams& ep, int64_t row, int64_t col, const uint32_t (&r0)[32],
                                               const uint32_t (&r1)[32]) {
    float v[32];
    if constexpr (KIND == EPI_BF16) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t* r = h ? r1 : r0;
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * ep.alpha;
            if (ep.R != nullptr) {
                float rr[32];
                load_bf16x32(ep.R + row * ep.ldr + col + 32 * h, rr);
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] += rr[i];
            }
            store_bf16x32(reinterpret_cast<bf16*>(ep.C) + row * ep.ldc + col + 32 * h, v);
        }
    } else if constexpr (KIND == EPI_F32 || KIND == EPI_F32_STATS) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t* r = h ? r1 : r0;
            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(ep.C) + row * ep.ldc + col + 32 * h);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                float4 o = make_float4(__uint_as_float(r[4 * q]) * ep.alpha, __uint_as_float(r[4 * q + 1]) * ep.alpha,
                                       __uint_as_float(r[4 * q + 2]) * ep.alpha, __uint_as_float(r[4 * q + 3]) * ep.alpha);
                if (ep.accumulate) {
                    float4 c = dst[q];
                    o.x += c.x; o.y += c.y; o.z += c.z; o.w += c.w;
                }
                dst[q] = o;
            }
        }
    } else if constexpr (KIND == EPI_SWIGLU) {
        // r0 = g[j..j+32), r1 = u[j..j+32) with j = col/2
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const float g = __uint_as_float(r0[i]), u = __uint_as_float(r1[i]);
            v[i] = silu_f(g) * u;
        }
        store_bf16x32(reinterpret_cast<bf16*>(ep.C) + row * ep.ldc + col / 2, v);
    } else if constexpr (KIND == EPI_SWIGLU_BWD) {
        float da[32], dg[32], du[32];
        load_bf16x32(ep.aux + row * ep.ldaux + col / 2, da);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const float g = __uint_as_float(r0[i]), u = __uint_as_float(r1[i]);
            const float sg = 1.f / (1.f + __expf(-g));
            const float si = g * sg;
            v[i] = si * u;
            du[i] = da[i] * si;
            dg[i] = da[i] * u * sg * (1.f + g * (1.f - sg));
        }
        store_bf16x32(ep.C2 + row * ep.ldc2 + col / 2, v);
        bf16* dgu = reinterpret_cast<bf16*>(ep.C) + row * ep.ldc + col;
        store_bf16x32(dgu, dg);
        store_bf16x32(dgu + 32, du);
    }
}

// EPI_EXP_STATS for one accumulator row (thread = TMEM lane = row) of a BN-column tile: pass 1 reads the row's
// columns out of TMEM for the max m (and picks the label's logit), pass 2 re-reads them and stores e = exp(x - m)
// as bf16 together with sum(e).  e is in (0, 1] with its largest entries exactly where the probabilities are,
// so bf16 keeps them to 2^-9 relative; the loss uses the fp32 label logit, never a rounded value.  The fp32
// logits never reach memory (the CE pass needs only e, the stats and the label logit).  tcgen05.ld is
// warp-collective: every lane runs both passes, only the stores are predicated on the row.
template <int BN>
__device__ __forceinline__ void exp_stats_tile(const EpiParams& ep, uint32_t tbase, int64_t row, int nb, int64_t M,
                                               int64_t N) {
    const int64_t col0 = (int64_t)nb * BN;
    const int64_t lab = row < M ? ep.labels[row] : -1;
    float mx = -INFINITY, ll = 0.f;
    bool has = false;
#pragma unroll 1
    for (int c = 0; c < BN && col0 + c < N; c += 64) {
        uint32_t r0[32], r1[32];
        tmem_ld32(tbase + c, r0);
        tmem_ld32(tbase + c + 32, r1);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) mx = fmaxf(mx, fmaxf(__uint_as_float(r0[i]), __uint_as_float(r1[i])));
        const int64_t j = lab - (col0 + c);
        if (j >= 0 && j < 64) {
            has = true;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                if (j == i) ll = __uint_as_float(r0[i]);
                if (j == i + 32) ll = __uint_as_float(r1[i]);
            }
        }
    }
    float sum = 0.f;
#pragma unroll 1
    for (int c = 0; c < BN && col0 + c < N; c += 64) {
        uint32_t r0[32], r1[32];
        tmem_ld32(tbase + c, r0);
        tmem_ld32(tbase + c + 32, r1);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t* r = h ? r1 : r0;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                v[i] = __expf(__uint_as_float(r[i]) - mx);
                sum += v[i];
            }
            if (row < M) store_bf16x32(reinterpret_cast<bf16*>(ep.C) + row * ep.ldc + col0 + c + 32 * h, v);
        }
    }
    if (row < M && col0 < N) {
        reinterpret_cast<float2*>(ep.stats)[row * ep.ld_stats + nb] = make_float2(mx, sum);
        if (has) ep.label_logit[row] = ll;
    }
}

template <int BN, bool A_MN, bool B_MN, int KIND>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                   int K, EpiParams ep, const __grid_constant__ CUtensorMap tmC) {
    using Cfg = GemmCfg<BN>;
    constexpr int STAGES = Cfg::STAGES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* tbuf = reinterpret_cast<float*>(smem + Cfg::OFF_EPI);  // epilogue transpose tiles (non-TMA paths)

    const int warp = warp_id(), lane = lane_id();
    const int num_m = (M + GEMM_BM - 1) / GEMM_BM;
    const int num_n = (N + BN - 1) / BN;
    const int ntiles = num_m * num_n;
    const int nk = (K + GEMM_BK - 1) / GEMM_BK;
    const int GROUP_M = ep.group_m > 0 ? ep.group_m : 16;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 128);
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    if (warp == 2) {
        tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    auto tile_coords = [&](int t, int& mb, int& nb) {
        if (ep.raster == 1) {
            mb = t / num_n;
            nb = t - mb * num_n;
            return;
        }
        if (ep.raster == 2) {
            nb = t / num_m;
            mb = t - nb * num_m;
            return;
        }
        if (ep.raster == 3) {  // groups of GROUP_M column blocks sweeping all row blocks (B slice stays in L2)
            const int per_group_n = GROUP_M * num_m;
            const int gid = t / per_group_n;
            const int first_n = gid * GROUP_M;
            const int gsz = min(num_n - first_n, GROUP_M);
            const int in = t % per_group_n;
            nb = first_n + in % gsz;
            mb = in / gsz;
            return;
        }
        const int per_group = GROUP_M * num_n;
        const int gid = t / per_group;
        const int first_m = gid * GROUP_M;
        const int gsz = min(num_m - first_m, GROUP_M);
        const int in = t % per_group;
        mb = first_m + in % gsz;
        nb = in / gsz;
    };

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint64_t pol_a = l2_policy(ep.hint_a), pol_b = l2_policy(ep.hint_b);
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int mb, nb;
                tile_coords(t, mb, nb);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sA = smem + stage * Cfg::STAGE_BYTES;
                    uint8_t* sB = sA + Cfg::A_BYTES;
                    mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
                    if constexpr (!A_MN) {
                        tma_load_2d_hint(&tmA, &full[stage], sA, kb * GEMM_BK, mb * GEMM_BM, pol_a);
                    } else {
#pragma unroll
                        for (int i = 0; i < GEMM_BM / 64; ++i)
                            tma_load_2d_hint(&tmA, &full[stage], sA + i * 8192, mb * GEMM_BM + i * 64, kb * GEMM_BK, pol_a);
                    }
                    if constexpr (!B_MN) {
                        tma_load_2d_hint(&tmB, &full[stage], sB, kb * GEMM_BK, nb * BN, pol_b);
                    } else {
#pragma unroll
                        for (int i = 0; i < BN / 64; ++i)
                            tma_load_2d_hint(&tmB, &full[stage], sB + i * 8192, nb * BN + i * 64, kb * GEMM_BK, pol_b);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = make_idesc_bf16(GEMM_BM, BN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(smem + stage * Cfg::STAGE_BYTES);
                    const uint32_t b0 = a0 + Cfg::A_BYTES;
                    const uint64_t ad0 = A_MN ? make_sdesc_sw128(a0, 8192, 1024) : make_sdesc_sw128(a0, 16, 1024);
                    const uint64_t bd0 = B_MN ? make_sdesc_sw128(b0, 8192, 1024) : make_sdesc_sw128(b0, 16, 1024);
#pragma unroll
                    for (int k = 0; k < GEMM_BK / 16; ++k) {
                        // K step of 16: +32 B (K-major) or +16 rows = 2048 B (MN-major), in 16-byte units
                        const uint64_t ad = ad0 + (A_MN ? 128 : 2) * k;
                        const uint64_t bd = bd0 + (B_MN ? 128 : 2) * k;
                        mma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
                    }
                    mma_commit(&empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        const int sub = warp & 3;  // TMEM lane quarter this warp may access
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            int mb, nb;
            tile_coords(t, mb, nb);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int64_t row = (int64_t)mb * GEMM_BM + sub * 32 + lane;
            const uint32_t tbase = tmem_base + ((uint32_t)(sub * 32) << 16) + acc * BN;
            float st_m = -INFINITY, st_s = 0.f;  // EPI_F32_STATS running (max, sum exp) over the tile row
            if constexpr (KIND == EPI_EXP_STATS) exp_stats_tile<BN>(ep, tbase, row, nb, M, N);
#pragma unroll 1
            for (int c = 0; c < (KIND == EPI_EXP_STATS ? 0 : BN); c += 64) {
                const int64_t col = (int64_t)nb * BN + c;
                uint32_t r0[32], r1[32];
                tmem_ld32(tbase + c, r0);
                tmem_ld32(tbase + c + 32, r1);
                tmem_ld_wait();
                if constexpr (KIND == EPI_F32) {
                    if (col < N && ep.tstore == 2) {  // TMA store / reduce-add (rows and columns clipped by TMA)
                        const uint32_t stg = smem_u32(smem + Cfg::OFF_EPI) + (uint32_t)(warp & 3) * 8192u;
                        const int64_t row0 = row - lane;
                        epi_tma_block(&tmC, stg, row0, col, reinterpret_cast<const float*>(r0), ep.alpha,
                                      ep.accumulate != 0);
                        epi_tma_block(&tmC, stg + 4096, row0, col + 32, reinterpret_cast<const float*>(r1), ep.alpha,
                                      ep.accumulate != 0);
                    }
                }
                if constexpr (KIND == EPI_F32 || KIND == EPI_F32_STATS) {
                    if (col < N && ep.tstore == 1) {  // warp-uniform (N % 64 == 0); rows bounds-checked inside
                        float* tb = tbuf + (warp & 3) * EPI_TBUF_FLOATS;
                        const int64_t row0 = row - lane;
                        store_block_t<KIND>(ep, tb, row0, col, M, reinterpret_cast<const float*>(r0));
                        store_block_t<KIND>(ep, tb, row0, col + 32, M, reinterpret_cast<const float*>(r1));
                    }
                }
                if (row < M && col < N) {
                    if (!(KIND == EPI_F32 || KIND == EPI_F32_STATS) || !ep.tstore)
                        epilogue_chunk<KIND>(ep, row, col, r0, r1);
                    if constexpr (KIND == EPI_F32_STATS) {
                        float mx = st_m;
#pragma unroll
                        for (int i = 0; i < 32; ++i) mx = fmaxf(mx, fmaxf(__uint_as_float(r0[i]), __uint_as_float(r1[i])));
                        float acc_s = st_s * __expf(st_m - mx);
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            acc_s += __expf(__uint_as_float(r0[i]) - mx) + __expf(__uint_as_float(r1[i]) - mx);
                        st_m = mx;
                        st_s = acc_s;
                    }
                }
            }
            if constexpr (KIND == EPI_F32_STATS) {
                if (row < M && (int64_t)nb * BN < N)
                    reinterpret_cast<float2*>(ep.stats)[row * ep.ld_stats + nb] = make_float2(st_m, st_s);
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if constexpr (KIND == EPI_F32) {
            if (ep.tstore == 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        __syncwarp();  // role branches diverged lane 0; dealloc is warp-collective (.sync.aligned)
        tc_fence_after();
        tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
}

// ----------------------------------------------------------------------------------------------
// CTA-pair variant (cluster of 2, tcgen05.mma.cta_group::2): cluster tile 256 x BN, each CTA holds
// 128 rows of A and BN/2 rows of B per stage and receives 128 rows x BN of the accumulator in its
// own TMEM.  Per SM this halves the B-operand smem traffic and TMA bytes per flop, and doubles the
// prefetch distance of the same smem budget.  The leader (rank 0) issues all MMAs; both CTAs run
// producer and epilogue roles.  Stage/accumulator release is multicast to both CTAs.
template <int BN>
struct Gemm2Cfg {
    static constexpr int STAGES = 6;
    static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;        // 16 KiB (this CTA's 128 rows)
    static constexpr int B_BYTES = (BN / 2) * GEMM_BK * 2;       // this CTA's half of B
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = 2 * BN;
    static constexpr int OFF_EPI = STAGES * STAGE_BYTES + 1024;   // staging / transpose tiles, 1 KiB-aligned
    static constexpr int SMEM_BYTES = OFF_EPI + EPI_STG_BYTES + 1024;
};

template <int BN, bool A_MN, bool B_MN, int KIND>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                    int K, EpiParams ep, const __grid_constant__ CUtensorMap tmC) {
    using Cfg = Gemm2Cfg<BN>;
    constexpr int STAGES = Cfg::STAGES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* tbuf = reinterpret_cast<float*>(smem + Cfg::OFF_EPI);  // epilogue transpose tiles (non-TMA paths)

    const int warp = warp_id(), lane = lane_id();
    const uint32_t rank = cluster_ctarank();
    const int num_m = (M + 2 * GEMM_BM - 1) / (2 * GEMM_BM);
    const int num_n = (N + BN - 1) / BN;
    const int ntiles = num_m * num_n;
    const int nk = (K + GEMM_BK - 1) / GEMM_BK;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    // 16 cluster rows: the logits GEMM's x-tile group (16 x 256 rows x K=4096, 32 MB) stays in L2 while all of W_lm
    // streams past it twice per loss tile instead of four times
    const int GROUP_M = ep.group_m > 0 ? ep.group_m : 16;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is the one used)
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    if (warp == 2) {
        tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);
        tmem_relinquish_pair();
    }
    tc_fence_before();
    cluster_sync();  // barriers of both CTAs initialised before any remote arrive / TMA
    // The cluster barrier (release / acquire) already orders tcgen05.alloc's write of the slot; the CTA barrier
    // makes that ordering visible to compute-sanitizer's racecheck too (it models bar.sync, not barrier.cluster),
    // once per kernel.
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    auto tile_coords = [&](int t, int& mb, int& nb) {
        if (ep.raster == 1) {
            mb = t / num_n;
            nb = t - mb * num_n;
            return;
        }
        if (ep.raster == 2) {
            nb = t / num_m;
            mb = t - nb * num_m;
            return;
        }
        if (ep.raster == 3) {  // groups of GROUP_M column blocks sweeping all row blocks (B slice stays in L2)
            const int per_group_n = GROUP_M * num_m;
            const int gid = t / per_group_n;
            const int first_n = gid * GROUP_M;
            const int gsz = min(num_n - first_n, GROUP_M);
            const int in = t % per_group_n;
            nb = first_n + in % gsz;
            mb = in / gsz;
            return;
        }
        const int per_group = GROUP_M * num_n;
        const int gid = t / per_group;
        const int first_m = gid * GROUP_M;
        const int gsz = min(num_m - first_m, GROUP_M);
        const int in = t % per_group;
        mb = first_m + in % gsz;
        nb = in / gsz;
    };

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint64_t pol_a = l2_policy(ep.hint_a), pol_b = l2_policy(ep.hint_b);
            for (int t = cid; t < ntiles; t += ncl) {
                int mb, nb;
                tile_coords(t, mb, nb);
                const int m0 = mb * 2 * GEMM_BM + rank * GEMM_BM;
                const int n0 = nb * BN + rank * (BN / 2);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sA = smem + stage * Cfg::STAGE_BYTES;
                    uint8_t* sB = sA + Cfg::A_BYTES;
                    if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * Cfg::STAGE_BYTES);
                    if constexpr (!A_MN) {
                        tma_load_2d_pair_hint(&tmA, &full[stage], sA, kb * GEMM_BK, m0, pol_a);
                    } else {
#pragma unroll
                        for (int i = 0; i < GEMM_BM / 64; ++i)
                            tma_load_2d_pair_hint(&tmA, &full[stage], sA + i * 8192, m0 + i * 64, kb * GEMM_BK, pol_a);
                    }
                    if constexpr (!B_MN) {
                        tma_load_2d_pair_hint(&tmB, &full[stage], sB, kb * GEMM_BK, n0, pol_b);
                    } else {
#pragma unroll
                        for (int i = 0; i < BN / 128; ++i)
                            tma_load_2d_pair_hint(&tmB, &full[stage], sB + i * 8192, n0 + i * 64, kb * GEMM_BK, pol_b);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = make_idesc_bf16(2 * GEMM_BM, BN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = cid; t < ntiles; t += ncl) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(smem + stage * Cfg::STAGE_BYTES);
                    const uint32_t b0 = a0 + Cfg::A_BYTES;
                    const uint64_t ad0 = A_MN ? make_sdesc_sw128(a0, 8192, 1024) : make_sdesc_sw128(a0, 16, 1024);
                    const uint64_t bd0 = B_MN ? make_sdesc_sw128(b0, 8192, 1024) : make_sdesc_sw128(b0, 16, 1024);
#pragma unroll
                    for (int k = 0; k < GEMM_BK / 16; ++k)
                        mma_bf16_ss_pair(d_tmem, ad0 + (A_MN ? 128 : 2) * k, bd0 + (B_MN ? 128 : 2) * k, idesc,
                                         (kb | k) != 0);
                    mma_commit_pair(&empty[stage], 0x3);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit_pair(&tfull[acc], 0x3);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        const int sub = warp & 3;
        int acc = 0;
        uint32_t acc_phase = 0;
        const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
        const uint32_t tempty_leader1 = mapa_shared(smem_u32(&tempty[1]), 0);
        for (int t = cid; t < ntiles; t += ncl) {
            int mb, nb;
            tile_coords(t, mb, nb);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int64_t row = (int64_t)mb * 2 * GEMM_BM + rank * GEMM_BM + sub * 32 + lane;
            const uint32_t tbase = tmem_base + ((uint32_t)(sub * 32) << 16) + acc * BN;
            float st_m = -INFINITY, st_s = 0.f;  // EPI_F32_STATS running (max, sum exp) over the tile row
            if constexpr (KIND == EPI_EXP_STATS) exp_stats_tile<BN>(ep, tbase, row, nb, M, N);
#pragma unroll 1
            for (int c = 0; c < (KIND == EPI_EXP_STATS ? 0 : BN); c += 64) {
                const int64_t col = (int64_t)nb * BN + c;
                uint32_t r0[32], r1[32];
                tmem_ld32(tbase + c, r0);
                tmem_ld32(tbase + c + 32, r1);
                tmem_ld_wait();
                if constexpr (KIND == EPI_F32) {
                    if (col < N && ep.tstore == 2) {  // TMA store / reduce-add (rows and columns clipped by TMA)
                        const uint32_t stg = smem_u32(smem + Cfg::OFF_EPI) + (uint32_t)(warp & 3) * 8192u;
                        const int64_t row0 = row - lane;
                        epi_tma_block(&tmC, stg, row0, col, reinterpret_cast<const float*>(r0), ep.alpha,
                                      ep.accumulate != 0);
                        epi_tma_block(&tmC, stg + 4096, row0, col + 32, reinterpret_cast<const float*>(r1), ep.alpha,
                                      ep.accumulate != 0);
                    }
                }
                if constexpr (KIND == EPI_F32 || KIND == EPI_F32_STATS) {
                    if (col < N && ep.tstore == 1) {  // warp-uniform (N % 64 == 0); rows bounds-checked inside
                        float* tb = tbuf + (warp & 3) * EPI_TBUF_FLOATS;
                        const int64_t row0 = row - lane;
                        store_block_t<KIND>(ep, tb, row0, col, M, reinterpret_cast<const float*>(r0));
                        store_block_t<KIND>(ep, tb, row0, col + 32, M, reinterpret_cast<const float*>(r1));
                    }
                }
                if (row < M && col < N) {
                    if (!(KIND == EPI_F32 || KIND == EPI_F32_STATS) || !ep.tstore)
                        epilogue_chunk<KIND>(ep, row, col, r0, r1);
                    if constexpr (KIND == EPI_F32_STATS) {
                        float mx = st_m;
#pragma unroll
                        for (int i = 0; i < 32; ++i) mx = fmaxf(mx, fmaxf(__uint_as_float(r0[i]), __uint_as_float(r1[i])));
                        float acc_s = st_s * __expf(st_m - mx);
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            acc_s += __expf(__uint_as_float(r0[i]) - mx) + __expf(__uint_as_float(r1[i]) - mx);
                        st_m = mx;
                        st_s = acc_s;
                    }
                }
            }
            if constexpr (KIND == EPI_F32_STATS) {
                if (row < M && (int64_t)nb * BN < N)
                    reinterpret_cast<float2*>(ep.stats)[row * ep.ld_stats + nb] = make_float2(st_m, st_s);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if constexpr (KIND == EPI_F32) {
            if (ep.tstore == 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // peer TMEM is written by the leader's MMAs: both CTAs done before dealloc
    if (warp == 2) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
    }
}

}  // namespace spt
