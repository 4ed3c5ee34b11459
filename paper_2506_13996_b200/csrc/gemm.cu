// Host side of the tcgen05 GEMM: TMA descriptor encoding, instantiation dispatch, C-ABI entry.
#include <cstdlib>
#include <mutex>
#include <string>

#include "common.h"
#include "gemm.cuh"
#include "launch.h"
#include "prof.h"

namespace spt {

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t encode_fn() {
    static PFN_encodeTiled_t fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled_t>(p);
    });
    SPT_CHECK(fn != nullptr, SPT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
    return fn;
}

// 2-D bf16 tensor map over a row-major [outer, inner] view with row pitch ld (elements), SW128.
CUtensorMap make_tmap_bf16_2d(const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                              uint32_t box_outer) {
    CUtensorMap m;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    SPT_CHECK((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, SPT_ERR_SHAPE, "TMA base must be 16-byte aligned");
    SPT_CHECK((ld * 2) % 16 == 0, SPT_ERR_SHAPE, "row pitch must be a multiple of 16 bytes");
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    SPT_CHECK(r == CUDA_SUCCESS, SPT_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

CUtensorMap make_tmap_f32_3d(const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_bytes,
                             uint64_t stride2_bytes, uint32_t b0, uint32_t b1, uint32_t b2) {
    CUtensorMap m;
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
    cuuint32_t box[3] = {b0, b1, b2};
    cuuint32_t es[3] = {1, 1, 1};
    SPT_CHECK((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, SPT_ERR_SHAPE, "TMA base must be 16-byte aligned");
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    SPT_CHECK(r == CUDA_SUCCESS, SPT_ERR_CUDA, "cuTensorMapEncodeTiled (f32 3d) failed: " + std::to_string((int)r));
    return m;
}

// fp32 [M, N] output with row pitch ldc as a 2-D TMA map, 32 x 32 boxes, 128-byte swizzle (epi_tma_block)
static CUtensorMap make_tmap_f32_c(void* C, int64_t M, int64_t N, int64_t ldc) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)ldc * 4};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t es[2] = {1, 1};
    SPT_CHECK((reinterpret_cast<uintptr_t>(C) & 15) == 0 && (ldc * 4) % 16 == 0, SPT_ERR_SHAPE,
              "fp32 TMA epilogue needs 16-byte aligned C and pitch");
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    SPT_CHECK(r == CUDA_SUCCESS, SPT_ERR_CUDA, "cuTensorMapEncodeTiled (fp32 C) failed: " + std::to_string((int)r));
    return m;
}

// Algorithmic HBM bytes of one GEMM: each operand read once, the output written once (read too for an fp32
// accumulate or a residual), plus the epilogue's side inputs / outputs.  The per-site "bytes" of the profiler and
// bench.py's roofline.algorithmic_bytes_per_launch, against which ncu's dram bytes (roofline.traffic) are read.
static double gemm_alg_bytes(int64_t M, int64_t N, int64_t K, int kind, const EpiParams& ep) {
    const double mn = (double)M * N;
    double b = 2.0 * M * K + 2.0 * N * K;
    switch (kind) {
        case EPI_BF16: b += 2 * mn * (ep.R ? 2 : 1); break;
        case EPI_F32: b += 4 * mn * (ep.accumulate ? 2 : 1); break;
        case EPI_SWIGLU: b += mn; break;                              // bf16 [M, N/2]
        case EPI_SWIGLU_BWD: b += mn + 2 * mn + mn; break;            // dA in, dGU + act out
        case EPI_F32_STATS: b += 4 * mn + mn / 256 * 8; break;
        case EPI_EXP_STATS: b += 2 * mn + mn / 256 * 8 + 12.0 * M; break;  // e, stats, labels + label logits
    }
    return b;
}

template <int BN, bool A_MN, bool B_MN, int KIND>
static void launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const EpiParams& ep_in,
                        cudaStream_t st) {
    EpiParams ep = ep_in;
    CUtensorMap tc = ta;  // unused unless the TMA fp32 epilogue runs
    if (KIND == EPI_F32 && ep.tstore == 2) tc = make_tmap_f32_c(ep.C, M, N, ep.ldc);
    auto kern = gemm_tc_kernel<BN, A_MN, B_MN, KIND>;
    constexpr int smem = GemmCfg<BN>::SMEM_BYTES;
    static bool attr_done = false;
    if (!attr_done) {
        SPT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_done = true;
    }
    const int ntiles = ((M + GEMM_BM - 1) / GEMM_BM) * ((N + BN - 1) / BN);
    const int grid = std::min(ntiles, num_sms());
    prof_run(P_GEMM, 2.0 * M * N * K, gemm_alg_bytes(M, N, K, KIND, ep), st, [&] {
        kern<<<grid, GEMM_THREADS, smem, st>>>(ta, tb, M, N, K, ep, tc);
        count_launch("gemm");
    });
    SPT_CUDA(cudaGetLastError());
}

template <int BN, bool A_MN, bool B_MN, int KIND>
static void launch_gemm2(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const EpiParams& ep,
                         cudaStream_t st) {
    CUtensorMap tc = ta;  // unused unless the TMA fp32 epilogue runs
    if (KIND == EPI_F32 && ep.tstore == 2) tc = make_tmap_f32_c(ep.C, M, N, ep.ldc);
    auto kern = gemm_tc2_kernel<BN, A_MN, B_MN, KIND>;
    constexpr int smem = Gemm2Cfg<BN>::SMEM_BYTES;
    static bool attr_done = false;
    if (!attr_done) {
        SPT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_done = true;
    }
    const int ntiles = ((M + 2 * GEMM_BM - 1) / (2 * GEMM_BM)) * ((N + BN - 1) / BN);
    const int clusters = std::min(ntiles, num_sms() / 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    prof_run(P_GEMM, 2.0 * M * N * K, gemm_alg_bytes(M, N, K, KIND, ep), st, [&] {
        SPT_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, M, N, K, ep, tc));
        count_launch("gemm2");
    });
}

static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return (e && e[0]) ? atoi(e) : dflt;
}
// Experiment / tuning switches: initialised from the environment, changeable at run time through
// spt_tuning_set (A/B comparisons inside one process).  gemm_1sm=1 disables CTA pairs, gemm_pair_mn selects
// which MN-major operand shapes run as pairs (0 = default none, 1 all, 2 by shape, 3 lm_head dX only: see pair_mn), gemm_bn=128|256 forces the N tile (0 = 256, 2 = 128 where it fills the last wave better),
// epi_tstore = fp32 epilogue mode: 0 per-thread stores, 1 smem-transposed coalesced stores, 2 (default) TMA
// store / reduce-add on the 1-SM kernel (the pair kernel and the stats epilogue use mode 1).
struct GemmTuning {
    int gemm_1sm = env_int("SPT_GEMM_1SM", 0);
    int gemm_pair_mn = env_int("SPT_GEMM_PAIR_MN", 0);
    int gemm_bn = env_int("SPT_GEMM_BN", 0);
    int epi_tstore = env_int("SPT_EPI_TSTORE", 2);
    int gemm_raster = env_int("SPT_GEMM_RASTER", 0);
    // tile-group size override (0: the defaults — row groups of 16 cluster rows for CTA pairs, whose earlier 8 read
    // 6.0 vs 3.6 GB of HBM on the logits GEMM, and column groups of gemm_colgroup for 1-SM tiles; see gemm())
    int gemm_group_m = env_int("SPT_GEMM_GROUP_M", 0);
    int gemm_colgroup = env_int("SPT_GEMM_COLGROUP", 8);
};
static GemmTuning& tuning() {
    static GemmTuning t;
    return t;
}
static bool use_pair_gemm() { return tuning().gemm_1sm != 1; }
// MN-major operand shapes as CTA pairs: 0 never, 1 always, 3 the vocab-long-K data gradient only (+0.8% per
// sustained L1 step, profiles/r2l_pair_mn_ab.json), 2 by shape — pairs where the isolated per-site
// A/B (profiles/README.md, gemm_sites) had them ahead: fp32-accumulate weight gradients with a long K
// (lm_head, QKV / O projections over the whole sequence) and bf16 data gradients except the short-M /
// long-K TiledMLP dX (whose 1-SM kernel keeps the TMA reduce-add epilogue and fills the SMs better).
static bool pair_mn(int64_t M, int64_t K, int kind) {
    const int v = tuning().gemm_pair_mn;
    if (v == 3) return kind == EPI_BF16 && K >= 65536;  // the lm_head dX (vocab-long K) only
    if (v != 2) return v == 1;
    if (kind == EPI_F32) return K >= 8192;
    if (kind == EPI_BF16) return !(M <= 4096 && K >= 16384);
    return false;
}
static int forced_bn() { return tuning().gemm_bn; }
static int epi_tstore() { return tuning().epi_tstore; }

template <int BN>
static void dispatch_pair(const GemmOperand& A, const GemmOperand& B, int64_t M, int64_t N, int64_t K, int kind,
                          const EpiParams& ep, cudaStream_t st) {
    CUtensorMap ta = A.mn_major ? make_tmap_bf16_2d(A.ptr, M, K, A.ld, 64, GEMM_BK)
                                : make_tmap_bf16_2d(A.ptr, K, M, A.ld, GEMM_BK, GEMM_BM);
    CUtensorMap tb = B.mn_major ? make_tmap_bf16_2d(B.ptr, N, K, B.ld, 64, GEMM_BK)
                                : make_tmap_bf16_2d(B.ptr, K, N, B.ld, GEMM_BK, BN / 2);
    const int m = (int)M, n = (int)N, k = (int)K;
    const int sel = (A.mn_major ? 2 : 0) + (B.mn_major ? 1 : 0);
    switch (sel * 8 + kind) {
        case 0 * 8 + EPI_BF16: launch_gemm2<BN, false, false, EPI_BF16>(ta, tb, m, n, k, ep, st); return;
        case 0 * 8 + EPI_F32: launch_gemm2<BN, false, false, EPI_F32>(ta, tb, m, n, k, ep, st); return;
        case 0 * 8 + EPI_SWIGLU: launch_gemm2<BN, false, false, EPI_SWIGLU>(ta, tb, m, n, k, ep, st); return;
        case 0 * 8 + EPI_SWIGLU_BWD: launch_gemm2<BN, false, false, EPI_SWIGLU_BWD>(ta, tb, m, n, k, ep, st); return;
        case 0 * 8 + EPI_F32_STATS: launch_gemm2<BN, false, false, EPI_F32_STATS>(ta, tb, m, n, k, ep, st); return;
        case 0 * 8 + EPI_EXP_STATS: launch_gemm2<BN, false, false, EPI_EXP_STATS>(ta, tb, m, n, k, ep, st); return;
        case 1 * 8 + EPI_BF16: launch_gemm2<BN, false, true, EPI_BF16>(ta, tb, m, n, k, ep, st); return;
        case 1 * 8 + EPI_F32: launch_gemm2<BN, false, true, EPI_F32>(ta, tb, m, n, k, ep, st); return;
        case 3 * 8 + EPI_BF16: launch_gemm2<BN, true, true, EPI_BF16>(ta, tb, m, n, k, ep, st); return;
        case 3 * 8 + EPI_F32: launch_gemm2<BN, true, true, EPI_F32>(ta, tb, m, n, k, ep, st); return;
        default: SPT_THROW(SPT_ERR_INTERNAL, "gemm: unsupported major/epilogue combination");
    }
}

template <int BN>
static void dispatch_1sm(const GemmOperand& A, const GemmOperand& B, int64_t M, int64_t N, int64_t K, int kind,
                         const EpiParams& ep, cudaStream_t st) {
    CUtensorMap ta = A.mn_major ? make_tmap_bf16_2d(A.ptr, M, K, A.ld, 64, GEMM_BK)
                                : make_tmap_bf16_2d(A.ptr, K, M, A.ld, GEMM_BK, GEMM_BM);
    CUtensorMap tb = B.mn_major ? make_tmap_bf16_2d(B.ptr, N, K, B.ld, 64, GEMM_BK)
                                : make_tmap_bf16_2d(B.ptr, K, N, B.ld, GEMM_BK, BN);
    const int m = (int)M, n = (int)N, k = (int)K;
    const int sel = (A.mn_major ? 2 : 0) + (B.mn_major ? 1 : 0);
    switch (sel * 8 + kind) {
        case 0 * 8 + EPI_BF16: launch_gemm<BN, false, false, EPI_BF16>(ta, tb, m, n, k, ep, st); break;
        case 0 * 8 + EPI_F32: launch_gemm<BN, false, false, EPI_F32>(ta, tb, m, n, k, ep, st); break;
        case 0 * 8 + EPI_SWIGLU: launch_gemm<BN, false, false, EPI_SWIGLU>(ta, tb, m, n, k, ep, st); break;
        case 0 * 8 + EPI_SWIGLU_BWD: launch_gemm<BN, false, false, EPI_SWIGLU_BWD>(ta, tb, m, n, k, ep, st); break;
        case 0 * 8 + EPI_F32_STATS: launch_gemm<BN, false, false, EPI_F32_STATS>(ta, tb, m, n, k, ep, st); break;
        case 0 * 8 + EPI_EXP_STATS: launch_gemm<BN, false, false, EPI_EXP_STATS>(ta, tb, m, n, k, ep, st); break;
        case 1 * 8 + EPI_BF16: launch_gemm<BN, false, true, EPI_BF16>(ta, tb, m, n, k, ep, st); break;
        case 1 * 8 + EPI_F32: launch_gemm<BN, false, true, EPI_F32>(ta, tb, m, n, k, ep, st); break;
        case 3 * 8 + EPI_BF16: launch_gemm<BN, true, true, EPI_BF16>(ta, tb, m, n, k, ep, st); break;
        case 3 * 8 + EPI_F32: launch_gemm<BN, true, true, EPI_F32>(ta, tb, m, n, k, ep, st); break;
        default: SPT_THROW(SPT_ERR_INTERNAL, "gemm: unsupported major/epilogue combination");
    }
}

void gemm(const GemmOperand& A, const GemmOperand& B, int64_t M, int64_t N, int64_t K, int kind, const EpiParams& ep_in,
          cudaStream_t st) {
    EpiParams ep = ep_in;
    ep.tstore = epi_tstore();
    if (Prof* pf = current_prof(); pf && pf->on) {
        static const char* kn[] = {"bf16", "f32", "swiglu", "swiglu_bwd", "f32_stats", "exp_stats"};
        pf->next_tag = std::string(A.mn_major ? "MN" : "K") + (B.mn_major ? "MN" : "K") + "_" + kn[kind] + "_" +
                       std::to_string(M) + "x" + std::to_string(N) + "x" + std::to_string(K);
    }
    SPT_CHECK(M > 0 && N > 0 && K > 0, SPT_ERR_SHAPE, "gemm: empty problem");
    SPT_CHECK(N % 64 == 0, SPT_ERR_SHAPE, "gemm: N must be a multiple of 64, got " + std::to_string(N));
    SPT_CHECK(M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31), SPT_ERR_SHAPE, "gemm: dims exceed int32");
    // The SwiGLU epilogues pair gate/up 32-column blocks inside a 64-column chunk and the logits stats are
    // per 256 columns, so those kinds keep BN = 256.
    const bool bn_free = kind == EPI_BF16 || kind == EPI_F32;
    // CTA pairs win for K-major x K-major (forward / logits) GEMMs.  MN-major operand shapes (backward) go
    // by pair_mn: pairs win short bursts (3 steps: -1.4..-3.3% per L1 step with the shape rule) but lose
    // sustained, power-capped runs (12 steps: +3.7%), so the default keeps them on the 1-SM kernel.
    const bool pair = M >= 2 * GEMM_BM && ((!A.mn_major && !B.mn_major) || pair_mn(M, K, kind)) && use_pair_gemm();
    // N tile: 256, or forced by gemm_bn (128 / 256), or (gemm_bn = 2) 128 where the tile count leaves the
    // last wave of the persistent grid mostly idle and 128-wide tiles fill it (the TiledMLP GEMMs with
    // 4096-row tiles and a long K: 512 tiles = 3.46 waves of 148 SMs at BN=256, 6.92 at BN=128).  That rule
    // measured 4% slower per sustained L1 step (168.7 -> 175.5 ms): the 128-wide MMAs read a third more
    // smem per flop, and under the power cap that costs more than the idle tail.
    int bn = 256;
    if (bn_free) {
        if (forced_bn() == 128 || forced_bn() == 256) bn = forced_bn();
        else if (forced_bn() == 2) {
            const int64_t units = pair ? num_sms() / 2 : num_sms(), rows = pair ? 2 * GEMM_BM : GEMM_BM;
            auto eff = [&](int64_t bnx) {
                const int64_t tiles = ((M + rows - 1) / rows) * ((N + bnx - 1) / bnx);
                const int64_t waves = (tiles + units - 1) / units;
                return (double)tiles / (double)(waves * units);
            };
            if (eff(128) >= eff(256) + 0.06) bn = 128;
        }
    }
    // Tile order by operand footprint (gemm_raster = 1, opt-in): when one operand fits in L2 with room to spare
    // (<= 80 MB of the 126 MB), sweep the tiles so that it is re-read from L2 and the other operand streams from
    // HBM exactly once, and tell the L2 so (evict_last on the resident operand, evict_first on the streamed one).
    // The lm_head weight gradient (B = the x tile, 67 MB; A = dlogits^T streamed) and the logits GEMM (A = the
    // x tile; B = W_lm streamed) are the cases that matter; with neither operand resident the grouped order stays.
    // gemm_raster = 0 (default): grouped order and no hints everywhere; 1: order only, 2: hints only, 3: both;
    // 16 + n: tile order n forced on every GEMM (A/B only).
    // Measured (profiles/r2b_gemm_raster.txt): 3 is 4.7% SLOWER per L1 step — the lm_head GEMMs read 40-50% MORE
    // from HBM with the resident-operand order than with the grouped one.
    if (tuning().gemm_raster >= 16) {
        ep.raster = tuning().gemm_raster - 16;  // A/B: force tile order n on every GEMM
    } else if (const int rm = tuning().gemm_raster; rm != 0) {  // bit 0: tile order, bit 1: L2 hints
        const double ba = 2.0 * M * K, bb = 2.0 * N * K, cap = 80.0 * (1 << 20);
        if (bb <= cap && bb <= ba) {
            if (rm & 1) ep.raster = 1;
            if (rm & 2) {
                ep.hint_a = 1;
                ep.hint_b = 2;
            }
        } else if (ba <= cap) {
            if (rm & 1) ep.raster = 2;
            if (rm & 2) {
                ep.hint_a = 2;
                ep.hint_b = 1;
            }
        }
    }
    ep.group_m = tuning().gemm_group_m;
    // 1-SM GEMMs (the MN-major data / weight gradients) sweep groups of gemm_colgroup column blocks over all row
    // blocks (raster 3): 8 x 256 columns at a time.  Measured on the lm_head backward GEMMs: dW 11.7 -> 9.1 GB and dX
    // 10.5 -> 8.5 GB of HBM reads, and -3.7% per sustained L1 step over all 1-SM GEMMs (row groups of 16 before;
    // column groups of 2 / 4 / 16: +1.4% / -2.4% / +0.8%; lm_head GEMMs only: -3.1%) — profiles/r2d_gemm_group.txt.
    // gemm_colgroup = 0: row groups (raster 0); G + 1000: column groups on the lm_head (vocab-sized M or K) only.
    if (const int cg = tuning().gemm_colgroup; cg > 0 && !pair && ep.raster == 0) {
        if (cg < 1000 || std::max(M, K) >= 65536) {
            ep.raster = 3;
            if (ep.group_m <= 0) ep.group_m = cg % 1000;
        }
    }
    if (pair) {
        if (ep.tstore == 2 && kind != EPI_F32) ep.tstore = 1;
        if (bn == 128) dispatch_pair<128>(A, B, M, N, K, kind, ep, st);
        else dispatch_pair<256>(A, B, M, N, K, kind, ep, st);
        return;
    }
    if (ep.tstore == 2 && kind != EPI_F32) ep.tstore = 1;
    if (bn == 128) dispatch_1sm<128>(A, B, M, N, K, kind, ep, st);
    else dispatch_1sm<256>(A, B, M, N, K, kind, ep, st);
}

}  // namespace spt

extern "C" spt_status spt_gemm_bf16(const void* A, int64_t lda, int32_t a_mn_major, const void* B, int64_t ldb,
                                    int32_t b_mn_major, void* C, int64_t ldc, int32_t c_f32, int32_t accumulate,
                                    const void* residual, int64_t ldr, int64_t M, int64_t N, int64_t K, float alpha,
                                    void* stream) {
    return spt::capi_guard([&] {
        spt::EpiParams ep;
        ep.C = C;
        ep.ldc = ldc;
        ep.R = reinterpret_cast<const spt::bf16*>(residual);
        ep.ldr = ldr;
        ep.accumulate = accumulate;
        ep.alpha = alpha;
        spt::gemm({A, lda, a_mn_major != 0}, {B, ldb, b_mn_major != 0}, M, N, K, c_f32 ? spt::EPI_F32 : spt::EPI_BF16,
                  ep, reinterpret_cast<cudaStream_t>(stream));
    });
}

namespace spt {
extern int g_attn_dq_tmem;   // attention_tc.cu
extern int g_attn_fwd_tmem;  // attention_tc.cu
extern int g_mlp_bwd_group;  // engine.cu
extern int g_rope_fused;     // engine.cu
extern int g_attn_dkdv_pair;  // attention_tc.cu
extern int g_attn_dkdv_kt;    // attention_tc.cu
extern int g_attn_kv_group;   // attention_tc.cu
extern int g_attn_fwd_bk128;  // attention_tc.cu
extern int g_attn_fwd_hybrid;  // attention_tc.cu
extern int g_replay_fault;     // engine.cu
extern int g_attn_bwd;         // attention_tc.cu
extern int g_attn_bwd4_dbg;    // attention_tc.cu
}

extern "C" spt_status spt_tuning_set(const char* name, int32_t value) {
    return spt::capi_guard([&] {
        const std::string n(name);
        auto& t = spt::tuning();
        if (n == "gemm_raster") {
            t.gemm_raster = value;
            return;
        }
        if (n == "gemm_group_m") {
            t.gemm_group_m = value;
            return;
        }
        if (n == "gemm_colgroup") {
            t.gemm_colgroup = value;
            return;
        }
        if (n == "attn_dq_tmem") {
            spt::g_attn_dq_tmem = value;
            return;
        }
        if (n == "attn_fwd_tmem") {
            spt::g_attn_fwd_tmem = value;
            return;
        }
        if (n == "attn_fwd_hybrid") {
            spt::g_attn_fwd_hybrid = value;
            return;
        }
        if (n == "attn_fwd_bk128") {
            spt::g_attn_fwd_bk128 = value;
            return;
        }
        if (n == "attn_kv_group") {
            spt::g_attn_kv_group = value;
            return;
        }
        if (n == "attn_dkdv_kt") {
            spt::g_attn_dkdv_kt = value;
            return;
        }
        if (n == "attn_dkdv_pair") {
            spt::g_attn_dkdv_pair = value;
            return;
        }
        if (n == "rope_fused") {
            spt::g_rope_fused = value;
            return;
        }
        if (n == "attn_bwd") {  // 0 two-pass, 1 fused (ordered L2 reductions), 2 fused on clusters of 4
            spt::g_attn_bwd = value;
            return;
        }
        if (n == "attn_bwd4_dbg") {  // timing experiments of the cluster-4 backward (results wrong when set)
            spt::g_attn_bwd4_dbg = value;
            return;
        }
        if (n == "replay_fault") {  // test-only: corrupt the next checkpoint replay (DeterminismError path)
            spt::g_replay_fault = value;
            return;
        }
        if (n == "mlp_bwd_group") {
            spt::g_mlp_bwd_group = value;
            return;
        }
        if (n == "gemm_1sm") t.gemm_1sm = value;
        else if (n == "gemm_pair_mn") t.gemm_pair_mn = value;
        else if (n == "gemm_bn") t.gemm_bn = value;
        else if (n == "epi_tstore") t.epi_tstore = value;
        else SPT_THROW(SPT_ERR_CONFIG, "unknown tuning switch '" + n + "'");
    });
}
