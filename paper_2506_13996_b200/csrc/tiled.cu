// Sequence-tiled compute on the tcgen05 GEMM family:
//   * fused tiled logits + cross-entropy fwd+bwd (K5; tiled_logits_loss)
//   * TiledMLP fwd / bwd with per-tile recompute (K6/K7; tiled_mlp)
// plus the C-ABI wrappers of the HBM-bound kernels.
#include "common.h"
#include "gemm.cuh"
#include "launch.h"

namespace spt {

static inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// ---------------------------------------------------------------- K5: fused logits + CE
static int64_t flce_ntile(int64_t V) { return (V + 255) / 256; }

// SPT_FLCE_EXP (read once at load): 1 (default) the logits GEMM's epilogue writes e = exp(x - m_tile) in bf16
// straight into the dlogits buffer and the CE pass rewrites it in place (no fp32 [tile, V] buffer); 0 the
// earlier form (fp32 logits from the epilogue, CE pass reads them and writes bf16 dlogits), kept for A/B.
int g_flce_exp = [] {
    const char* e = getenv("SPT_FLCE_EXP");
    return (e && e[0]) ? atoi(e) : 1;
}();

// Default loss tile for n_loc local tokens (engine and memest): the fewest tiles whose [tile, V] workspace
// stays within 4 GiB (SPEC.md:423 budget), split evenly, multiples of 128.  The budget is counted at 4 bytes
// per logit whichever form runs, so both forms use the same tiles (8192 tokens at V=128256: the 4096 x 4096
// dx GEMM then has 2x the cluster tiles of 4096 and dW is re-read half as often).
int64_t flce_default_tile(int64_t n_loc, int64_t V) {
    const int64_t tmax = std::max<int64_t>(128, (int64_t)((4ll << 30) / (V * 4)) / 128 * 128);
    const int64_t ntl = std::max<int64_t>(1, (n_loc + tmax - 1) / tmax);
    const int64_t t = ((n_loc + ntl - 1) / ntl + 127) / 128 * 128;
    return std::max<int64_t>(1, std::min<int64_t>(std::min(t, tmax), n_loc));
}

size_t flce_workspace(int64_t tile_n, int64_t V) {
    return (g_flce_exp ? 0 : align256((size_t)tile_n * V * 4)) + align256((size_t)tile_n * V * 2) +
           2 * align256((size_t)tile_n * 4) + align256((size_t)tile_n * flce_ntile(V) * 8);
}

// Per tile t (ascending): logits_t = x_t W^T (only per-256-column exp / stats of it reach memory, in the bf16
// [tile_n, V] buffer that becomes dlogits — SPEC.md:408),
// CE rows -> (loss_sum, dlogits scaled by 1/global_count), dx_t = dlogits W, dW += dlogits^T x_t.
// Gradient-in-forward: loss is terminal, so dlogits is formed while the tile's logits are live and no
// backward recompute is needed (results equal the spec's recompute up to fp order).
void flce(const void* x, const void* w, const int64_t* labels, int64_t n, int64_t h, int64_t V, int64_t tile_n,
          const float* scale_dev, double* loss_sum_accum, void* dx, float* dw, bool dw_accumulate, int32_t* err,
          void* ws, cudaStream_t st) {
    SPT_CHECK(tile_n > 0 && n >= 0, SPT_ERR_SHAPE, "flce: tile_n must be > 0");
    uint8_t* p = (uint8_t*)ws;
    float* logits = (float*)p;
    if (!g_flce_exp) p += align256((size_t)tile_n * V * 4);
    bf16* dlog = (bf16*)p;
    p += align256((size_t)tile_n * V * 2);
    float* loss_rows = (float*)p;
    p += align256((size_t)tile_n * 4);
    float* label_logit = (float*)p;
    p += align256((size_t)tile_n * 4);
    float* stats = (float*)p;
    const int64_t ntile = flce_ntile(V);
    const bf16* xb = (const bf16*)x;
    for (int64_t a = 0, t = 0; a < n; a += tile_n, ++t) {
        const int64_t rows = std::min(tile_n, n - a);
        // logits + per-(row, 256-col tile) softmax stats from the GEMM epilogue: the CE pass reads the
        // fp32 logits once (SPEC.md:69 cross_entropy on the tile, never an [s, V] tensor — :408)
        EpiParams e1;
        e1.ldc = V;
        e1.stats = stats;
        e1.ld_stats = ntile;
        if (g_flce_exp) {
            e1.C = dlog;
            e1.labels = labels + a;
            e1.label_logit = label_logit;
            gemm({xb + a * h, h, false}, {w, h, false}, rows, V, h, EPI_EXP_STATS, e1, st);
            ce_rows_exp(dlog, stats, (int)ntile, labels + a, label_logit, rows, V, scale_dev, loss_rows, err, st);
        } else {
            e1.C = logits;
            gemm({xb + a * h, h, false}, {w, h, false}, rows, V, h, EPI_F32_STATS, e1, st);
            ce_rows_stats(logits, stats, (int)ntile, labels + a, rows, V, scale_dev, loss_rows, dlog, err, st);
        }
        sum_rows(loss_rows, rows, loss_sum_accum, st);
        EpiParams e2;
        e2.C = (bf16*)dx + a * h;
        e2.ldc = h;
        gemm({dlog, V, false}, {w, h, true}, rows, h, V, EPI_BF16, e2, st);
        EpiParams e3;
        e3.C = dw;
        e3.ldc = h;
        e3.accumulate = (t > 0 || dw_accumulate) ? 1 : 0;
        gemm({dlog, V, true}, {xb + a * h, h, true}, V, h, rows, EPI_F32, e3, st);
    }
}

// ---------------------------------------------------------------- K6/K7: TiledMLP
size_t mlp_workspace(int64_t tile_n, int64_t I) {
    return align256((size_t)tile_n * I * 2) * 2 + align256((size_t)tile_n * I * 4);
}

void mlp_fwd(const void* x, const void* wgu, const void* wd, const void* x_res, void* y, int64_t n, int64_t h,
             int64_t I, int64_t tile_n, void* ws, cudaStream_t st) {
    bf16* act = (bf16*)ws;
    const bf16* xb = (const bf16*)x;
    for (int64_t a = 0; a < n; a += tile_n) {
        const int64_t rows = std::min(tile_n, n - a);
        EpiParams e1;
        e1.C = act;
        e1.ldc = I;
        gemm({xb + a * h, h, false}, {wgu, h, false}, rows, 2 * I, h, EPI_SWIGLU, e1, st);
        EpiParams e2;
        e2.C = (bf16*)y + a * h;
        e2.ldc = h;
        e2.R = x_res ? (const bf16*)x_res + a * h : nullptr;
        e2.ldr = h;
        gemm({act, I, false}, {wd, I, false}, rows, h, I, EPI_BF16, e2, st);
    }
}

void mlp_bwd(const void* x, const void* wgu, const void* wd, const void* dy, void* dx, float* dwgu, float* dwd,
             bool accumulate, int64_t n, int64_t h, int64_t I, int64_t tile_n, void* ws, cudaStream_t st) {
    uint8_t* p = (uint8_t*)ws;
    bf16* da = (bf16*)p;
    p += align256((size_t)tile_n * I * 2);
    bf16* act = (bf16*)p;
    p += align256((size_t)tile_n * I * 2);
    bf16* dgu = (bf16*)p;
    const bf16* xb = (const bf16*)x;
    const bf16* dyb = (const bf16*)dy;
    for (int64_t a = 0, t = 0; a < n; a += tile_n, ++t) {
        const int64_t rows = std::min(tile_n, n - a);
        const int acc = (t > 0 || accumulate) ? 1 : 0;
        // dA = dY Wd
        EpiParams e1;
        e1.C = da;
        e1.ldc = I;
        gemm({dyb + a * h, h, false}, {wd, I, true}, rows, I, h, EPI_BF16, e1, st);
        // recompute [g|u] = x Wgu^T; epilogue: act = silu(g)u, dGU from dA
        EpiParams e2;
        e2.C = dgu;
        e2.ldc = 2 * I;
        e2.aux = da;
        e2.ldaux = I;
        e2.C2 = act;
        e2.ldc2 = I;
        gemm({xb + a * h, h, false}, {wgu, h, false}, rows, 2 * I, h, EPI_SWIGLU_BWD, e2, st);
        // dWd += dY^T act
        EpiParams e3;
        e3.C = dwd;
        e3.ldc = I;
        e3.accumulate = acc;
        gemm({dyb + a * h, h, true}, {act, I, true}, h, I, rows, EPI_F32, e3, st);
        // dX = dGU Wgu
        EpiParams e4;
        e4.C = (bf16*)dx + a * h;
        e4.ldc = h;
        gemm({dgu, 2 * I, false}, {wgu, h, true}, rows, h, 2 * I, EPI_BF16, e4, st);
        // dWgu += dGU^T x
        EpiParams e5;
        e5.C = dwgu;
        e5.ldc = h;
        e5.accumulate = acc;
        gemm({dgu, 2 * I, true}, {xb + a * h, h, true}, 2 * I, h, rows, EPI_F32, e5, st);
    }
}

}  // namespace spt

using namespace spt;
#define ST reinterpret_cast<cudaStream_t>(stream)

extern "C" {

spt_status spt_rmsnorm_fwd(const void* x, const void* gamma, void* y, float* rstd, int64_t n, int64_t h, float eps,
                           void* stream) {
    return capi_guard([&] { rmsnorm_fwd(x, gamma, y, rstd, n, h, eps, ST); });
}
size_t spt_rmsnorm_bwd_workspace(int64_t n, int64_t h) {
    size_t r = 0;
    capi_guard([&] { r = rmsnorm_bwd_workspace(n, h); });
    return r;
}
spt_status spt_rmsnorm_bwd(const void* x, const void* gamma, const float* rstd, const void* dy, const void* dres,
                           void* dx, float* dgamma_accum, void* workspace, int64_t n, int64_t h, void* stream) {
    return capi_guard([&] { rmsnorm_bwd(x, gamma, rstd, dy, dres, dx, dgamma_accum, workspace, n, h, ST); });
}
spt_status spt_reshard_pack(const void* src, int64_t s_loc, int32_t heads_in, int32_t head_dim, int32_t P,
                            int32_t heads_out, const int32_t* head_map, void* dst, void* stream) {
    return capi_guard([&] { reshard_pack(src, s_loc, heads_in, head_dim, P, heads_out, head_map, dst, ST); });
}
spt_status spt_reshard_pack_rope(const void* src, int64_t s_loc, int32_t heads_in, int32_t head_dim, int32_t P,
                                 int32_t heads_out, const int32_t* head_map, void* dst, int32_t n_rot,
                                 const int64_t* position_ids, int64_t pos_offset, float theta,
                                 const void* cos_sin_table, void* stream) {
    return capi_guard([&] {
        SPT_CHECK(theta > 0.f, SPT_ERR_CONFIG, "rope: theta must be > 0");
        // the caller's table covers every position it passes (spt_rope_table documents the extent)
        SPT_CHECK(reshard_pack_rope(src, s_loc, heads_in, head_dim, P, heads_out, head_map,
                                    contiguous_rows(dst, P, s_loc, (int64_t)heads_out * head_dim * 2), n_rot,
                                    position_ids, pos_offset, theta, ST, cos_sin_table, INT64_MAX),
                  SPT_ERR_SHAPE, "reshard_pack_rope: head_dim must be 32, 64 or 128 and the head map fit in smem");
    });
}
spt_status spt_rope_table(void* cos_sin_table, int64_t npos, int32_t head_dim, float theta, void* stream) {
    return capi_guard([&] { rope_table(cos_sin_table, npos, head_dim, theta, ST); });
}
spt_status spt_reshard_unpack(const void* recv, int64_t s_loc, int32_t heads_in, int32_t head_dim, int32_t P,
                              int32_t heads_out, const int32_t* gather, int32_t max_src, void* dst, void* stream) {
    return capi_guard([&] { reshard_unpack(recv, s_loc, heads_in, head_dim, P, heads_out, gather, max_src, dst, ST); });
}
spt_status spt_label_stats(const int64_t* labels, int64_t n, int64_t vocab, int64_t* count_accum, int32_t* err_flag,
                           void* stream) {
    return capi_guard([&] { label_stats(labels, n, vocab, count_accum, err_flag, ST); });
}
spt_status spt_segment_starts(const int64_t* position_ids, int64_t n, int32_t* starts, int32_t* err_flag,
                              void* stream) {
    return capi_guard([&] { segment_starts(position_ids, n, starts, err_flag, ST); });
}
size_t spt_flce_workspace(int64_t tile_n, int64_t vocab) { return flce_workspace(tile_n, vocab); }
spt_status spt_flce(const void* x, const void* w, const int64_t* labels, int64_t n, int64_t h, int64_t vocab,
                    int64_t tile_n, const float* grad_scale_dev, double* loss_sum_accum, void* dx, float* dw,
                    int32_t dw_accumulate, int32_t* err_flag, void* workspace, void* stream) {
    return capi_guard([&] {
        flce(x, w, labels, n, h, vocab, tile_n, grad_scale_dev, loss_sum_accum, dx, dw, dw_accumulate != 0, err_flag,
             workspace, ST);
    });
}
size_t spt_mlp_workspace(int64_t tile_n, int64_t inter) { return mlp_workspace(tile_n, inter); }
spt_status spt_mlp_fwd(const void* x, const void* wgu, const void* wd, const void* x_res, void* y, int64_t n, int64_t h,
                       int64_t inter, int64_t tile_n, void* workspace, void* stream) {
    return capi_guard([&] { mlp_fwd(x, wgu, wd, x_res, y, n, h, inter, tile_n, workspace, ST); });
}
spt_status spt_mlp_bwd(const void* x, const void* wgu, const void* wd, const void* dy, void* dx, float* dwgu,
                       float* dwd, int32_t accumulate, int64_t n, int64_t h, int64_t inter, int64_t tile_n,
                       void* workspace, void* stream) {
    return capi_guard(
        [&] { mlp_bwd(x, wgu, wd, dy, dx, dwgu, dwd, accumulate != 0, n, h, inter, tile_n, workspace, ST); });
}
spt_status spt_rope(void* x, int64_t n, int32_t heads, int32_t n_rot, int32_t head_dim, const int64_t* position_ids,
                    int64_t pos_offset, float theta, int32_t inverse, void* stream) {
    return capi_guard([&] {
        SPT_CHECK(n_rot >= 0 && n_rot <= heads, SPT_ERR_SHAPE, "rope: n_rot must be in [0, heads]");
        rope_apply(x, n, heads, n_rot, head_dim, position_ids, pos_offset, theta, inverse != 0,
                   (cudaStream_t)stream);
    });
}

size_t spt_attn_bwd_workspace(int64_t s, int32_t hq, int32_t hkv, int32_t head_dim) {
    size_t r = 0;
    capi_guard([&] { r = attn_bwd_workspace(s, hq, hkv, head_dim); });
    return r;
}
spt_status spt_attn_fwd(const void* qkv, int64_t s, int32_t hq, int32_t hkv, int32_t head_dim,
                        const int32_t* seg_start, float scale, void* o, float* lse, void* stream) {
    return capi_guard([&] { attn_fwd(qkv, s, hq, hkv, head_dim, seg_start, scale, o, lse, ST); });
}
spt_status spt_attn_bwd(const void* qkv, const void* o, const float* lse, const void* dout, int64_t s, int32_t hq,
                        int32_t hkv, int32_t head_dim, const int32_t* seg_start, float scale, void* dqkv,
                        void* workspace, void* stream) {
    return capi_guard(
        [&] { attn_bwd(qkv, o, lse, dout, s, hq, hkv, head_dim, seg_start, scale, dqkv, workspace, ST); });
}

}  // extern "C"
