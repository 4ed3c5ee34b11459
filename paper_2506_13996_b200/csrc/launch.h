// Internal launch API shared by the kernel translation units and the C++ host engine.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace spt {

struct EpiParams;

struct GemmOperand {
    const void* ptr;
    int64_t ld;     // row pitch in elements of the stored matrix
    bool mn_major;  // false: element (row, k) at ptr[row*ld + k]; true: at ptr[k*ld + row]
};

void count_launch(const char* tag = nullptr);
int64_t launch_count();
void add_launches(int64_t n);  // kernels replayed inside a CUDA graph

// 3-D fp32 tensor map (no swizzle): dims {d0, d1, d2} innermost first, byte strides of dims 1 and 2.
CUtensorMap make_tmap_f32_3d(const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_bytes,
                             uint64_t stride2_bytes, uint32_t b0, uint32_t b1, uint32_t b2);
CUtensorMap make_tmap_bf16_2d(const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                              uint32_t box_outer);

// C[m,n] = sum_k A(m,k) B(n,k) with the fused epilogue `kind` (EpiKind in gemm.cuh).
void gemm(const GemmOperand& A, const GemmOperand& B, int64_t M, int64_t N, int64_t K, int kind, const EpiParams& ep,
          cudaStream_t st);

// kernels.cu
void rmsnorm_fwd(const void* x, const void* gamma, void* y, float* rstd, int64_t n, int64_t h, float eps,
                 cudaStream_t st);
size_t rmsnorm_bwd_workspace(int64_t n, int64_t h);
void rmsnorm_bwd(const void* x, const void* gamma, const float* rstd, const void* dy, const void* dres, void* dx,
                 float* dgamma_accum, void* ws, int64_t n, int64_t h, cudaStream_t st);
// Per-rank row bases of a reshard's far side: K1 writes destination rank j's rows at p[j] + (row_off + t) * row,
// K2 reads source rank j's rows at p[j] + (row_off + t) * row.  Contiguous [P][s_loc][row] buffers (NCCL
// send / receive staging) have p[j] = base + j * s_loc * row and row_off = 0; the fused peer collectives point
// p[j] straight at rank j's receive (K1) / attention output (K2) buffer, mapped over NVLink, with
// row_off = rank * s_loc (SPEC.md:351 payload layout: rank i's block of the global sequence).
constexpr int kMaxSP = 64;
struct RowTab {
    void* p[kMaxSP];
    int64_t row_off;
};
RowTab contiguous_rows(const void* base, int P, int64_t s_loc, int64_t row_bytes);
void reshard_pack(const void* src, int64_t s_loc, int heads_in, int head_dim, int P, int heads_out,
                  const int32_t* head_map, void* dst, cudaStream_t st);
void reshard_pack(const void* src, int64_t s_loc, int heads_in, int head_dim, int P, int heads_out,
                  const int32_t* head_map, const RowTab& dst, cudaStream_t st);
void reshard_unpack(const void* recv, int64_t s_loc, int heads_in, int head_dim, int P, int heads_out,
                    const int32_t* gather, int max_src, void* dst, cudaStream_t st);
void reshard_unpack(const RowTab& src, int64_t s_loc, int heads_in, int head_dim, int P, int heads_out,
                    const int32_t* gather, int max_src, void* dst, cudaStream_t st);
void label_stats(const int64_t* labels, int64_t n, int64_t vocab, int64_t* count_accum, int32_t* err, cudaStream_t st);
void segment_starts(const int64_t* pos, int64_t n, int32_t* starts, int32_t* err, cudaStream_t st);
// token embedding (embed.cu)
size_t embed_bwd_workspace(int64_t n, int64_t V);
void embed_fwd(const int64_t* ids, int64_t n, int64_t V, int64_t h, const void* E, void* x, int32_t* err,
               cudaStream_t st);
void embed_bwd(const int64_t* ids, int64_t n, int64_t V, int64_t h, const void* dx, float* dE, bool accumulate,
               int32_t* err, void* ws, cudaStream_t st);
// Row-wise CE over fp32 logits [rows, V]: loss_rows[r] (0 if ignored), dlogits bf16 = (softmax-onehot)*scale.
void ce_rows(const float* logits, const int64_t* labels, int64_t rows, int64_t V, const float* scale_dev,
             float* loss_rows, void* dlogits, int32_t* err, cudaStream_t st);
// Same, from per-(row, 256-column tile) (max, sumexp) stats written by the logits GEMM epilogue.
void ce_rows_exp(void* e_dlogits, const float* stats, int ntile, const int64_t* labels, const float* label_logit,
                 int64_t rows, int64_t V, const float* scale_dev, float* loss_rows, int32_t* err, cudaStream_t st);
void ce_rows_stats(const float* logits, const float* stats, int ntile, const int64_t* labels, int64_t rows, int64_t V,
                   const float* scale_dev, float* loss_rows, void* dlogits, int32_t* err, cudaStream_t st);
// Deterministic fixed-order sum of n fp32 values into an fp64 accumulator.
void sum_rows(const float* v, int64_t n, double* accum, cudaStream_t st);
// loss = loss_sum / count (device scalars) and scale = 1/count.
void finalize_scale(const int64_t* count, float* scale, cudaStream_t st);
void window_accumulate(const double* loss_sum, const int64_t* count, double* win_sum, int64_t* win_count, bool first,
                       cudaStream_t st);
void window_finalize(const double* win_sum, const int64_t* win_count, double* loss_sum, int64_t* count, float* loss,
                     cudaStream_t st);
void scale_by_inverse_count(float* g, int64_t n, const int64_t* count, cudaStream_t st);
// RoPE on the first n_rot heads of x [n][heads][d] (bf16, in place); inverse = backward rotation.
// K1 pack / K2 unpack with RoPE fused (false: shape not supported by the fused kernels, caller falls back)
// tab: optional (cos, sin) table from rope_table covering every position used (NULL: computed in-kernel)
// tab: (cos, sin) rows for positions [0, npos); a position outside that range sets *err = 4 (when err is
// given) and takes the in-kernel angles instead of reading past the table
bool reshard_pack_rope(const void* src, int64_t s_loc, int heads_in, int head_dim, int P, int heads_out,
                       const int32_t* head_map, const RowTab& dst, int n_rot, const int64_t* pos, int64_t pos_offset,
                       float theta, cudaStream_t st, const void* tab = nullptr, int64_t npos = 0,
                       int32_t* err = nullptr);
bool reshard_unpack_rope(const RowTab& src, int64_t s_loc, int heads_in, int head_dim, int heads_out,
                         const int32_t* gather, int max_src, void* dst, int n_rot, const int64_t* pos,
                         int64_t pos_offset, float theta, cudaStream_t st, const void* tab = nullptr,
                         int64_t npos = 0, int32_t* err = nullptr);
void rope_table(void* tab, int64_t npos, int d, float theta, cudaStream_t st);
extern int g_rope_fused;  // engine.cu: 1 (default) fuse RoPE into K1 / K2 when P > 1
void rope_apply(void* x, int64_t n, int heads, int n_rot, int d, const int64_t* pos, int64_t pos_offset, float theta,
                bool inverse, cudaStream_t st, const void* tab = nullptr, int64_t npos = 0, int32_t* err = nullptr);
void finalize_loss(const double* loss_sum, const int64_t* count, float* loss_out, cudaStream_t st);
// checkpoint replay verification (autograd.hpp:26-30): *out += order-independent fingerprint of n bf16 values;
// compare sets *err = tag when the fingerprints differ; flip_lowest_bit is the test-only fault injection
void fingerprint_bf16(const void* x, int64_t n, uint64_t* out, cudaStream_t st);
void fingerprint_compare(const uint64_t* want, const uint64_t* got, int32_t* err, int32_t tag, cudaStream_t st);
void flip_lowest_bit(void* x, cudaStream_t st);
// W(bf16) -= lr * G(fp32)
void sgd_update(void* w, const float* g, int64_t n, float lr, cudaStream_t st);
// Interleave/deinterleave gate/up in blocks of 32 rows: dst [2I, h] from wg [I,h], wu [I,h].
void interleave_gu(const void* wg, const void* wu, void* wgu, int64_t inter, int64_t h, cudaStream_t st);
void deinterleave_gu_f32(const float* gu, float* g, float* u, int64_t inter, int64_t h, cudaStream_t st);

// attention.cu
void attn_fwd(const void* qkv, int64_t s, int hq, int hkv, int d, const int32_t* seg_start, float scale, void* o,
              float* lse, cudaStream_t st);
size_t attn_bwd_workspace(int64_t s, int hq, int hkv, int d);
void attn_bwd(const void* qkv, const void* o, const float* lse, const void* dout, int64_t s, int hq, int hkv, int d,
              const int32_t* seg_start, float scale, void* dqkv, void* ws, cudaStream_t st);

}  // namespace spt
