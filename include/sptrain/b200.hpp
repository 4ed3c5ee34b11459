// sptrain/b200.hpp — C++ host API of the B200 path, header-only over the C-ABI in sptrain_b200.h.
//
// This is the layer a maintainer of the reference (namespace `sptrain`, proj/include/sptrain/*.hpp) calls:
// the SPEC operations of the hot path with the reference's names, argument meaning and error behaviour.
//   * errors: every spt_status is rethrown as the reference's exception type (errors.hpp:12-72).  When the
//     reference headers are on the include path (-I <reference>/proj/include) its own errors.hpp is used, so
//     callers catch the same classes they already catch; otherwise identical classes are declared here.
//   * host logic: plan_head_shards, preshift_labels (:512), pad_to_multiple (:531),
//     block_causal_starts (:243), all-to-all schedule (:145, :307, :317).
//   * the training step: ProcessGroup (NCCL rank or in-process loopback ranks) and
//     UlyssesLayerStep — n decoder layers + lm_head fwd+bwd with ulysses_attention, tiled_mlp and
//     tiled_logits_loss, activation checkpointing / offload (:79, :462) and
//     gradient-accumulation windows (:548).
//   * single device ops (caller-owned device pointers, stream-ordered): matmul, rmsnorm, attention
//     fwd/bwd (the inner AttentionCallback), tiled_logits_loss, tiled_mlp.
// Link: -I<repo>/include -L<repo>/paper_2506_13996_b200 -lsptrain_b200 (C++17).
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "sptrain_b200.h"

#if defined(__has_include)
#if __has_include(<sptrain/errors.hpp>) && !defined(SPTRAIN_B200_OWN_ERRORS)
#include <sptrain/errors.hpp>
#define SPTRAIN_B200_REFERENCE_ERRORS 1
#endif
#endif

#ifndef SPTRAIN_B200_REFERENCE_ERRORS
#include <stdexcept>
namespace sptrain {  // same taxonomy and constructors as the reference's errors.hpp:12-72
class ValidationError : public std::runtime_error {
public:
    explicit ValidationError(const std::string& m) : std::runtime_error(m) {}
};
class ShapeError : public ValidationError {
public:
    explicit ShapeError(const std::string& m) : ValidationError(m) {}
};
class CollectiveError : public std::runtime_error {
public:
    explicit CollectiveError(const std::string& m) : std::runtime_error(m) {}
};
class ProtocolError : public CollectiveError {
public:
    explicit ProtocolError(const std::string& m) : CollectiveError(m) {}
};
class DeterminismError : public std::runtime_error {
public:
    explicit DeterminismError(const std::string& m) : std::runtime_error(m) {}
};
class SimulatedOomError : public std::runtime_error {
public:
    SimulatedOomError(const std::string& tier, std::size_t required, std::size_t available)
        : std::runtime_error("simulated " + tier + " OOM: required " + std::to_string(required) + " bytes, available " +
                             std::to_string(available)),
          required_bytes(required),
          available_bytes(available) {}
    std::size_t required_bytes;
    std::size_t available_bytes;
};
class ConfigError : public std::runtime_error {
public:
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
}  // namespace sptrain
#endif

namespace sptrain {
namespace b200 {

// spt_status -> the reference exception (errors.hpp); SPT_ERR_CUDA / INTERNAL -> std::runtime_error.
inline void check(spt_status s) {
    if (s == SPT_OK) return;
    const std::string m = spt_last_error();
    switch (s) {
        case SPT_ERR_SHAPE: throw ShapeError(m);
        case SPT_ERR_VALIDATION: throw ValidationError(m);
        case SPT_ERR_COLLECTIVE: throw CollectiveError(m);
        case SPT_ERR_PROTOCOL: throw ProtocolError(m);
        case SPT_ERR_DETERMINISM: throw DeterminismError(m);
        case SPT_ERR_CONFIG: throw ConfigError(m);
        case SPT_ERR_OOM: throw SimulatedOomError("device (" + m + ")", 0, 0);
        default: throw std::runtime_error(m);
    }
}

// ---------------------------------------------------------------- host logic (no GPU)
using HeadShardPlan = spt_head_shard_plan;

inline HeadShardPlan plan_head_shards(int q_heads, int kv_heads, int sp_degree) {
    HeadShardPlan p{};
    check(spt_plan_head_shards(q_heads, kv_heads, sp_degree, &p));
    return p;
}
// global q (kind 0) / kv (kind 1) heads rank `rank` owns after seq_to_head
inline std::vector<int> heads_of(const HeadShardPlan& p, int rank, int kind) {
    std::vector<int32_t> h(256);
    int32_t n = 0;
    check(spt_plan_heads_of(&p, rank, kind, h.data(), (int32_t)h.size(), &n));
    return std::vector<int>(h.begin(), h.begin() + n);
}
inline std::vector<int64_t> preshift_labels(const std::vector<int64_t>& labels) {
    std::vector<int64_t> out(labels.size());
    check(spt_preshift_labels(labels.data(), (int64_t)labels.size(), out.data()));
    return out;
}
struct Batch {
    std::vector<int64_t> input_ids, position_ids, shift_labels;
};
inline Batch pad_to_multiple(Batch b, int sp_degree) {
    int64_t n = 0;
    const int64_t s = (int64_t)b.input_ids.size();
    check(spt_pad_to_multiple(nullptr, nullptr, nullptr, s, sp_degree, 0, &n));
    b.input_ids.resize(n);
    b.position_ids.resize(n);
    b.shift_labels.resize(n);
    check(spt_pad_to_multiple(b.input_ids.data(), b.position_ids.data(), b.shift_labels.data(), s, sp_degree, n, &n));
    return b;
}
// contiguous equal shards in rank order
inline Batch shard_sequence(const Batch& b, int sp_degree, int rank) {
    const size_t n = b.input_ids.size() / (size_t)sp_degree, o = n * (size_t)rank;
    auto cut = [&](const std::vector<int64_t>& v) { return std::vector<int64_t>(v.begin() + o, v.begin() + o + n); };
    return {cut(b.input_ids), cut(b.position_ids), cut(b.shift_labels)};
}
inline std::vector<int64_t> block_causal_starts(const std::vector<int64_t>& position_ids) {
    std::vector<int64_t> out(position_ids.size());
    check(spt_block_causal_starts(position_ids.data(), (int64_t)position_ids.size(), out.data()));
    return out;
}

// ---------------------------------------------------------------- collectives
class ProcessGroup {
public:
    // one rank of an NCCL group (one process or thread per GPU); `id` from ProcessGroup::unique_id() on rank 0
    ProcessGroup(const std::vector<uint8_t>& id, int world_size, int rank, int device) {
        check(spt_comm_init_rank(id.data(), world_size, rank, device, &c_));
    }
    // in-process SPMD: `world_size` virtual ranks on one device (the reference's simulated ranks)
    static ProcessGroup loopback(int world_size, int device = 0) {
        spt_comm* c = nullptr;
        check(spt_comm_init_loopback(world_size, device, &c));
        return ProcessGroup(c);
    }
    static std::vector<uint8_t> unique_id() {
        std::vector<uint8_t> id(128);
        check(spt_comm_unique_id(id.data()));
        return id;
    }
    ProcessGroup(ProcessGroup&& o) noexcept : c_(std::exchange(o.c_, nullptr)) {}
    ProcessGroup(const ProcessGroup&) = delete;
    ProcessGroup& operator=(const ProcessGroup&) = delete;
    ~ProcessGroup() {
        if (c_) spt_comm_destroy(c_);
    }
    std::string stats_json() const {  // CommStats: calls and bytes per collective
        std::string b(1 << 14, '\0');
        check(spt_comm_stats_json(c_, b.data(), b.size()));
        return b.c_str();
    }
    spt_comm* handle() const { return c_; }

    // Collectives and reshards of SPEC.md:145-163 / :307-341 on caller-owned device buffers: one pointer per LOCAL
    // rank (loopback: every virtual rank's; peer mode: buffers from spt_comm_alloc).  `stream` is a cudaStream_t.
    void all_reduce_f32(const std::vector<void*>& bufs, int64_t n, void* stream = nullptr) {
        check(spt_all_reduce_f32(c_, bufs.data(), n, stream));
    }
    void all_to_all(const std::vector<const void*>& send, const std::vector<void*>& recv, size_t bytes_per_peer,
                    void* stream = nullptr) {
        check(spt_all_to_all(c_, send.data(), recv.data(), bytes_per_peer, stream));
    }
    void seq_to_head(const HeadShardPlan& plan, int kind, const std::vector<const void*>& x, int64_t s_loc,
                     int head_dim, const std::vector<void*>& out, void* scratch = nullptr, void* stream = nullptr) {
        check(spt_seq_to_head(c_, &plan, kind, x.data(), s_loc, head_dim, out.data(), scratch, stream));
    }
    void head_to_seq(const HeadShardPlan& plan, int kind, const std::vector<const void*>& x, int64_t s_loc,
                     int head_dim, const std::vector<void*>& out, void* scratch = nullptr, void* stream = nullptr) {
        check(spt_head_to_seq(c_, &plan, kind, x.data(), s_loc, head_dim, out.data(), scratch, stream));
    }
    // ulysses_attention: seq_to_head -> tcgen05 attention -> head_to_seq, and its backward
    void ulysses_attention_fwd(const HeadShardPlan& plan, const std::vector<const void*>& qkv, int64_t s_loc,
                               int head_dim, const int32_t* seg, float scale, const std::vector<void*>& qkv_head,
                               const std::vector<void*>& o_head, const std::vector<float*>& lse,
                               const std::vector<void*>& out, void* scratch = nullptr, void* stream = nullptr) {
        check(spt_ulysses_attention_fwd(c_, &plan, qkv.data(), s_loc, head_dim, seg, scale, qkv_head.data(),
                                        o_head.data(), lse.data(), out.data(), scratch, stream));
    }
    void ulysses_attention_bwd(const HeadShardPlan& plan, const std::vector<const void*>& qkv_head,
                               const std::vector<const void*>& o_head, const std::vector<const float*>& lse,
                               const std::vector<const void*>& dout, int64_t s_loc, int head_dim, const int32_t* seg,
                               float scale, const std::vector<void*>& do_head, const std::vector<void*>& dqkv_head,
                               const std::vector<void*>& ws, const std::vector<void*>& dqkv, void* scratch = nullptr,
                               void* stream = nullptr) {
        check(spt_ulysses_attention_bwd(c_, &plan, qkv_head.data(), o_head.data(), lse.data(), dout.data(), s_loc,
                                        head_dim, seg, scale, do_head.data(), dqkv_head.data(), ws.data(),
                                        dqkv.data(), scratch, stream));
    }

private:
    explicit ProcessGroup(spt_comm* c) : c_(c) {}
    spt_comm* c_ = nullptr;
};

// ---------------------------------------------------------------- the training step
struct ModelShape {  // ModelConfig with head_dim explicit
    int hidden, q_heads, kv_heads, head_dim, intermediate;
    int64_t vocab;
};
struct StepOptions {
    int n_layers = 1;            // > 1: per-layer activation checkpointing
    bool ckpt_offload = false;   // checkpoints in pinned host memory
    bool packed = false;         // block-causal attention from position_ids
    int mlp_tiles = 0;           // 0: 2 GiB intermediate budget; -1: ceil(s_loc / hidden)
    int64_t loss_tile = 0;       // tokens per logits tile, 0 -> auto
    float lr = 0.f;              // > 0: plain SGD update after the step
    float rms_eps = 1e-5f;
    float rope_theta = 0.f;      // > 0: rotary embedding on q/k (row f4; the reference model has none)
    bool embed = false;          // token embedding "emb" in front of the stack; step x = int64 input_ids
    bool verify_replay = false;  // fingerprint checkpoint replays vs the recorded forward (autograd.hpp:26-30)
};

class UlyssesLayerStep {
public:
    UlyssesLayerStep(const ModelShape& m, int64_t seq_len, const ProcessGroup& group, const StepOptions& o = {}) {
        spt_layer_config c{};
        c.hidden = m.hidden;
        c.q_heads = m.q_heads;
        c.kv_heads = m.kv_heads;
        c.head_dim = m.head_dim;
        c.intermediate = m.intermediate;
        c.vocab = m.vocab;
        c.seq_len = seq_len;
        c.mlp_tiles = o.mlp_tiles;
        c.loss_tile = o.loss_tile;
        c.rms_eps = o.rms_eps;
        c.packed = o.packed ? 1 : 0;
        c.lr = o.lr;
        c.n_layers = o.n_layers;
        c.ckpt_offload = o.ckpt_offload ? 1 : 0;
        c.rope_theta = o.rope_theta;
        c.embed = o.embed ? 1 : 0;
        c.verify_replay = o.verify_replay ? 1 : 0;
        check(spt_layer_create(&c, group.handle(), &l_));
    }
    UlyssesLayerStep(const UlyssesLayerStep&) = delete;
    UlyssesLayerStep& operator=(const UlyssesLayerStep&) = delete;
    ~UlyssesLayerStep() {
        if (l_) spt_layer_destroy(l_);
    }
    // name: g1 wqkv wo g2 wg wu wd (layer 0) | "layers.<i>.<name>" | g3 wlm; bf16 bits [out, in] row-major
    void set_param(const std::string& name, const void* bf16_bits, bool on_host = true) {
        check(spt_layer_set_param(l_, name.c_str(), bf16_bits, on_host ? 1 : 0));
    }
    // checked form: throws sptrain::ShapeError unless `numel` is what the engine copies for `name`
    void set_param(const std::string& name, const void* bf16_bits, int64_t numel, bool on_host) {
        if (numel != param_numel(name))
            throw ShapeError("set_param(" + name + "): " + std::to_string(numel) + " elements given, the engine expects " +
                             std::to_string(param_numel(name)));
        set_param(name, bf16_bits, on_host);
    }
    int64_t param_numel(const std::string& name) const {  // bf16 elements set_param copies for `name`
        int64_t n = 0;
        check(spt_layer_param_numel(l_, name.c_str(), &n));
        return n;
    }
    // one fwd+bwd step (SPEC.md:655 train step): returns (global mean loss, global valid count)
    std::pair<float, int64_t> step(const void* x_bf16, const int64_t* shift_labels, const int64_t* position_ids = nullptr,
                                   bool on_host = true, void* stream = nullptr) {
        float loss = 0.f;
        int64_t count = 0;
        check(spt_layer_step(l_, x_bf16, shift_labels, position_ids, on_host ? 1 : 0, &loss, &count, stream));
        return {loss, count};
    }
    // gradient-accumulation window
    void step_accumulate(const void* x_bf16, const int64_t* shift_labels, const int64_t* position_ids, bool first,
                         bool on_host = true, void* stream = nullptr) {
        check(spt_layer_step_accumulate(l_, x_bf16, shift_labels, position_ids, on_host ? 1 : 0, first ? 1 : 0, stream));
    }
    std::pair<float, int64_t> finish_accumulation(void* stream = nullptr) {
        float loss = 0.f;
        int64_t count = 0;
        check(spt_layer_finish_accumulation(l_, &loss, &count, stream));
        return {loss, count};
    }
    std::vector<float> grad(const std::string& name, size_t numel) const {  // SP-group all-reduced fp32 grad
        std::vector<float> g(numel);
        check(spt_layer_get_grad(l_, name.c_str(), g.data()));
        return g;
    }
    std::string memory_json() const {  // MemoryLedger::summary_json (ledger.hpp:85)
        std::string b(1 << 16, '\0');
        check(spt_layer_memory_json(l_, b.data(), b.size()));
        return b.c_str();
    }
    spt_layer* handle() const { return l_; }

private:
    spt_layer* l_ = nullptr;
};

// ---------------------------------------------------------------- single device ops (stream-ordered)
// matmul: C = alpha * A(m,k) B(n,k) [+ residual | + C]
inline void matmul(const void* A, int64_t lda, bool a_mn, const void* B, int64_t ldb, bool b_mn, void* C, int64_t ldc,
                   bool c_f32, bool accumulate, int64_t M, int64_t N, int64_t K, void* stream = nullptr) {
    check(spt_gemm_bf16(A, lda, a_mn, B, ldb, b_mn, C, ldc, c_f32, accumulate, nullptr, 0, M, N, K, 1.f, stream));
}
// inner AttentionCallback: causal / block-causal GQA over [s][hq + 2hkv][d]
inline void attention_fwd(const void* qkv, int64_t s, int hq, int hkv, int d, const int32_t* seg_start, float scale,
                          void* o, float* lse, void* stream = nullptr) {
    check(spt_attn_fwd(qkv, s, hq, hkv, d, seg_start, scale, o, lse, stream));
}
inline void attention_bwd(const void* qkv, const void* o, const float* lse, const void* dout, int64_t s, int hq, int hkv,
                          int d, const int32_t* seg_start, float scale, void* dqkv, void* workspace,
                          void* stream = nullptr) {
    check(spt_attn_bwd(qkv, o, lse, dout, s, hq, hkv, d, seg_start, scale, dqkv, workspace, stream));
}
// tiled_logits_loss, fused fwd+bwd
inline void tiled_logits_loss(const void* x, const void* w, const int64_t* labels, int64_t n, int64_t h, int64_t vocab,
                              int64_t tile_n, const float* grad_scale_dev, double* loss_sum_accum, void* dx, float* dw,
                              bool dw_accumulate, int32_t* err_flag, void* workspace, void* stream = nullptr) {
    check(spt_flce(x, w, labels, n, h, vocab, tile_n, grad_scale_dev, loss_sum_accum, dx, dw, dw_accumulate ? 1 : 0,
                   err_flag, workspace, stream));
}
// tiled_mlp
inline void tiled_mlp_fwd(const void* x, const void* wgu, const void* wd, const void* x_res, void* y, int64_t n,
                          int64_t h, int64_t inter, int64_t tile_n, void* workspace, void* stream = nullptr) {
    check(spt_mlp_fwd(x, wgu, wd, x_res, y, n, h, inter, tile_n, workspace, stream));
}
inline void tiled_mlp_bwd(const void* x, const void* wgu, const void* wd, const void* dy, void* dx, float* dwgu,
                          float* dwd, bool accumulate, int64_t n, int64_t h, int64_t inter, int64_t tile_n,
                          void* workspace, void* stream = nullptr) {
    check(spt_mlp_bwd(x, wgu, wd, dy, dx, dwgu, dwd, accumulate ? 1 : 0, n, h, inter, tile_n, workspace, stream));
}
// Token embedding: x[t] = table[input_ids[t]]; backward = per-id sums of dx rows in ascending
// token order (deterministic).  An id outside [0, vocab) sets *err_flag (device) to 3.
inline void embedding_fwd(const int64_t* input_ids, int64_t n, int64_t vocab, int64_t h, const void* table, void* x,
                          int32_t* err_flag, void* stream = nullptr) {
    check(spt_embed_fwd(input_ids, n, vocab, h, table, x, err_flag, stream));
}
inline void embedding_bwd(const int64_t* input_ids, int64_t n, int64_t vocab, int64_t h, const void* dx, float* dtable,
                          bool accumulate, int32_t* err_flag, void* workspace, void* stream = nullptr) {
    check(spt_embed_bwd(input_ids, n, vocab, h, dx, dtable, accumulate ? 1 : 0, err_flag, workspace, stream));
}
inline size_t embedding_bwd_workspace(int64_t n, int64_t vocab) { return spt_embed_bwd_workspace(n, vocab); }

}  // namespace b200
}  // namespace sptrain
