// Collective-level Ulysses reshard ops behind the C-ABI: seq_to_head / head_to_seq with the
// all-to-all fused into the K1 pack / K2 unpack kernels (comm.h fused_seq_to_head / fused_head_to_seq).
// These are the single ops a host-side ulysses_attention composes around any inner
// attention; the layer engine (engine.cu) runs the same helpers inside its step.
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "comm.h"
#include "common.h"
#include "launch.h"
#include "plan.h"

using namespace spt;

namespace {

struct Maps {
    int32_t* map = nullptr;  // K1 head map [P][heads_out] or K2 gather [heads_out][max_src]
    int max_src = 1;
};

// Device copies of the plan's index maps, built once per (plan, op, device) and kept for the process.
Maps device_maps(const spt_head_shard_plan& pl, int op, int device) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, int, int>, Maps> cache;
    std::lock_guard<std::mutex> g(mu);
    const auto key = std::make_tuple(pl.q_heads, pl.kv_heads, pl.sp_degree, op, device);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    Maps m;
    std::vector<int32_t> v;
    switch (op) {
        case 0: v = qkv_pack_map(pl); break;
        case 1: v = q_pack_map(pl); break;
        case 2: v = o_gather_map(pl, &m.max_src); break;
        default: v = qkv_gather_map(pl, &m.max_src); break;
    }
    SPT_CUDA(cudaMalloc(&m.map, v.size() * 4));
    SPT_CUDA(cudaMemcpy(m.map, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
    cache[key] = m;
    return m;
}

struct Dims {
    int heads_full, heads_loc;  // [s_loc][heads_full][d] sequence side, [s][heads_loc][d] head side
};

Dims dims_of(const spt_head_shard_plan& pl, int kind) {
    if (kind == 0) return {pl.q_heads + 2 * pl.kv_heads, pl.q_heads_per_rank + 2 * pl.kv_heads_per_rank};
    return {pl.q_heads, pl.q_heads_per_rank};
}

// Rethrow a nested C-ABI call's failure with its own status and message.
void ck(spt_status st) {
    if (st != SPT_OK) SPT_THROW(st, spt_last_error());
}

void check_plan(spt_comm* comm, const spt_head_shard_plan* plan, int kind, int head_dim) {
    SPT_CHECK(comm && plan, SPT_ERR_CONFIG, "null comm / plan");
    SPT_CHECK(kind == 0 || kind == 1, SPT_ERR_CONFIG, "kind must be 0 (q|k|v) or 1 (q-shaped)");
    SPT_CHECK(plan->sp_degree == comm->nranks, SPT_ERR_SHAPE,
              "plan SP degree " + std::to_string(plan->sp_degree) + " != group size " + std::to_string(comm->nranks));
    SPT_CHECK(head_dim > 0 && head_dim % 8 == 0, SPT_ERR_SHAPE, "head_dim must be a positive multiple of 8");
}

}  // namespace

extern "C" {

size_t spt_reshard_scratch_bytes(const spt_head_shard_plan* plan, int32_t kind, int64_t s_loc, int32_t head_dim) {
    if (!plan) return 0;
    const Dims dm = dims_of(*plan, kind);
    return (size_t)plan->sp_degree * s_loc * dm.heads_loc * head_dim * 2;
}

spt_status spt_seq_to_head(spt_comm* comm, const spt_head_shard_plan* plan, int32_t kind, const void* const* x,
                           int64_t s_loc, int32_t head_dim, void* const* out, void* scratch, void* stream) {
    return capi_guard([&] {
        check_plan(comm, plan, kind, head_dim);
        SPT_CHECK(comm->mode != spt_comm::kNccl || scratch || comm->nranks == 1, SPT_ERR_CONFIG,
                  "NCCL transport needs the staging scratch (spt_reshard_scratch_bytes)");
        cudaStream_t st = (cudaStream_t)stream;
        const Dims dm = dims_of(*plan, kind);
        const Maps m = device_maps(*plan, kind, comm->device);
        const int P = comm->nranks;
        std::vector<void*> outs(out, out + comm->local_ranks());
        if (P == 1) {  // identity (SPEC.md:307 with one rank): the head side is the sequence side
            SPT_CUDA(cudaMemcpyAsync(outs[0], x[0], (size_t)s_loc * dm.heads_full * head_dim * 2,
                                     cudaMemcpyDeviceToDevice, st));
            return;
        }
        fused_seq_to_head(comm, kind == 0 ? "all_to_all_qkv" : "all_to_all_do", outs, scratch, s_loc,
                          (int64_t)dm.heads_loc * head_dim * 2, st, [&](int r, const RowTab& t) {
                              reshard_pack(x[r], s_loc, dm.heads_full, head_dim, P, dm.heads_loc, m.map, t, st);
                          });
    });
}

spt_status spt_head_to_seq(spt_comm* comm, const spt_head_shard_plan* plan, int32_t kind, const void* const* x,
                           int64_t s_loc, int32_t head_dim, void* const* out, void* scratch, void* stream) {
    return capi_guard([&] {
        check_plan(comm, plan, kind, head_dim);
        SPT_CHECK(comm->mode != spt_comm::kNccl || scratch || comm->nranks == 1, SPT_ERR_CONFIG,
                  "NCCL transport needs the staging scratch (spt_reshard_scratch_bytes)");
        cudaStream_t st = (cudaStream_t)stream;
        // kind 0: O (q heads, no replicas); kind 1: d(q|k|v) (kv replicas summed)
        const Dims dm = kind == 0 ? dims_of(*plan, 1) : dims_of(*plan, 0);
        const Maps m = device_maps(*plan, kind == 0 ? 2 : 3, comm->device);
        const int P = comm->nranks;
        std::vector<void*> srcs;
        for (int r = 0; r < comm->local_ranks(); ++r) srcs.push_back(const_cast<void*>(x[r]));
        if (P == 1) {
            SPT_CUDA(cudaMemcpyAsync(out[0], x[0], (size_t)s_loc * dm.heads_full * head_dim * 2,
                                     cudaMemcpyDeviceToDevice, st));
            return;
        }
        fused_head_to_seq(comm, kind == 0 ? "all_to_all_o" : "all_to_all_dqkv", srcs, scratch, s_loc,
                          (int64_t)dm.heads_loc * head_dim * 2, st, [&](int r, const RowTab& t) {
                              reshard_unpack(t, s_loc, dm.heads_loc, head_dim, P, dm.heads_full, m.map, m.max_src,
                                             out[r], st);
                          });
    });
}

// SPEC.md:333-341 ulysses_attention over a group: seq_to_head (K1 + all-to-all) -> the tcgen05 inner attention on
// each rank's heads over the whole sequence -> head_to_seq (K2 + all-to-all), and the mirrored backward.  The same
// sequence the layer engine runs inside its step, as one op for a host that composes its own layer.
spt_status spt_ulysses_attention_fwd(spt_comm* comm, const spt_head_shard_plan* plan, const void* const* qkv,
                                     int64_t s_loc, int32_t head_dim, const int32_t* seg, float scale,
                                     void* const* qkv_head, void* const* o_head, float* const* lse, void* const* out,
                                     void* scratch, void* stream) {
    return capi_guard([&] {
        check_plan(comm, plan, 0, head_dim);
        SPT_CHECK(qkv && qkv_head && o_head && lse && out, SPT_ERR_CONFIG, "ulysses_attention_fwd: null buffer array");
        const int64_t s = s_loc * comm->nranks;
        ck(spt_seq_to_head(comm, plan, 0, qkv, s_loc, head_dim, qkv_head, scratch, stream));
        for (int r = 0; r < comm->local_ranks(); ++r)
            ck(spt_attn_fwd(qkv_head[r], s, plan->q_heads_per_rank, plan->kv_heads_per_rank, head_dim, seg, scale,
                            o_head[r], lse[r], stream));
        ck(spt_head_to_seq(comm, plan, 0, o_head, s_loc, head_dim, out, scratch, stream));
    });
}

spt_status spt_ulysses_attention_bwd(spt_comm* comm, const spt_head_shard_plan* plan, const void* const* qkv_head,
                                     const void* const* o_head, const float* const* lse, const void* const* dout,
                                     int64_t s_loc, int32_t head_dim, const int32_t* seg, float scale,
                                     void* const* do_head, void* const* dqkv_head, void* const* ws,
                                     void* const* dqkv, void* scratch, void* stream) {
    return capi_guard([&] {
        check_plan(comm, plan, 1, head_dim);
        SPT_CHECK(qkv_head && o_head && lse && dout && do_head && dqkv_head && ws && dqkv, SPT_ERR_CONFIG,
                  "ulysses_attention_bwd: null buffer array");
        const int64_t s = s_loc * comm->nranks;
        ck(spt_seq_to_head(comm, plan, 1, dout, s_loc, head_dim, do_head, scratch, stream));
        for (int r = 0; r < comm->local_ranks(); ++r)
            ck(spt_attn_bwd(qkv_head[r], o_head[r], lse[r], do_head[r], s, plan->q_heads_per_rank,
                            plan->kv_heads_per_rank, head_dim, seg, scale, dqkv_head[r], ws[r], stream));
        ck(spt_head_to_seq(comm, plan, 1, dqkv_head, s_loc, head_dim, dqkv, scratch, stream));
    });
}

}  // extern "C"
