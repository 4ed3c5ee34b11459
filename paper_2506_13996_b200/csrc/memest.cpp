// memest: the paper's closed-form memory expressions and the max-seqlen solver, plus the
// byte counts of THIS engine's own ledger tags (the formulas are exact for it — SPEC.md:622 ledger
// cross-validation).  Host-only, pure functions.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "common.h"

namespace spt {
size_t flce_workspace(int64_t tile_n, int64_t V);  // tiled.cu
int64_t flce_default_tile(int64_t n_loc, int64_t V);
size_t mlp_workspace(int64_t tile_n, int64_t I);  // tiled.cu

// The engine's default TiledMLP tile (engine.cu: fewest tiles whose tile * I * 8 bytes of intermediates fit 2 GiB,
// split evenly) and the workspace it sizes: fixed once the local sequence exceeds one tile.
static double mlp_ws_bytes(const spt_memest_engine& e, double nl) {
    if (nl < 1) return 0.0;
    const int64_t n = (int64_t)nl, I = e.intermediate;
    const int64_t tmax = std::max<int64_t>(128, (int64_t)((2ll << 30) / (I * 8)) / 128 * 128);
    const int64_t mt = std::max<int64_t>(1, (n + tmax - 1) / tmax);
    return (double)mlp_workspace((n + mt - 1) / mt, I);
}
namespace {
constexpr double GiB = 1024.0 * 1024.0 * 1024.0;

// estimate_fixed (PAPER §2.1): weights 2 B/param, Adam states 8, fp32 master 4, grads 4
spt_memest_fixed fixed(double params, int world, int zero3, int offload_optimizer) {
    SPT_CHECK(params > 0, SPT_ERR_VALIDATION, "param_count must be > 0");
    spt_memest_fixed f{};
    f.weights_bytes = 2.0 * params;
    f.optimizer_bytes = 8.0 * params;
    f.master_weights_bytes = 4.0 * params;
    f.grads_bytes = 4.0 * params;
    f.total_bytes = f.weights_bytes + f.optimizer_bytes + f.master_weights_bytes + f.grads_bytes;
    const double share = zero3 ? 1.0 / std::max(1, world) : 1.0;
    const double dev = (f.weights_bytes + f.grads_bytes) * share +
                       (offload_optimizer ? 0.0 : (f.optimizer_bytes + f.master_weights_bytes) * share);
    f.device_bytes_per_gpu = dev;
    f.host_bytes_per_gpu = offload_optimizer ? (f.optimizer_bytes + f.master_weights_bytes) * share : 0.0;
    return f;
}

// estimate_activation_ckpt (PAPER §3.3): s/sp tokens * h * layers * bytes per GPU; the host
// copy of the offloaded checkpoints is per node (gpus_per_node GPUs)
void act_ckpt(double s, double h, double layers, double bytes, int sp, int gpus_per_node, double* dev, double* host) {
    const double per_gpu = s / std::max(1, sp) * h * layers * bytes;
    *dev = per_gpu;
    *host = per_gpu * gpus_per_node;
}
}  // namespace
}  // namespace spt

using namespace spt;

extern "C" {

spt_status spt_memest_fixed_bytes(double param_count, int32_t world_size, int32_t zero3, int32_t offload_optimizer,
                                  spt_memest_fixed* out) {
    return capi_guard([&] { *out = fixed(param_count, world_size, zero3, offload_optimizer); });
}

// estimate_logits: fp32 [s, V]; the loss keeps 2x of it (PAPER §3.1)
double spt_memest_logits_bytes(double seqlen, double vocab, double bytes) { return seqlen * vocab * bytes; }

spt_status spt_memest_activation_ckpt_bytes(double seqlen, double hidden, double layers, double bytes, int32_t sp,
                                            int32_t gpus_per_node, double* device_bytes, double* host_bytes_per_node) {
    return capi_guard([&] {
        SPT_CHECK(seqlen >= 0 && hidden > 0 && layers > 0 && bytes > 0, SPT_ERR_VALIDATION, "bad memest arguments");
        act_ckpt(seqlen, hidden, layers, bytes, sp, gpus_per_node, device_bytes, host_bytes_per_node);
    });
}

// estimate_4d_mask / estimate_position_ids (PAPER §3.4)
double spt_memest_4d_mask_bytes(double seqlen, double bytes) { return seqlen * seqlen * bytes; }
double spt_memest_position_ids_bytes(double seqlen, double bytes) { return seqlen * bytes; }

// This engine's per-rank device bytes at sequence length s (exact for its ledger, tools/max_seq.py measures
// the same quantity): weights + grads + logits and TiledMLP tile workspaces + per-token activations.
static double engine_device_bytes(const spt_memest_engine& e, double s) {
    const double nl = s / std::max(1, e.sp);
    const double qkv = (double)(e.q_heads + 2 * e.kv_heads) * e.head_dim, qd = (double)e.q_heads * e.head_dim;
    const double p_layer = e.hidden * qkv + e.hidden * qd + 3.0 * e.hidden * e.intermediate + 2.0 * e.hidden;
    const double p_fixed = e.n_layers * p_layer + (e.embed ? 2.0 : 1.0) * e.vocab * e.hidden + e.hidden;
    const double weights = 2.0 * p_fixed, grads = 4.0 * p_fixed;
    // the engine's loss tile and FLCE workspace (tiled.cu), exactly
    const double logits_ws = nl >= 1 ? (double)flce_workspace(flce_default_tile((int64_t)nl, e.vocab), e.vocab) : 0.0;
    const double ckpt = e.n_layers > 1 || e.ckpt_offload ? (e.ckpt_offload ? 0.0 : e.n_layers * nl * e.hidden * 2.0) : 0.0;
    return weights + grads + logits_ws + mlp_ws_bytes(e, nl) + ckpt + e.act_bytes_per_token * nl +
           e.act_bytes_per_seq_token * s;
}

spt_status spt_memest_engine_device_bytes(const spt_memest_engine* e, double seqlen, double* out) {
    return capi_guard([&] { *out = engine_device_bytes(*e, seqlen); });
}

// max_seqlen_solver: largest s (multiple of `granularity`) whose estimate fits the budget,
// by bisection on the monotone estimate; SPT_ERR_OOM when even s = granularity does not fit.
spt_status spt_max_seqlen_solver(const spt_memest_engine* e, double device_budget_bytes, int64_t granularity,
                                 int64_t* out) {
    return capi_guard([&] {
        const int64_t g = std::max<int64_t>(1, granularity);
        if (engine_device_bytes(*e, (double)g) > device_budget_bytes)
            SPT_THROW(SPT_ERR_OOM, "infeasible: " + std::to_string(engine_device_bytes(*e, (double)g)) +
                                       " bytes needed at s=" + std::to_string(g) + ", budget " +
                                       std::to_string(device_budget_bytes));
        int64_t lo = 1, hi = 2;  // in units of g
        while (engine_device_bytes(*e, (double)(hi * g)) <= device_budget_bytes && hi < (int64_t(1) << 40) / g) hi *= 2;
        while (hi - lo > 1) {
            const int64_t mid = lo + (hi - lo) / 2;
            if (engine_device_bytes(*e, (double)(mid * g)) <= device_budget_bytes) lo = mid;
            else hi = mid;
        }
        *out = lo * g;
    });
}

}  // extern "C"
