// The sptrain layer-step engine: n_layers Llama-shaped decoder layers + lm_head, fwd + bwd, Ulysses SP.
//
// n_layers == 1 and no offload: the layer's activations stay live from forward to backward.  Otherwise
// every layer input is an activation checkpoint (autograd.hpp:23 CheckpointMode): forward
// keeps only the checkpoints, backward re-runs each layer's forward before its backward; with
// ckpt_offload the checkpoints live in pinned host memory (SPEC.md:462-475 checkpoint_offload), copied
// out on a side stream during forward and prefetched one layer ahead during backward.
//
//   forward:  x1 = x + Wo . ulysses_attention(Wqkv . rms1(x))
//                                  x2 = x1 + tiled_mlp(rms2(x1))
//                                  (loss_sum, count) = tiled_logits_loss(rms3(x2))
//   backward : explicit reverse of the above (the tape order of autograd.hpp:14-17, fixed at build
//              time instead of recorded), weight grads all-reduced over the SP group.
//
// ulysses_attention: K1 pack -> all_to_all (NCCL / loopback) -> attention over the
// full sequence for the local heads -> all_to_all -> K2 unpack; the backward mirrors it with the
// replicate_kv reduction folded into K2.  With the payload layout of SPEC.md:351 the
// seq_to_head receive buffer IS the attention input ([s][heads][d]) and the head_to_seq send buffer
// IS the attention output, so exactly one permutation kernel runs per direction.
//
// Memory: every device byte goes through a MemoryLedger-compatible device ledger (ledger.hpp:37-113
// semantics: per-tag live/peak, largest_single, budgets, summary_json) — the peak-HBM observable.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <unordered_map>
#include <vector>

#include "comm.h"
#include "common.h"
#include "gemm.cuh"
#include "launch.h"
#include "plan.h"
#include "prof.h"

namespace spt {

size_t flce_workspace(int64_t tile_n, int64_t V);
int64_t flce_default_tile(int64_t n_loc, int64_t V);
void flce(const void* x, const void* w, const int64_t* labels, int64_t n, int64_t h, int64_t V, int64_t tile_n,
          const float* scale_dev, double* loss_sum_accum, void* dx, float* dw, bool dw_accumulate, int32_t* err,
          void* ws, cudaStream_t st);
size_t mlp_workspace(int64_t tile_n, int64_t I);
void mlp_fwd(const void* x, const void* wgu, const void* wd, const void* x_res, void* y, int64_t n, int64_t h,
             int64_t I, int64_t tile_n, void* ws, cudaStream_t st);
void mlp_bwd(const void* x, const void* wgu, const void* wd, const void* dy, void* dx, float* dwgu, float* dwd,
             bool accumulate, int64_t n, int64_t h, int64_t I, int64_t tile_n, void* ws, cudaStream_t st);

// ---------------------------------------------------------------- device ledger (ledger.hpp:19-113)
enum Tag { kWeights = 0, kGrads, kOptimizer, kActivationCkpt, kLogits, kWorkspace, kCommBuffer, kNumTags };
static const char* tag_name(int t) {
    static const char* n[] = {"weights", "grads", "optimizer", "activation-checkpoint", "logits", "workspace",
                              "comm-buffer"};
    return n[t];
}

struct DeviceLedger {
    uint64_t host_live = 0, host_peak = 0;  // slow tier: pinned host activation checkpoints
    std::unordered_map<void*, size_t> host_allocs;
    uint64_t live = 0, peak = 0, budget = 0;
    uint64_t tag_live[kNumTags] = {}, tag_peak[kNumTags] = {}, largest[kNumTags] = {};
    uint64_t events = 0;
    // event timeline in the reference's MemoryLedger::timeline_csv form (ledger.cpp:149-157): kind 'A' track /
    // 'R' release, tier device / host, the tag, the signed byte delta and both tiers' live bytes after it
    struct Event {
        uint64_t ordinal;
        char kind;
        bool host;
        int tag;
        int64_t delta;
        uint64_t device_live, host_live;
    };
    std::vector<Event> timeline;
    void push(char kind, bool host, int tag, int64_t delta) {
        timeline.push_back(Event{events, kind, host, tag, delta, live, host_live});
    }
    std::unordered_map<void*, std::pair<int, size_t>> allocs;
    spt_comm* sym_comm = nullptr;  // peer mode: allocations made with alloc_sym are symmetric (comm.h)
    std::unordered_map<void*, char> sym_allocs;

    // symmetric == true: a peer-group allocation, mapped into every rank (same call order on every rank)
    void* alloc(size_t bytes, int tag, bool symmetric = false) {
        if (budget && live + bytes > budget)
            SPT_THROW(SPT_ERR_OOM, "simulated device OOM: required " + std::to_string(live + bytes) +
                                       " bytes, available " + std::to_string(budget));
        void* p = nullptr;
        if (symmetric && sym_comm) {
            p = sym_comm->sym_alloc(bytes);
            sym_allocs[p] = 1;
        } else {
            cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 256));
            if (e != cudaSuccess)
                SPT_THROW(SPT_ERR_OOM, "cudaMalloc(" + std::to_string(bytes) + ") failed: " + cudaGetErrorString(e));
        }
        live += bytes;
        peak = std::max(peak, live);
        tag_live[tag] += bytes;
        tag_peak[tag] = std::max(tag_peak[tag], tag_live[tag]);
        largest[tag] = std::max<uint64_t>(largest[tag], bytes);
        allocs[p] = {tag, bytes};
        push('A', false, tag, (int64_t)bytes);
        ++events;
        return p;
    }
    void release(void* p) {
        auto it = allocs.find(p);
        if (it == allocs.end()) return;
        live -= it->second.second;
        tag_live[it->second.first] -= it->second.second;
        auto si = sym_allocs.find(p);
        if (si != sym_allocs.end()) {
            sym_comm->sym_free(p);
            sym_allocs.erase(si);
        } else {
            cudaFree(p);
        }
        push('R', false, it->second.first, -(int64_t)it->second.second);
        allocs.erase(it);
        ++events;
    }
    void* alloc_host(size_t bytes) {
        void* p = nullptr;
        cudaError_t e = cudaMallocHost(&p, std::max<size_t>(bytes, 256));
        if (e != cudaSuccess)
            SPT_THROW(SPT_ERR_OOM, "host OOM: cudaMallocHost(" + std::to_string(bytes) + ") failed: " +
                                       cudaGetErrorString(e));
        host_live += bytes;
        host_peak = std::max(host_peak, host_live);
        host_allocs[p] = bytes;
        push('A', true, kActivationCkpt, (int64_t)bytes);
        ++events;
        return p;
    }
    void release_all() {
        std::vector<void*> ps;
        for (auto& kv : allocs) ps.push_back(kv.first);
        for (void* p : ps) release(p);
        for (auto& kv : host_allocs) {
            cudaFreeHost(kv.first);
            host_live -= kv.second;
            push('R', true, kActivationCkpt, -(int64_t)kv.second);
            ++events;
        }
        host_allocs.clear();
    }
    std::string timeline_csv() const {
        std::ostringstream os;
        os << "ordinal,kind,tier,tag,delta_bytes,device_live,host_live\n";
        for (const Event& e : timeline)
            os << e.ordinal << "," << e.kind << "," << (e.host ? "host" : "device") << "," << tag_name(e.tag) << ","
               << e.delta << "," << e.device_live << "," << e.host_live << "\n";
        return os.str();
    }
    std::string summary_json() const {
        std::ostringstream os;
        os << "{\"device\":{\"live_bytes\":" << live << ",\"peak_bytes\":" << peak << ",\"tags\":{";
        for (int t = 0; t < kNumTags; ++t)
            os << (t ? "," : "") << "\"" << tag_name(t) << "\":{\"live\":" << tag_live[t] << ",\"peak\":" << tag_peak[t]
               << "}";
        os << "}},\"largest_single\":{";
        for (int t = 0; t < kNumTags; ++t) os << (t ? "," : "") << "\"" << tag_name(t) << "\":" << largest[t];
        os << "},\"host\":{\"live_bytes\":" << host_live << ",\"peak_bytes\":" << host_peak
           << ",\"tags\":{\"activation-checkpoint\":{\"live\":" << host_live << ",\"peak\":" << host_peak << "}}}";
        os << ",\"events\":" << events;
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) == cudaSuccess)
            os << ",\"cuda_mem_used_bytes\":" << (tot - fr) << ",\"cuda_mem_total_bytes\":" << tot;
        os << "}";
        return os.str();
    }
};

// RoPE fused into the K1 pack / K2 unpack when P > 1 (row f4); SPT_ROPE_FUSED=0 or
// spt_tuning_set("rope_fused", 0) keeps the separate in-place rotation pass
int g_rope_fused = [] {
    const char* e = getenv("SPT_ROPE_FUSED");
    return e ? atoi(e) : 1;
}();

// TiledMLP backward tile grouping (1 = the forward's tiles, 2 = pairs of consecutive tiles per recompute /
// weight-gradient pass); SPT_MLP_BWD_GROUP or spt_tuning_set("mlp_bwd_group", v)
// test-only fault injection for the replay verification: flip one bit of the restored checkpoint before the
// next replay (spt_tuning_set("replay_fault", 1)); cleared after use
int g_replay_fault = 0;

int g_mlp_bwd_group = [] {
    const char* e = getenv("SPT_MLP_BWD_GROUP");
    return e ? atoi(e) : 1;
}();

}  // namespace spt

using namespace spt;

struct Scalars {
    double loss_sum;
    int64_t count;
    float scale;
    float loss;
    int32_t err_label;
    int32_t err_pos;
    int32_t err_embed;
    int32_t err_rope;  // a RoPE position outside [0, seq_len) (packed chunk whose ids run past the table)
    int32_t err_replay;  // 1 + layer index whose checkpoint replay differed from its recorded forward
};
// Gradient-accumulation window ("divide by global valid_count summed over the accumulation
// window"): micro-steps accumulate grads of the loss SUM; finish divides by the window's global count.
struct Window {
    double loss_sum;
    int64_t count;
    int64_t one;  // constant 1: finalize_scale(&one) gives the unit grad scale of a micro-step
};

struct RankBufs {
    bf16 *x, *xn1, *qkv, *o, *x1, *xn2, *x2, *z;
    float *rstd1, *rstd2, *rstd3, *lse;
    int64_t *labels, *pos, *ids;
    bf16 *send_qkv, *qkv_head, *o_head, *recv_o;
    bf16 *dz, *dx1, *dO, *dx, *send_do, *do_head, *dqkv_head, *recv_dqkv, *dqkv;
};

struct spt_layer {
    spt_layer_config cfg;
    spt_comm* comm;
    spt_head_shard_plan plan;
    int P, L;
    int64_t N, n_loc, h, I, V, qkv_out, qd, qkv_loc, hq_loc, hkv_loc, mlp_tile, loss_tile, mlp_bwd_tile_max;
    float eps;
    DeviceLedger led;
    Prof prof;
    // weights: per decoder layer + the shared final norm / lm_head
    struct LayerW {
        bf16 *g1, *wqkv, *wo, *g2, *wgu, *wd;
        float *dg1, *dwqkv, *dwo, *dg2, *dwgu, *dwd;
    };
    int NL = 1;            // decoder layers
    bool ckpt = false;     // activation checkpointing (every layer input saved, layers re-run in backward)
    bool offload = false;  // checkpoints in pinned host memory
    bool verify = false;   // checkpoint replays fingerprinted against the recorded forward (autograd.hpp:26-30)
    uint64_t* fp = nullptr;  // [NL + 1]: recorded fingerprint of each layer's output, scratch for the replay's
    std::vector<LayerW> lw;
    bf16 *g3, *wlm;
    void* rope_tab = nullptr;  // RoPE (cos, sin) per (position < N, j < d/2), built once at creation
    bool embed = false;      // token embedding in front of the stack: step inputs are input_ids
    bf16* emb = nullptr;     // [V][h]
    void* ws_emb = nullptr;
    // grads (one contiguous fp32 buffer; SP all-reduce is one call)
    float* gbuf;
    size_t gsize;
    float *dg3, *dwlm, *demb = nullptr;
    std::vector<RankBufs> rb;
    std::vector<std::vector<bf16*>> ck;  // [layer][local rank] checkpointed layer inputs (device or host)
    std::vector<bf16*> xpf;              // [local rank] prefetch buffer for offloaded checkpoints
    // host inputs: copied on their own stream into one of two device staging slots, so the H2D of step i+1
    // overlaps step i's compute when the caller enqueues steps asynchronously (spt_layer_step_async)
    cudaStream_t in_stream = nullptr;
    bf16* in_x[2] = {nullptr, nullptr};
    int64_t* in_lab[2] = {nullptr, nullptr};
    int64_t* in_pos[2] = {nullptr, nullptr};
    cudaEvent_t ev_in_ready[2] = {nullptr, nullptr}, ev_in_free[2] = {nullptr, nullptr};
    int in_slot = 0;
    Scalars* loss_host = nullptr;  // pinned ring for spt_layer_loss_async
    int loss_ring = 0;
    cudaStream_t cstream = nullptr;      // checkpoint copy stream
    cudaEvent_t ev_x_ready = nullptr, ev_ck_done = nullptr, ev_pf_free = nullptr, ev_pf_done = nullptr;
    void *ws_flce, *ws_mlp, *ws_rms, *ws_attn;
    int32_t *map_qkv, *map_q, *gather_o, *gather_qkv;
    int max_src_o, max_src_qkv;
    int32_t* seg;
    int64_t* pos_full;
    Scalars* sc;
    Scalars* sc_host;
    Window* win;
    cudaEvent_t ev_step0, ev_step1;
    float last_step_ms = 0.f;
    cudaGraphExec_t graph_exec = nullptr;  // spt_layer_graph_capture: one device-resident step
    int64_t graph_kernels = 0;             // kernel nodes per replay (launch accounting)
    std::map<std::string, spt_comm::Stat> graph_comm;  // collectives per replay (CommStats accounting)

    bf16* abf(int64_t n, int tag = kWorkspace, bool sym = false) { return (bf16*)led.alloc((size_t)n * 2, tag, sym); }
    float* af32(int64_t n, int tag = kWorkspace, bool sym = false) { return (float*)led.alloc((size_t)n * 4, tag, sym); }
};

static void build_layer(spt_layer* Ly) {
    auto& c = Ly->cfg;
    spt_comm* cm = Ly->comm;
    SPT_CHECK(c.hidden > 0 && c.q_heads > 0 && c.kv_heads > 0 && c.head_dim > 0 && c.intermediate > 0 && c.vocab >= 2,
              SPT_ERR_CONFIG, "invalid layer config");
    Ly->P = cm->nranks;
    Ly->L = cm->local_ranks();
    // peer mode: the buffers other ranks read or write (reshard receive / source buffers, grads and step
    // scalars for the all-reduces, position ids for the all-gather) are symmetric allocations
    const bool sym = cm->peer() && cm->nranks > 1;
    if (sym) Ly->led.sym_comm = cm;
    Ly->plan = plan_head_shards(c.q_heads, c.kv_heads, Ly->P);
    SPT_CHECK(c.seq_len % Ly->P == 0, SPT_ERR_SHAPE,
              "seq_len " + std::to_string(c.seq_len) + " not divisible by SP degree; pad_to_multiple first");
    Ly->N = c.seq_len;
    Ly->n_loc = c.seq_len / Ly->P;
    Ly->h = c.hidden;
    Ly->I = c.intermediate;
    Ly->V = c.vocab;
    Ly->qd = (int64_t)c.q_heads * c.head_dim;
    Ly->qkv_out = (int64_t)(c.q_heads + 2 * c.kv_heads) * c.head_dim;
    Ly->hq_loc = Ly->plan.q_heads_per_rank;
    Ly->hkv_loc = Ly->plan.kv_heads_per_rank;
    Ly->qkv_loc = Ly->hq_loc + 2 * Ly->hkv_loc;
    Ly->eps = c.rms_eps > 0 ? c.rms_eps : 1e-5f;
    SPT_CHECK(Ly->h % 64 == 0 && Ly->qkv_out % 64 == 0 && Ly->I % 32 == 0 && Ly->V % 64 == 0, SPT_ERR_CONFIG,
              "hidden, qkv width and vocab must be multiples of 64, intermediate of 32");
    SPT_CHECK(Ly->N % 128 == 0, SPT_ERR_CONFIG, "seq_len must be a multiple of 128 (attention tile)");
    // TiledMLP tiles.  mlp_tiles > 0: that many; -1: the SPEC default ceil(s/h); 0 (default): the
    // fewest tiles whose per-tile intermediates ([tile, I] x 2 + [tile, 2I] bf16 = tile * I * 8 bytes) fit a
    // fixed 2 GiB budget, split evenly — still O(1) in the sequence length, but 16384-token tiles at
    // Llama-3-8B shapes instead of 4096: the weight-gradient GEMMs accumulate over 4x longer K and the
    // 4096-row GEMMs stop wasting a partial last wave (tools/config_ab.py mlp_tiles: -2.3% step time at L1,
    // profiles/r2_mlp_tiles_ab.json).  Values are tiling-invariant.
    int64_t mtiles;
    if (c.mlp_tiles > 0) mtiles = c.mlp_tiles;
    else if (c.mlp_tiles < 0) mtiles = std::max<int64_t>(1, (Ly->n_loc + Ly->h - 1) / Ly->h);
    else {
        const int64_t tmax = std::max<int64_t>(128, (int64_t)((2ll << 30) / (Ly->I * 8)) / 128 * 128);
        mtiles = std::max<int64_t>(1, (Ly->n_loc + tmax - 1) / tmax);
    }
    Ly->mlp_tile = (Ly->n_loc + mtiles - 1) / mtiles;
    if (c.loss_tile > 0) Ly->loss_tile = std::min<int64_t>(c.loss_tile, Ly->n_loc);
    else {
        Ly->loss_tile = flce_default_tile(Ly->n_loc, Ly->V);  // tiled.cu
    }
    auto& L_ = Ly->led;
    const int64_t h = Ly->h, I = Ly->I, V = Ly->V;
    Ly->NL = std::max(1, c.n_layers);
    Ly->offload = c.ckpt_offload != 0;
    Ly->ckpt = Ly->NL > 1 || Ly->offload;
    Ly->verify = Ly->ckpt && c.verify_replay != 0;
    // weights
    Ly->lw.resize(Ly->NL);
    for (auto& w : Ly->lw) {
        w.g1 = Ly->abf(h, kWeights);
        w.wqkv = Ly->abf(Ly->qkv_out * h, kWeights);
        w.wo = Ly->abf(h * Ly->qd, kWeights);
        w.g2 = Ly->abf(h, kWeights);
        w.wgu = Ly->abf(2 * I * h, kWeights);
        w.wd = Ly->abf(h * I, kWeights);
    }
    Ly->g3 = Ly->abf(h, kWeights);
    Ly->wlm = Ly->abf(V * h, kWeights);
    Ly->embed = c.embed != 0;
    if (Ly->embed) Ly->emb = Ly->abf(V * h, kWeights);
    // grads: [layer 0 .. NL-1: g1, wqkv, wo, g2, wgu, wd] [g3] [wlm] [emb], 64-float aligned segments
    const size_t lsz[6] = {(size_t)h, (size_t)(Ly->qkv_out * h), (size_t)(h * Ly->qd), (size_t)h, (size_t)(2 * I * h),
                           (size_t)(h * I)};
    auto al = [](size_t s) { return (s + 63) / 64 * 64; };
    size_t tot = al((size_t)h) + al((size_t)(V * h)) + (Ly->embed ? al((size_t)(V * h)) : 0);
    for (int l = 0; l < Ly->NL; ++l)
        for (size_t s : lsz) tot += al(s);
    Ly->gsize = tot;
    Ly->gbuf = Ly->af32(tot, kGrads, sym);
    float* gp = Ly->gbuf;
    for (auto& w : Ly->lw) {
        float** dst[6] = {&w.dg1, &w.dwqkv, &w.dwo, &w.dg2, &w.dwgu, &w.dwd};
        for (int i = 0; i < 6; ++i) {
            *dst[i] = gp;
            gp += al(lsz[i]);
        }
    }
    Ly->dg3 = gp;
    gp += al((size_t)h);
    Ly->dwlm = gp;
    gp += al((size_t)(V * h));
    if (Ly->embed) Ly->demb = gp;
    // per-rank activations
    const int64_t nl = Ly->n_loc, N = Ly->N, P = Ly->P;
    Ly->rb.resize(Ly->L);
    for (auto& r : Ly->rb) {
        // the layer input: it IS the saved activation when layers are not checkpointed; with checkpointing the
        // saved copies live in Ly->ck and this is the working buffer
        r.x = Ly->abf(nl * h, Ly->ckpt ? kWorkspace : kActivationCkpt);
        r.xn1 = Ly->abf(nl * h);
        r.qkv = Ly->abf(nl * Ly->qkv_out);
        r.o = Ly->abf(nl * Ly->qd);
        r.x1 = Ly->abf(nl * h);
        r.xn2 = Ly->abf(nl * h);
        r.x2 = Ly->abf(nl * h);
        r.z = Ly->abf(nl * h);
        r.rstd1 = Ly->af32(nl);
        r.rstd2 = Ly->af32(nl);
        r.rstd3 = Ly->af32(nl);
        r.lse = Ly->af32(Ly->hq_loc * N);
        r.labels = (int64_t*)L_.alloc(nl * 8, kWorkspace);
        r.pos = (int64_t*)L_.alloc(nl * 8, kWorkspace, sym);
        r.ids = Ly->embed ? (int64_t*)L_.alloc(nl * 8, kWorkspace) : nullptr;
        r.dz = Ly->abf(nl * h);
        r.dx1 = Ly->abf(nl * h);
        r.dO = Ly->abf(nl * Ly->qd);
        r.dx = Ly->abf(nl * h);
        if (P > 1) {
            // head-sharded buffers [N][heads_loc][d]: the seq_to_head receive buffers (q|k|v, dO) and the
            // head_to_seq sources (O, dq|dk|dv).  Only NCCL needs the contiguous send / receive staging: the
            // loopback and peer transports store into / load from these directly (comm.h fused_*).
            const bool staged = cm->mode == spt_comm::kNccl;
            r.qkv_head = Ly->abf(N * Ly->qkv_loc * c.head_dim, kCommBuffer, sym);
            r.o_head = Ly->abf(N * Ly->hq_loc * c.head_dim, kCommBuffer, sym);
            r.do_head = Ly->abf(N * Ly->hq_loc * c.head_dim, kCommBuffer, sym);
            r.dqkv_head = Ly->abf(N * Ly->qkv_loc * c.head_dim, kCommBuffer, sym);
            r.send_qkv = staged ? Ly->abf(N * Ly->qkv_loc * c.head_dim, kCommBuffer) : nullptr;
            r.recv_o = staged ? Ly->abf(N * Ly->hq_loc * c.head_dim, kCommBuffer) : nullptr;
            r.send_do = staged ? Ly->abf(N * Ly->hq_loc * c.head_dim, kCommBuffer) : nullptr;
            r.recv_dqkv = staged ? Ly->abf(N * Ly->qkv_loc * c.head_dim, kCommBuffer) : nullptr;
            r.dqkv = Ly->abf(nl * Ly->qkv_out);
        } else {
            r.send_qkv = r.recv_o = r.send_do = r.recv_dqkv = nullptr;
            r.qkv_head = r.qkv;
            r.o_head = r.o;
            r.do_head = r.dO;
            r.dqkv = Ly->abf(nl * Ly->qkv_out);
            r.dqkv_head = r.dqkv;
        }
    }
    // activation checkpoints: L * (s/P) * h * 2 bytes per rank (SPEC.md:470 closed form)
    if (Ly->ckpt) {
        Ly->ck.assign(Ly->NL, std::vector<bf16*>(Ly->L, nullptr));
        for (int l = 0; l < Ly->NL; ++l)
            for (int r = 0; r < Ly->L; ++r)
                Ly->ck[l][r] = Ly->offload ? (bf16*)L_.alloc_host((size_t)nl * h * 2) : Ly->abf(nl * h, kActivationCkpt);
        if (Ly->offload) {
            Ly->xpf.resize(Ly->L);
            for (auto& p : Ly->xpf) p = Ly->abf(nl * h);
            SPT_CUDA(cudaStreamCreateWithFlags(&Ly->cstream, cudaStreamNonBlocking));
            for (cudaEvent_t* e : {&Ly->ev_x_ready, &Ly->ev_ck_done, &Ly->ev_pf_free, &Ly->ev_pf_done})
                SPT_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
    }
    // workspaces (shared by local ranks; phases run back to back on one stream)
    Ly->ws_flce = L_.alloc(flce_workspace(Ly->loss_tile, V), kLogits);
    // the backward may run the TiledMLP tiles in groups of g_mlp_bwd_group (fewer, longer weight-gradient
    // accumulation passes); the workspace is sized for the group in force at construction and the backward
    // never uses a larger one
    Ly->mlp_bwd_tile_max = std::min<int64_t>(Ly->n_loc, Ly->mlp_tile * std::max(1, std::min(2, g_mlp_bwd_group)));
    Ly->ws_mlp = L_.alloc(mlp_workspace(Ly->mlp_bwd_tile_max, I), kWorkspace);
    Ly->ws_rms = L_.alloc(rmsnorm_bwd_workspace(nl, h), kWorkspace);
    Ly->ws_attn = L_.alloc(attn_bwd_workspace(N, Ly->hq_loc, Ly->hkv_loc, c.head_dim), kWorkspace);
    if (Ly->embed) Ly->ws_emb = L_.alloc(embed_bwd_workspace(nl, V), kWorkspace);
    if (c.rope_theta > 0.f) {  // every position a step can use is < N (global index, or within a packed sample)
        Ly->rope_tab = L_.alloc((size_t)N * (c.head_dim / 2) * 8, kWorkspace);
        rope_table(Ly->rope_tab, N, c.head_dim, c.rope_theta, nullptr);
        SPT_CUDA(cudaStreamSynchronize(nullptr));
    }
    // reshard tables
    auto up = [&](const std::vector<int32_t>& v) {
        int32_t* d = (int32_t*)L_.alloc(v.size() * 4, kWorkspace);
        SPT_CUDA(cudaMemcpy(d, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
        return d;
    };
    Ly->map_qkv = up(qkv_pack_map(Ly->plan));
    Ly->map_q = up(q_pack_map(Ly->plan));
    Ly->gather_o = up(o_gather_map(Ly->plan, &Ly->max_src_o));
    Ly->gather_qkv = up(qkv_gather_map(Ly->plan, &Ly->max_src_qkv));
    Ly->seg = c.packed ? (int32_t*)L_.alloc(N * 4, kWorkspace) : nullptr;
    Ly->pos_full = c.packed ? (int64_t*)L_.alloc(N * 8, kWorkspace) : nullptr;
    Ly->sc = (Scalars*)L_.alloc(sizeof(Scalars), kWorkspace, sym);
    if (Ly->verify) Ly->fp = (uint64_t*)L_.alloc((Ly->NL + 1) * 8, kWorkspace);
    Ly->win = (Window*)L_.alloc(sizeof(Window), kWorkspace);
    {
        const Window w0{0.0, 0, 1};
        SPT_CUDA(cudaMemcpy(Ly->win, &w0, sizeof(Window), cudaMemcpyHostToDevice));
    }
    SPT_CUDA(cudaMallocHost(&Ly->sc_host, sizeof(Scalars)));
    SPT_CUDA(cudaEventCreate(&Ly->ev_step0));
    SPT_CUDA(cudaEventCreate(&Ly->ev_step1));
    if (sym) cm->connect();  // collective: map every rank's symmetric allocations of this engine
}

static double gflop(int64_t m, int64_t n, int64_t k) { return 2.0 * (double)m * n * k; }

static void apply_update(spt_layer* Ly, cudaStream_t st);

// mode 0: one complete step (mean loss of this step, grads all-reduced).  mode 1 / 2: first / later micro-step
// of a gradient-accumulation window (grads of the loss sum accumulated locally; spt_layer_finish_accumulation
// all-reduces them and divides by the window's global valid count).
static void layer_step(spt_layer* Ly, const void* x, const int64_t* labels, const int64_t* pos, bool on_host,
                       cudaStream_t st, int mode = 0) {
    auto& c = Ly->cfg;
    const bool gbase = mode == 2;  // grads accumulate onto the previous micro-steps'
    const bool micro = mode != 0;
    const bool rope_on = c.rope_theta > 0.f;
    spt_comm* cm = Ly->comm;
    const int L = Ly->L, P = Ly->P, d = c.head_dim, NL = Ly->NL;
    const int64_t nl = Ly->n_loc, N = Ly->N, h = Ly->h, I = Ly->I, V = Ly->V, qd = Ly->qd, qo = Ly->qkv_out;
    const int hq = Ly->hq_loc, hkv = Ly->hkv_loc;
    const float scale = 1.f / std::sqrt((float)d);
    Prof& pf = Ly->prof;
    pf.reset();
    current_prof() = &pf;
    struct ProfReset {
        ~ProfReset() { current_prof() = nullptr; }
    } prof_reset_guard;
    SPT_CUDA(cudaEventRecord(Ly->ev_step0, st));
    const cudaMemcpyKind kind = on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;

    // ---- inputs, label pre-pass, global count
    SPT_CUDA(cudaMemsetAsync(Ly->sc, 0, sizeof(Scalars), st));
    // x rows: bf16 hidden rows, or (embedding on) int64 input_ids gathered through the table
    const size_t xrow = Ly->embed ? 8 : (size_t)h * 2;
    auto load_x = [&](RankBufs& b, const uint8_t* src, cudaMemcpyKind kd) {
        if (!Ly->embed) {
            SPT_CUDA(cudaMemcpyAsync(b.x, src, nl * h * 2, kd, st));
            return;
        }
        SPT_CUDA(cudaMemcpyAsync(b.ids, src, nl * 8, kd, st));
        pf.run(P_OTHER, 0, 2.0 * nl * h * 2, st, [&] { embed_fwd(b.ids, nl, V, h, Ly->emb, b.x, &Ly->sc->err_embed, st); });
    };
    if (on_host) {
        // H2D on the input stream into a staging slot (overlaps the previous step's compute), then one fast
        // D2D into the working buffers once the copy landed
        if (!Ly->in_stream) {
            SPT_CUDA(cudaStreamCreateWithFlags(&Ly->in_stream, cudaStreamNonBlocking));
            for (int k = 0; k < 2; ++k) {
                Ly->in_x[k] = Ly->abf((int64_t)L * nl * h);
                Ly->in_lab[k] = (int64_t*)Ly->led.alloc((size_t)L * nl * 8, kWorkspace);
                Ly->in_pos[k] = (int64_t*)Ly->led.alloc((size_t)L * nl * 8, kWorkspace);
                SPT_CUDA(cudaEventCreateWithFlags(&Ly->ev_in_ready[k], cudaEventDisableTiming));
                SPT_CUDA(cudaEventCreateWithFlags(&Ly->ev_in_free[k], cudaEventDisableTiming));
                SPT_CUDA(cudaEventRecord(Ly->ev_in_free[k], st));
            }
        }
        const int k = Ly->in_slot;
        Ly->in_slot ^= 1;
        SPT_CUDA(cudaStreamWaitEvent(Ly->in_stream, Ly->ev_in_free[k], 0));
        SPT_CUDA(cudaMemcpyAsync(Ly->in_x[k], x, (size_t)L * nl * xrow, cudaMemcpyHostToDevice, Ly->in_stream));
        SPT_CUDA(cudaMemcpyAsync(Ly->in_lab[k], labels, (size_t)L * nl * 8, cudaMemcpyHostToDevice, Ly->in_stream));
        if (c.packed)
            SPT_CUDA(cudaMemcpyAsync(Ly->in_pos[k], pos, (size_t)L * nl * 8, cudaMemcpyHostToDevice, Ly->in_stream));
        SPT_CUDA(cudaEventRecord(Ly->ev_in_ready[k], Ly->in_stream));
        SPT_CUDA(cudaStreamWaitEvent(st, Ly->ev_in_ready[k], 0));
        x = Ly->in_x[k];
        labels = Ly->in_lab[k];
        pos = c.packed ? Ly->in_pos[k] : pos;
        for (int r = 0; r < L; ++r) {
            auto& b = Ly->rb[r];
            load_x(b, (const uint8_t*)x + r * nl * xrow, cudaMemcpyDeviceToDevice);
            SPT_CUDA(cudaMemcpyAsync(b.labels, labels + r * nl, nl * 8, cudaMemcpyDeviceToDevice, st));
            if (c.packed) SPT_CUDA(cudaMemcpyAsync(b.pos, pos + r * nl, nl * 8, cudaMemcpyDeviceToDevice, st));
        }
        SPT_CUDA(cudaEventRecord(Ly->ev_in_free[k], st));  // staging slot consumed
        for (int r = 0; r < L; ++r) label_stats(Ly->rb[r].labels, nl, V, &Ly->sc->count, &Ly->sc->err_label, st);
    } else {
        for (int r = 0; r < L; ++r) {
            auto& b = Ly->rb[r];
            load_x(b, (const uint8_t*)x + r * nl * xrow, kind);
            SPT_CUDA(cudaMemcpyAsync(b.labels, labels + r * nl, nl * 8, kind, st));
            if (c.packed) SPT_CUDA(cudaMemcpyAsync(b.pos, pos + r * nl, nl * 8, kind, st));
            label_stats(b.labels, nl, V, &Ly->sc->count, &Ly->sc->err_label, st);
        }
    }
    cm->all_reduce("all_reduce_count", &Ly->sc->count, 1, ncclInt64, st);
    finalize_scale(micro ? &Ly->win->one : &Ly->sc->count, &Ly->sc->scale, st);
    if (c.packed) {  // position_ids_full -> run starts
        if (cm->loopback) {
            for (int r = 0; r < L; ++r)
                SPT_CUDA(cudaMemcpyAsync(Ly->pos_full + r * nl, Ly->rb[r].pos, nl * 8, cudaMemcpyDeviceToDevice, st));
        } else {
            cm->all_gather("all_gather_position_ids", Ly->rb[0].pos, Ly->pos_full, nl * 8, st);
        }
        segment_starts(Ly->pos_full, N, Ly->seg, &Ly->sc->err_pos, st);
    }
    if (!gbase) {
        SPT_CUDA(cudaMemsetAsync(Ly->dg3, 0, h * 4, st));
        for (auto& w : Ly->lw) {
            SPT_CUDA(cudaMemsetAsync(w.dg1, 0, h * 4, st));
            SPT_CUDA(cudaMemsetAsync(w.dg2, 0, h * 4, st));
        }
    }

    const size_t qkv_row = (size_t)Ly->qkv_loc * d * 2, o_row = (size_t)hq * d * 2;  // bytes per head-sharded row
    const double qkv_a2a = (double)nl * qkv_row * (P - 1), o_a2a = (double)nl * o_row * (P - 1);  // payload / rank
    auto ptrs = [&](bf16* RankBufs::*m) {
        std::vector<void*> v;
        for (auto& b : Ly->rb) v.push_back(b.*m);
        return v;
    };
    const double attn_f = 4.0 * (double)N * N * hq * d / 2.0;  // causal half
    // RoPE positions are < N (global index, or an index within a packed sample); anything else is flagged
    const int64_t npos = N;
    int32_t* rope_err = &Ly->sc->err_rope;
    // K1 fused with RoPE when the rotation runs on the way into the peers' buffers (row f4)
    const bool rope_in_pack = rope_on && P > 1 && g_rope_fused && d % 16 == 0 && (d == 32 || d == 64 || d == 128) &&
                              (size_t)P * Ly->qkv_loc * 4 <= 48 * 1024;

    // ---- one decoder layer forward: b.x -> b.x2 (intermediates left in the rank buffers)
    auto layer_fwd = [&](const spt_layer::LayerW& w) {
        for (int r = 0; r < L; ++r) {  // phase A: rms1, fused QKV projection (+ RoPE in place unless fused below)
            auto& b = Ly->rb[r];
            pf.run(P_NORM, 0, 2.0 * nl * h * 2, st, [&] { rmsnorm_fwd(b.x, w.g1, b.xn1, b.rstd1, nl, h, Ly->eps, st); });
            EpiParams e;
            e.C = b.qkv;
            e.ldc = qo;
            gemm({b.xn1, h, false}, {w.wqkv, h, false}, nl, qo, h, EPI_BF16, e, st);
            if (rope_on && !rope_in_pack)  // rotate q and k heads in place before the reshard / attention
                pf.run(P_OTHER, 0, 2.0 * nl * (c.q_heads + c.kv_heads) * d * 2, st, [&] {
                    rope_apply(b.qkv, nl, c.q_heads + 2 * c.kv_heads, c.q_heads + c.kv_heads, d,
                               c.packed ? b.pos : nullptr, (int64_t)cm->global_rank(r) * nl, c.rope_theta, false, st,
                               Ly->rope_tab, npos, rope_err);
                });
        }
        if (P > 1) {  // seq_to_head: K1 stores every packed row straight into its destination rank's buffer
            pf.next_tag = "a2a_qkv";
            pf.run(P_A2A, 0, qkv_a2a * L, st, [&] {
                fused_seq_to_head(cm, "all_to_all_qkv", ptrs(&RankBufs::qkv_head), Ly->rb[0].send_qkv, nl,
                                  (int64_t)qkv_row, st, [&](int r, const RowTab& t) {
                    auto& b = Ly->rb[r];
                    if (rope_in_pack)
                        reshard_pack_rope(b.qkv, nl, c.q_heads + 2 * c.kv_heads, d, P, (int)Ly->qkv_loc, Ly->map_qkv,
                                          t, c.q_heads + c.kv_heads, c.packed ? b.pos : nullptr,
                                          (int64_t)cm->global_rank(r) * nl, c.rope_theta, st, Ly->rope_tab, npos,
                                          rope_err);
                    else
                        reshard_pack(b.qkv, nl, c.q_heads + 2 * c.kv_heads, d, P, (int)Ly->qkv_loc, Ly->map_qkv, t, st);
                });
            });
        }
        for (int r = 0; r < L; ++r) {  // attention over the full sequence, local heads
            auto& b = Ly->rb[r];
            pf.run(P_ATTN_F, attn_f, 0, st, [&] { attn_fwd(b.qkv_head, N, hq, hkv, d, Ly->seg, scale, b.o_head, b.lse, st); });
        }
        if (P > 1) {  // head_to_seq: K2 loads every row straight from its source rank's attention output
            pf.next_tag = "a2a_o";
            pf.run(P_A2A, 0, o_a2a * L, st, [&] {
                fused_head_to_seq(cm, "all_to_all_o", ptrs(&RankBufs::o_head), Ly->rb[0].recv_o, nl, (int64_t)o_row,
                                  st, [&](int r, const RowTab& t) {
                    reshard_unpack(t, nl, hq, d, P, c.q_heads, Ly->gather_o, Ly->max_src_o, Ly->rb[r].o, st);
                });
            });
        }
        for (int r = 0; r < L; ++r) {  // phase B: O projection + residual, rms2, TiledMLP + residual
            auto& b = Ly->rb[r];
            EpiParams e;
            e.C = b.x1;
            e.ldc = h;
            e.R = b.x;
            e.ldr = h;
            gemm({b.o, qd, false}, {w.wo, qd, false}, nl, h, qd, EPI_BF16, e, st);
            pf.run(P_NORM, 0, 2.0 * nl * h * 2, st, [&] { rmsnorm_fwd(b.x1, w.g2, b.xn2, b.rstd2, nl, h, Ly->eps, st); });
            mlp_fwd(b.xn2, w.wgu, w.wd, b.x1, b.x2, nl, h, I, Ly->mlp_tile, Ly->ws_mlp, st);
        }
    };
    // ---- one decoder layer backward: dy = b.dx (d of the layer output) -> b.dx (d of the layer input)
    auto layer_bwd = [&](const spt_layer::LayerW& w) {
        for (int r = 0; r < L; ++r) {
            auto& b = Ly->rb[r];
            const bool acc = r > 0 || gbase;  // loopback ranks share the grad buffer: rank-ascending
            bf16* dx2 = b.dx;
            bf16* dxn2 = b.dz;
            mlp_bwd(b.xn2, w.wgu, w.wd, dx2, dxn2, w.dwgu, w.dwd, acc, nl, h, I,
                    std::min<int64_t>(Ly->mlp_bwd_tile_max, Ly->mlp_tile * std::max(1, g_mlp_bwd_group)), Ly->ws_mlp,
                    st);
            pf.run(P_NORM, 0, 4.0 * nl * h * 2, st,
                   [&] { rmsnorm_bwd(b.x1, w.g2, b.rstd2, dxn2, dx2, b.dx1, w.dg2, Ly->ws_rms, nl, h, st); });
            EpiParams e1;
            e1.C = b.dO;
            e1.ldc = qd;
            gemm({b.dx1, h, false}, {w.wo, qd, true}, nl, qd, h, EPI_BF16, e1, st);
            EpiParams e2;
            e2.C = w.dwo;
            e2.ldc = qd;
            e2.accumulate = acc;
            gemm({b.dx1, h, true}, {b.o, qd, true}, h, qd, nl, EPI_F32, e2, st);
        }
        if (P > 1) {  // seq_to_head of dO (the mirror of head_to_seq of O)
            pf.next_tag = "a2a_do";
            pf.run(P_A2A, 0, o_a2a * L, st, [&] {
                fused_seq_to_head(cm, "all_to_all_do", ptrs(&RankBufs::do_head), Ly->rb[0].send_do, nl,
                                  (int64_t)o_row, st, [&](int r, const RowTab& t) {
                    reshard_pack(Ly->rb[r].dO, nl, c.q_heads, d, P, hq, Ly->map_q, t, st);
                });
            });
        }
        for (int r = 0; r < L; ++r) {
            auto& b = Ly->rb[r];
            pf.run(P_ATTN_B, attn_f * 2.5, 0, st, [&] {
                attn_bwd(b.qkv_head, b.o_head, b.lse, b.do_head, N, hq, hkv, d, Ly->seg, scale, b.dqkv_head, Ly->ws_attn, st);
            });
        }
        bool dqkv_rotated = false;  // inverse RoPE already applied by the fused K2 unpack
        if (P > 1) {  // head_to_seq of d(q|k|v), replicas of a kv head summed in fp32 rank order
            dqkv_rotated = rope_in_pack;
            pf.next_tag = "a2a_dqkv";
            pf.run(P_A2A, 0, qkv_a2a * L, st, [&] {
                fused_head_to_seq(cm, "all_to_all_dqkv", ptrs(&RankBufs::dqkv_head), Ly->rb[0].recv_dqkv, nl,
                                  (int64_t)qkv_row, st, [&](int r, const RowTab& t) {
                    auto& b = Ly->rb[r];
                    if (rope_in_pack)  // row f4: inverse RoPE fused into the K2 unpack
                        reshard_unpack_rope(t, nl, (int)Ly->qkv_loc, d, c.q_heads + 2 * c.kv_heads, Ly->gather_qkv,
                                            Ly->max_src_qkv, b.dqkv, c.q_heads + c.kv_heads, c.packed ? b.pos : nullptr,
                                            (int64_t)cm->global_rank(r) * nl, c.rope_theta, st, Ly->rope_tab, npos,
                                            rope_err);
                    else
                        reshard_unpack(t, nl, (int)Ly->qkv_loc, d, P, c.q_heads + 2 * c.kv_heads, Ly->gather_qkv,
                                       Ly->max_src_qkv, b.dqkv, st);
                });
            });
        }
        for (int r = 0; r < L; ++r) {
            auto& b = Ly->rb[r];
            const bool acc = r > 0 || gbase;
            bf16* dxn1 = b.dz;
            if (rope_on && !dqkv_rotated)  // d(q, k) through the rotation's transpose, before the projection's backward
                pf.run(P_OTHER, 0, 2.0 * nl * (c.q_heads + c.kv_heads) * d * 2, st, [&] {
                    rope_apply(b.dqkv, nl, c.q_heads + 2 * c.kv_heads, c.q_heads + c.kv_heads, d,
                               c.packed ? b.pos : nullptr, (int64_t)cm->global_rank(r) * nl, c.rope_theta, true, st,
                               Ly->rope_tab, npos, rope_err);
                });
            EpiParams e1;
            e1.C = dxn1;
            e1.ldc = h;
            gemm({b.dqkv, qo, false}, {w.wqkv, h, true}, nl, h, qo, EPI_BF16, e1, st);
            EpiParams e2;
            e2.C = w.dwqkv;
            e2.ldc = h;
            e2.accumulate = acc;
            gemm({b.dqkv, qo, true}, {b.xn1, h, true}, qo, h, nl, EPI_F32, e2, st);
            pf.run(P_NORM, 0, 4.0 * nl * h * 2, st,
                   [&] { rmsnorm_bwd(b.x, w.g1, b.rstd1, dxn1, b.dx1, b.dx, w.dg1, Ly->ws_rms, nl, h, st); });
        }
    };
    // ---- activation checkpoints (offload SPEC.md:462-475)
    auto ckpt_save = [&](int l) {
        if (!Ly->offload) {
            for (int r = 0; r < L; ++r)
                SPT_CUDA(cudaMemcpyAsync(Ly->ck[l][r], Ly->rb[r].x, nl * h * 2, cudaMemcpyDeviceToDevice, st));
            return;
        }
        // D2H on the copy stream once the layer input is ready; the main stream only waits for it before it
        // overwrites b.x with the next layer's input (one layer forward later)
        SPT_CUDA(cudaEventRecord(Ly->ev_x_ready, st));
        SPT_CUDA(cudaStreamWaitEvent(Ly->cstream, Ly->ev_x_ready, 0));
        for (int r = 0; r < L; ++r)
            SPT_CUDA(cudaMemcpyAsync(Ly->ck[l][r], Ly->rb[r].x, nl * h * 2, cudaMemcpyDeviceToHost, Ly->cstream));
        SPT_CUDA(cudaEventRecord(Ly->ev_ck_done, Ly->cstream));
    };
    auto prefetch = [&](int l) {  // offload: H2D of checkpoint l into the prefetch buffers
        SPT_CUDA(cudaEventRecord(Ly->ev_pf_free, st));
        SPT_CUDA(cudaStreamWaitEvent(Ly->cstream, Ly->ev_pf_free, 0));
        for (int r = 0; r < L; ++r)
            SPT_CUDA(cudaMemcpyAsync(Ly->xpf[r], Ly->ck[l][r], nl * h * 2, cudaMemcpyHostToDevice, Ly->cstream));
        SPT_CUDA(cudaEventRecord(Ly->ev_pf_done, Ly->cstream));
    };
    auto ckpt_restore = [&](int l) {
        if (!Ly->offload) {
            for (int r = 0; r < L; ++r)
                SPT_CUDA(cudaMemcpyAsync(Ly->rb[r].x, Ly->ck[l][r], nl * h * 2, cudaMemcpyDeviceToDevice, st));
            return;
        }
        SPT_CUDA(cudaStreamWaitEvent(st, Ly->ev_pf_done, 0));
        for (int r = 0; r < L; ++r) std::swap(Ly->rb[r].x, Ly->xpf[r]);
    };

    // fingerprint of a layer's output (every local rank's rows), for the replay verification
    auto fingerprint = [&](uint64_t* out) {
        SPT_CUDA(cudaMemsetAsync(out, 0, 8, st));
        for (int r = 0; r < L; ++r) fingerprint_bf16(Ly->rb[r].x2, nl * h, out, st);
    };
    // ---- forward through the layers (only the checkpoints survive when checkpointing)
    for (int l = 0; l < NL; ++l) {
        if (Ly->ckpt) ckpt_save(l);
        layer_fwd(Ly->lw[l]);
        if (Ly->verify && l + 1 < NL) fingerprint(Ly->fp + l);  // the recorded forward of a replayed layer
        if (l + 1 < NL) {
            if (Ly->offload) SPT_CUDA(cudaStreamWaitEvent(st, Ly->ev_ck_done, 0));  // b.x copied out
            for (int r = 0; r < L; ++r)
                SPT_CUDA(cudaMemcpyAsync(Ly->rb[r].x, Ly->rb[r].x2, nl * h * 2, cudaMemcpyDeviceToDevice, st));
        }
    }
    if (Ly->offload) SPT_CUDA(cudaStreamWaitEvent(st, Ly->ev_ck_done, 0));
    // ---- final norm + tiled logits/loss (fwd+bwd fused) -> dy of the last layer in b.dx
    for (int r = 0; r < L; ++r) {
        auto& b = Ly->rb[r];
        const bool acc = r > 0 || gbase;
        pf.run(P_NORM, 0, 2.0 * nl * h * 2, st, [&] { rmsnorm_fwd(b.x2, Ly->g3, b.z, b.rstd3, nl, h, Ly->eps, st); });
        flce(b.z, Ly->wlm, b.labels, nl, h, V, Ly->loss_tile, &Ly->sc->scale, &Ly->sc->loss_sum, b.dz, Ly->dwlm,
             acc, &Ly->sc->err_label, Ly->ws_flce, st);
        pf.run(P_NORM, 0, 3.0 * nl * h * 2, st,
               [&] { rmsnorm_bwd(b.x2, Ly->g3, b.rstd3, b.dz, nullptr, b.dx, Ly->dg3, Ly->ws_rms, nl, h, st); });
    }
    // ---- backward through the layers (re-running each layer's forward from its checkpoint).  The last
    // layer's forward state is still live in the rank buffers (the head only touches z/dz/dx), so it is not
    // re-run; its checkpoint is still saved, keeping the SPEC.md:470 byte count L * (s/P) * h.
    if (Ly->offload && NL > 1) prefetch(NL - 2);
    for (int l = NL - 1; l >= 0; --l) {
        if (Ly->ckpt && l < NL - 1) {
            ckpt_restore(l);
            if (Ly->offload && l > 0) prefetch(l - 1);  // overlaps this layer's recompute + backward
            if (g_replay_fault) {
                flip_lowest_bit(Ly->rb[0].x, st);
                g_replay_fault = 0;
            }
            layer_fwd(Ly->lw[l]);
            if (Ly->verify) {  // the replay must be bit-identical to the recorded forward (autograd.hpp:26-30)
                fingerprint(Ly->fp + NL);
                fingerprint_compare(Ly->fp + l, Ly->fp + NL, &Ly->sc->err_replay, l + 1, st);
            }
        }
        layer_bwd(Ly->lw[l]);
    }
    if (Ly->embed) {  // d loss / d table: per-id sums of the stack's input gradient, ascending token order
        for (int r = 0; r < L; ++r) {
            auto& b = Ly->rb[r];
            pf.run(P_OTHER, 0, 2.0 * nl * h * 2, st, [&] {
                embed_bwd(b.ids, nl, V, h, b.dx, Ly->demb, r > 0 || gbase, &Ly->sc->err_embed, Ly->ws_emb, st);
            });
        }
    }
    // ---- SP-group reductions
    if (micro) {  // window totals only; the grad all-reduce waits for the end of the window
        cm->all_reduce("all_reduce_loss_sum", &Ly->sc->loss_sum, 1, ncclFloat64, st);
        window_accumulate(&Ly->sc->loss_sum, &Ly->sc->count, &Ly->win->loss_sum, &Ly->win->count, mode == 1, st);
        SPT_CUDA(cudaEventRecord(Ly->ev_step1, st));
        cm->check_async();
        return;
    }
    pf.run(P_COMM, 0, (double)Ly->gsize * 4, st, [&] {
        cm->all_reduce("all_reduce_grads", Ly->gbuf, Ly->gsize, ncclFloat32, st);
        cm->all_reduce("all_reduce_loss_sum", &Ly->sc->loss_sum, 1, ncclFloat64, st);
    });
    finalize_loss(&Ly->sc->loss_sum, &Ly->sc->count, &Ly->sc->loss, st);
    apply_update(Ly, st);
    SPT_CUDA(cudaEventRecord(Ly->ev_step1, st));
    cm->check_async();
}

// end of an accumulation window: all-reduce the accumulated grads, divide by the window's global count
static void finish_accumulation(spt_layer* Ly, cudaStream_t st) {
    spt_comm* cm = Ly->comm;
    cm->all_reduce("all_reduce_grads", Ly->gbuf, Ly->gsize, ncclFloat32, st);
    scale_by_inverse_count(Ly->gbuf, (int64_t)Ly->gsize, &Ly->win->count, st);
    window_finalize(&Ly->win->loss_sum, &Ly->win->count, &Ly->sc->loss_sum, &Ly->sc->count, &Ly->sc->loss, st);
    apply_update(Ly, st);
    cm->check_async();
}

static void apply_update(spt_layer* Ly, cudaStream_t st) {
    auto& c = Ly->cfg;
    const int64_t h = Ly->h, I = Ly->I, V = Ly->V, qd = Ly->qd, qo = Ly->qkv_out;
    Prof& pf = Ly->prof;
    if (c.lr > 0.f) {
        pf.run(P_OTHER, 0, 0, st, [&] {
            for (auto& w : Ly->lw) {
                sgd_update(w.wqkv, w.dwqkv, qo * h, c.lr, st);
                sgd_update(w.wo, w.dwo, h * qd, c.lr, st);
                sgd_update(w.wgu, w.dwgu, 2 * I * h, c.lr, st);
                sgd_update(w.wd, w.dwd, h * I, c.lr, st);
                sgd_update(w.g1, w.dg1, h, c.lr, st);
                sgd_update(w.g2, w.dg2, h, c.lr, st);
            }
            sgd_update(Ly->wlm, Ly->dwlm, V * h, c.lr, st);
            sgd_update(Ly->g3, Ly->dg3, h, c.lr, st);
            if (Ly->embed) sgd_update(Ly->emb, Ly->demb, V * h, c.lr, st);
        });
    }
}

static void read_scalars(spt_layer* Ly, cudaStream_t st, float* loss, int64_t* count) {
    SPT_CUDA(cudaMemcpyAsync(Ly->sc_host, Ly->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, st));
    Ly->comm->wait_stream(st);  // host watchdog: a stalled collective -> ProtocolError, not a hang
    SPT_CHECK(Ly->sc_host->err_label == 0, SPT_ERR_VALIDATION, "label out of range [0, vocab) and != -100");
    SPT_CHECK(Ly->sc_host->err_pos == 0, SPT_ERR_VALIDATION, "position_ids not zero-based ascending runs");
    SPT_CHECK(Ly->sc_host->err_embed == 0, SPT_ERR_VALIDATION, "input id out of range [0, vocab)");
    SPT_CHECK(Ly->sc_host->err_rope == 0, SPT_ERR_VALIDATION, "RoPE position id outside [0, seq_len)");
    SPT_CHECK(Ly->sc_host->err_replay == 0, SPT_ERR_DETERMINISM,
              "checkpoint replay of layer " + std::to_string(Ly->sc_host->err_replay - 1) +
                  " is not bit-identical to its recorded forward");
    if (loss) *loss = Ly->sc_host->loss;
    if (count) *count = Ly->sc_host->count;
}

// Parameter names: "g1", "wqkv", "wo", "g2", "wg", "wu", "wd" (layer 0) or "layers.<i>.<name>" for layer i,
// plus the shared "g3" and "wlm".  Returns the layer index (-1 for shared) and the bare name.
static int split_name(spt_layer* Ly, const std::string& full, std::string* bare) {
    if (full.rfind("layers.", 0) == 0) {
        const size_t dot = full.find('.', 7);
        SPT_CHECK(dot != std::string::npos, SPT_ERR_VALIDATION, "bad parameter name '" + full + "'");
        const int l = std::atoi(full.substr(7, dot - 7).c_str());
        SPT_CHECK(l >= 0 && l < Ly->NL, SPT_ERR_VALIDATION, "layer index out of range in '" + full + "'");
        *bare = full.substr(dot + 1);
        SPT_CHECK(*bare != "g3" && *bare != "wlm" && *bare != "emb", SPT_ERR_VALIDATION,
                  "'" + *bare + "' is not a per-layer parameter");
        return l;
    }
    *bare = full;
    return (full == "g3" || full == "wlm" || full == "emb") ? -1 : 0;
}

static bf16* param_ptr(spt_layer* Ly, const std::string& full, int64_t* numel, int* layer = nullptr) {
    const int64_t h = Ly->h, I = Ly->I;
    std::string n;
    const int l = split_name(Ly, full, &n);
    if (layer) *layer = l;
    if (n == "g3") return *numel = h, Ly->g3;
    if (n == "wlm") return *numel = Ly->V * h, Ly->wlm;
    if (n == "emb") {
        SPT_CHECK(Ly->embed, SPT_ERR_VALIDATION, "'emb' needs a layer created with embed = 1");
        return *numel = Ly->V * h, Ly->emb;
    }
    auto& w = Ly->lw[l];
    if (n == "g1") return *numel = h, w.g1;
    if (n == "g2") return *numel = h, w.g2;
    if (n == "wqkv") return *numel = Ly->qkv_out * h, w.wqkv;
    if (n == "wo") return *numel = h * Ly->qd, w.wo;
    if (n == "wd") return *numel = h * I, w.wd;
    if (n == "wg" || n == "wu") return *numel = I * h, nullptr;
    SPT_THROW(SPT_ERR_VALIDATION, "unknown parameter name '" + full + "'");
}

static float* grad_ptr(spt_layer* Ly, const std::string& full) {
    std::string n;
    const int l = split_name(Ly, full, &n);
    if (n == "g3") return Ly->dg3;
    if (n == "wlm") return Ly->dwlm;
    if (n == "emb") {
        SPT_CHECK(Ly->embed, SPT_ERR_VALIDATION, "'emb' needs a layer created with embed = 1");
        return Ly->demb;
    }
    auto& w = Ly->lw[l];
    if (n == "g1") return w.dg1;
    if (n == "g2") return w.dg2;
    if (n == "wqkv") return w.dwqkv;
    if (n == "wo") return w.dwo;
    if (n == "wd") return w.dwd;
    SPT_THROW(SPT_ERR_VALIDATION, "unknown parameter name '" + full + "'");
}

extern "C" {

spt_status spt_layer_create(const spt_layer_config* cfg, spt_comm* comm, spt_layer** out) {
    return capi_guard([&] {
        SPT_CHECK(cfg && comm && out, SPT_ERR_CONFIG, "null argument");
        SPT_CUDA(cudaSetDevice(comm->device));
        (void)num_sms();  // validates sm_100
        auto Ly = std::make_unique<spt_layer>();  // value-init: POD members zeroed
        Ly->cfg = *cfg;
        Ly->comm = comm;
        try {
            build_layer(Ly.get());
        } catch (...) {
            Ly->led.release_all();
            throw;
        }
        *out = Ly.release();
    });
}

spt_status spt_layer_destroy(spt_layer* Ly) {
    return capi_guard([&] {
        if (!Ly) return;
        cudaDeviceSynchronize();
        if (Ly->graph_exec) cudaGraphExecDestroy(Ly->graph_exec);
        Ly->led.release_all();
        if (Ly->sc_host) cudaFreeHost(Ly->sc_host);
        for (auto e : Ly->prof.pool) cudaEventDestroy(e);
        cudaEventDestroy(Ly->ev_step0);
        cudaEventDestroy(Ly->ev_step1);
        for (cudaEvent_t e : {Ly->ev_x_ready, Ly->ev_ck_done, Ly->ev_pf_free, Ly->ev_pf_done})
            if (e) cudaEventDestroy(e);
        if (Ly->cstream) cudaStreamDestroy(Ly->cstream);
        if (Ly->in_stream) cudaStreamDestroy(Ly->in_stream);
        for (int k = 0; k < 2; ++k) {
            if (Ly->ev_in_ready[k]) cudaEventDestroy(Ly->ev_in_ready[k]);
            if (Ly->ev_in_free[k]) cudaEventDestroy(Ly->ev_in_free[k]);
        }
        if (Ly->loss_host) cudaFreeHost(Ly->loss_host);
        delete Ly;
    });
}

spt_status spt_layer_param_numel(spt_layer* Ly, const char* name, int64_t* numel) {
    return capi_guard([&] {
        SPT_CHECK(numel != nullptr, SPT_ERR_CONFIG, "null numel");
        param_ptr(Ly, std::string(name), numel);
    });
}

spt_status spt_layer_set_param(spt_layer* Ly, const char* name, const void* data, int32_t data_on_host) {
    return capi_guard([&] {
        int64_t n = 0;
        std::string full(name), nm;
        int layer = 0;
        bf16* p = param_ptr(Ly, full, &n, &layer);
        split_name(Ly, full, &nm);
        const cudaMemcpyKind k = data_on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        if (p) {
            SPT_CUDA(cudaMemcpy(p, data, n * 2, k));
            return;
        }
        // gate / up rows go into the interleaved [2I, h] weight
        void* tmp = nullptr;
        SPT_CUDA(cudaMalloc(&tmp, n * 2));
        SPT_CUDA(cudaMemcpy(tmp, data, n * 2, k));
        interleave_gu(nm == "wg" ? tmp : nullptr, nm == "wu" ? tmp : nullptr, Ly->lw[layer].wgu, Ly->I, Ly->h, 0);
        SPT_CUDA(cudaDeviceSynchronize());
        cudaFree(tmp);
    });
}

spt_status spt_layer_step_async(spt_layer* Ly, const void* x, const int64_t* shift_labels, const int64_t* position_ids,
                                int32_t inputs_on_host, void* stream) {
    return capi_guard([&] {
        SPT_CHECK(!Ly->cfg.packed || position_ids, SPT_ERR_VALIDATION, "packed config needs position_ids");
        layer_step(Ly, x, shift_labels, position_ids, inputs_on_host != 0, (cudaStream_t)stream);
    });
}

// CUDA graph of one full step with device-resident inputs (fixed pointers; contents may change between
// replays): the ~100 launches of a step replay without per-launch host overhead or inter-kernel gaps.
// Capture on a non-default stream; tuning switches are read at capture time.  With profiling on, the per-kernel-class
// events are captured as external event-record nodes: spt_layer_timing_json after a replay reports that replay.
spt_status spt_layer_graph_capture(spt_layer* Ly, const void* x, const int64_t* shift_labels,
                                   const int64_t* position_ids, void* stream) {
    return capi_guard([&] {
        cudaStream_t st = (cudaStream_t)stream;
        SPT_CHECK(st != nullptr, SPT_ERR_CONFIG, "graph capture needs a non-default stream");
        SPT_CHECK(!Ly->cfg.packed || position_ids, SPT_ERR_VALIDATION, "packed config needs position_ids");
        // one eager step first: first-use setup (kernel attributes, lazily created buffers) stays out of the graph
        layer_step(Ly, x, shift_labels, position_ids, false, st);
        SPT_CUDA(cudaStreamSynchronize(st));
        cudaGraph_t g = nullptr;
        const auto stats0 = Ly->comm->stats;
        SPT_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        const int64_t n0 = launch_count();
        try {
            layer_step(Ly, x, shift_labels, position_ids, false, st);
        } catch (...) {
            cudaStreamEndCapture(st, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        SPT_CUDA(cudaStreamEndCapture(st, &g));
        if (Ly->graph_exec) cudaGraphExecDestroy(Ly->graph_exec);
        Ly->graph_exec = nullptr;
        const cudaError_t e = cudaGraphInstantiate(&Ly->graph_exec, g, 0);
        cudaGraphDestroy(g);
        SPT_CUDA(e);
        Ly->graph_kernels = launch_count() - n0;
        // the collectives one replay performs (CommStats keep counting across replays)
        Ly->graph_comm.clear();
        for (auto& kv : Ly->comm->stats) {
            auto it = stats0.find(kv.first);
            spt_comm::Stat d = kv.second;
            if (it != stats0.end()) {
                d.calls -= it->second.calls;
                d.bytes_sent -= it->second.bytes_sent;
            }
            if (d.calls) Ly->graph_comm[kv.first] = d;
        }
    });
}

spt_status spt_layer_graph_launch(spt_layer* Ly, void* stream) {
    return capi_guard([&] {
        SPT_CHECK(Ly->graph_exec != nullptr, SPT_ERR_CONFIG, "no captured step (spt_layer_graph_capture)");
        // step events recorded around the replay (inside the capture they were graph nodes, not records), so
        // spt_layer_timing_json reports the replayed step
        SPT_CUDA(cudaEventRecord(Ly->ev_step0, (cudaStream_t)stream));
        SPT_CUDA(cudaGraphLaunch(Ly->graph_exec, (cudaStream_t)stream));
        SPT_CUDA(cudaEventRecord(Ly->ev_step1, (cudaStream_t)stream));
        add_launches(Ly->graph_kernels);
        for (auto& kv : Ly->graph_comm) {
            auto& st = Ly->comm->stats[kv.first];
            st.calls += kv.second.calls;
            st.bytes_sent += kv.second.bytes_sent;
        }
    });
}

spt_status spt_layer_step_accumulate(spt_layer* Ly, const void* x, const int64_t* shift_labels,
                                     const int64_t* position_ids, int32_t inputs_on_host, int32_t first_micro_step,
                                     void* stream) {
    return capi_guard([&] {
        SPT_CHECK(!Ly->cfg.packed || position_ids, SPT_ERR_VALIDATION, "packed config needs position_ids");
        layer_step(Ly, x, shift_labels, position_ids, inputs_on_host != 0, (cudaStream_t)stream,
                   first_micro_step ? 1 : 2);
    });
}

spt_status spt_layer_finish_accumulation(spt_layer* Ly, float* loss_out, int64_t* count_out, void* stream) {
    return capi_guard([&] {
        finish_accumulation(Ly, (cudaStream_t)stream);
        read_scalars(Ly, (cudaStream_t)stream, loss_out, count_out);
    });
}

// Enqueue (no sync) a D2H copy of this step's scalars into slot `slot` of a pinned ring of 64 entries; the
// value is valid once the stream reaches it: read it with spt_layer_loss_slot after synchronising.
spt_status spt_layer_loss_async(spt_layer* Ly, int32_t slot, void* stream) {
    return capi_guard([&] {
        SPT_CHECK(slot >= 0 && slot < 64, SPT_ERR_SHAPE, "loss slot must be in [0, 64)");
        if (!Ly->loss_host) SPT_CUDA(cudaMallocHost(&Ly->loss_host, 64 * sizeof(Scalars)));
        SPT_CUDA(cudaMemcpyAsync(Ly->loss_host + slot, Ly->sc, sizeof(Scalars), cudaMemcpyDeviceToHost,
                                 (cudaStream_t)stream));
    });
}

spt_status spt_layer_loss_slot(spt_layer* Ly, int32_t slot, float* loss_out, int64_t* count_out) {
    return capi_guard([&] {
        SPT_CHECK(Ly->loss_host && slot >= 0 && slot < 64, SPT_ERR_SHAPE, "no such loss slot");
        const Scalars& v = Ly->loss_host[slot];
        SPT_CHECK(v.err_label == 0, SPT_ERR_VALIDATION, "label out of range [0, vocab) and != -100");
        SPT_CHECK(v.err_pos == 0, SPT_ERR_VALIDATION, "position_ids not zero-based ascending runs");
        SPT_CHECK(v.err_embed == 0, SPT_ERR_VALIDATION, "input id out of range [0, vocab)");
        SPT_CHECK(v.err_rope == 0, SPT_ERR_VALIDATION, "RoPE position id outside [0, seq_len)");
        SPT_CHECK(v.err_replay == 0, SPT_ERR_DETERMINISM,
                  "checkpoint replay of layer " + std::to_string(v.err_replay - 1) +
                      " is not bit-identical to its recorded forward");
        if (loss_out) *loss_out = v.loss;
        if (count_out) *count_out = v.count;
    });
}

spt_status spt_layer_read_loss(spt_layer* Ly, float* loss_out, int64_t* count_out, void* stream) {
    return capi_guard([&] { read_scalars(Ly, (cudaStream_t)stream, loss_out, count_out); });
}

spt_status spt_layer_step(spt_layer* Ly, const void* x, const int64_t* shift_labels, const int64_t* position_ids,
                          int32_t inputs_on_host, float* loss_out, int64_t* count_out, void* stream) {
    return capi_guard([&] {
        SPT_CHECK(!Ly->cfg.packed || position_ids, SPT_ERR_VALIDATION, "packed config needs position_ids");
        layer_step(Ly, x, shift_labels, position_ids, inputs_on_host != 0, (cudaStream_t)stream);
        read_scalars(Ly, (cudaStream_t)stream, loss_out, count_out);
    });
}

spt_status spt_layer_get_grad(spt_layer* Ly, const char* name, float* host_out) {
    return capi_guard([&] {
        std::string full(name), n;
        const int layer = split_name(Ly, full, &n);
        SPT_CUDA(cudaDeviceSynchronize());
        if (n == "wg" || n == "wu") {
            const size_t cnt = (size_t)Ly->I * Ly->h;
            float *g = nullptr, *u = nullptr;
            SPT_CUDA(cudaMalloc(&g, cnt * 4));
            SPT_CUDA(cudaMalloc(&u, cnt * 4));
            deinterleave_gu_f32(Ly->lw[layer].dwgu, g, u, Ly->I, Ly->h, 0);
            SPT_CUDA(cudaMemcpy(host_out, n == "wg" ? g : u, cnt * 4, cudaMemcpyDeviceToHost));
            cudaFree(g);
            cudaFree(u);
            return;
        }
        int64_t numel = 0;
        param_ptr(Ly, full, &numel);
        SPT_CUDA(cudaMemcpy(host_out, grad_ptr(Ly, full), numel * 4, cudaMemcpyDeviceToHost));
    });
}

spt_status spt_layer_get_dx(spt_layer* Ly, void* host_out) {
    return capi_guard([&] {
        SPT_CUDA(cudaDeviceSynchronize());
        const size_t per = (size_t)Ly->n_loc * Ly->h * 2;
        for (int r = 0; r < Ly->L; ++r)
            SPT_CUDA(cudaMemcpy((char*)host_out + r * per, Ly->rb[r].dx, per, cudaMemcpyDeviceToHost));
    });
}

spt_status spt_layer_memory_json(spt_layer* Ly, char* buf, size_t cap) {
    return capi_guard([&] {
        std::ostringstream os;
        os << "{\"ledger\":" << Ly->led.summary_json() << ",\"tokens_per_rank\":" << Ly->n_loc
           << ",\"local_ranks\":" << Ly->L << ",\"n_layers\":" << Ly->NL << ",\"activation_checkpointing\":"
           << (Ly->ckpt ? "true" : "false") << ",\"ckpt_offload\":" << (Ly->offload ? "true" : "false")
           << ",\"rope_theta\":" << Ly->cfg.rope_theta << ",\"mlp_tile\":" << Ly->mlp_tile
           << ",\"loss_tile\":" << Ly->loss_tile
           << ",\"comm\":" << Ly->comm->stats_json() << "}";
        std::string s = os.str();
        SPT_CHECK(s.size() + 1 <= cap, SPT_ERR_SHAPE, "buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

spt_status spt_layer_memory_timeline_csv(spt_layer* Ly, char* buf, size_t cap) {
    return capi_guard([&] {
        const std::string s = Ly->led.timeline_csv();
        SPT_CHECK(s.size() + 1 <= cap, SPT_ERR_SHAPE, "buffer too small: need " + std::to_string(s.size() + 1));
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

spt_status spt_layer_set_profiling(spt_layer* Ly, int32_t on) {
    return capi_guard([&] { Ly->prof.on = on != 0; });
}

spt_status spt_layer_timing_json(spt_layer* Ly, char* buf, size_t cap) {
    return capi_guard([&] {
        SPT_CUDA(cudaEventSynchronize(Ly->ev_step1));
        float ms = 0;
        SPT_CUDA(cudaEventElapsedTime(&ms, Ly->ev_step0, Ly->ev_step1));
        std::ostringstream os;
        os << "{\"step_ms\":" << ms << ",\"classes\":" << Ly->prof.json() << ",\"gaps\":" << Ly->prof.gaps_json()
           << "}";
        std::string s = os.str();
        SPT_CHECK(s.size() + 1 <= cap, SPT_ERR_SHAPE, "buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

}  // extern "C"
