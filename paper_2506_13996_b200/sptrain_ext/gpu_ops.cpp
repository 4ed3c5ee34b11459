// sptrain::gpu ops (include/sptrain/gpu.hpp): the B200 kernels behind the C-ABI as nodes of the reference's
// autograd graph (tensor.hpp detail::make_op), device memory registered with the ambient MemoryLedger.
//
// Streams and allocation: each host thread (= SP rank) works on its own non-blocking stream per
// device, temporaries come from the stream-ordered allocator (cudaMallocAsync / cudaFreeAsync) and the
// symmetric communication buffers from a per-group pool that is never freed while the group lives: nothing
// here calls a device-synchronising API (cudaFree, legacy-stream copies) while another rank of the same
// process may be waiting in a device-side barrier.
#include <sptrain/gpu.hpp>

#include <cuda_runtime.h>

#include <algorithm>
#include <barrier>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>

namespace sptrain::gpu {

namespace {

[[noreturn]] void raise(spt_status s, const std::string& where) {
    const std::string msg = where + ": " + spt_last_error();
    switch (s) {
        case SPT_ERR_SHAPE: throw ShapeError(msg);
        case SPT_ERR_VALIDATION: throw ValidationError(msg);
        case SPT_ERR_COLLECTIVE: throw CollectiveError(msg);
        case SPT_ERR_PROTOCOL: throw ProtocolError(msg);
        case SPT_ERR_CONFIG: throw ConfigError(msg);
        case SPT_ERR_DETERMINISM: throw DeterminismError(msg);
        case SPT_ERR_OOM: throw SimulatedOomError("device", 0, 0);
        default: throw std::runtime_error(msg);
    }
}

void ck(spt_status s, const char* where) {
    if (s != SPT_OK) raise(s, where);
}

void cu(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(where) + ": " + cudaGetErrorString(e));
}

cudaStream_t stream_for(int device) {
    thread_local std::map<int, cudaStream_t> streams;
    auto it = streams.find(device);
    if (it != streams.end()) return it->second;
    cu(cudaSetDevice(device), "cudaSetDevice");
    cudaStream_t s = nullptr;
    cu(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    streams[device] = s;
    return s;
}

// Device bytes held by an op, charged to the ambient ledger's device tier under `tag` for their lifetime.
struct Dev {
    void* p = nullptr;
    size_t bytes = 0;
    int device = 0;
    cudaStream_t st = nullptr;
    LedgerReg reg;
    Dev(size_t b, MemTag tag, int dev) : bytes(b), device(dev), st(stream_for(dev)),
                                          reg(current_ledger(), Tier::kDevice, tag, b) {
        cu(cudaSetDevice(device), "cudaSetDevice");
        cu(cudaMallocAsync(&p, std::max<size_t>(b, 256), st), "cudaMallocAsync");
    }
    ~Dev() {
        cudaSetDevice(device);
        cudaFreeAsync(p, st);
    }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
};
using DevP = std::shared_ptr<Dev>;

DevP dev(size_t bytes, MemTag tag, int device) { return std::make_shared<Dev>(bytes, tag, device); }

uint16_t to_bf16(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;  // NaN
    u += 0x7fffu + ((u >> 16) & 1u);                     // round to nearest even
    return (uint16_t)(u >> 16);
}

float from_bf16(uint16_t b) {
    const uint32_t u = (uint32_t)b << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

std::vector<uint16_t> bf16_of(const Tensor& t) {
    std::vector<uint16_t> v((size_t)t.numel());
    for (size_t i = 0; i < v.size(); ++i) v[i] = to_bf16((float)t.at(i));
    return v;
}

void h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    cu(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync H2D");
}

void sync(cudaStream_t st) { cu(cudaStreamSynchronize(st), "cudaStreamSynchronize"); }

DevP upload_bf16(const Tensor& t, MemTag tag, int device) {
    auto d = dev((size_t)t.numel() * 2, tag, device);
    const auto v = bf16_of(t);
    h2d(d->p, v.data(), v.size() * 2, d->st);
    sync(d->st);  // the host staging vector dies here
    return d;
}

std::vector<double> download_bf16(const void* p, size_t n, cudaStream_t st) {
    std::vector<uint16_t> h(n);
    cu(cudaMemcpyAsync(h.data(), p, n * 2, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync D2H");
    sync(st);
    std::vector<double> out(n);
    for (size_t i = 0; i < n; ++i) out[i] = from_bf16(h[i]);
    return out;
}

std::vector<double> download_f32(const void* p, size_t n, cudaStream_t st) {
    std::vector<float> h(n);
    cu(cudaMemcpyAsync(h.data(), p, n * 4, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync D2H");
    sync(st);
    return std::vector<double>(h.begin(), h.end());
}

void set_values(const NodePtr& n, const std::vector<double>& v) {
    for (size_t i = 0; i < v.size(); ++i) n->value->set(i, v[i]);
}

std::vector<double> grad_of(const TensorNode& self) {
    std::vector<double> g((size_t)self.numel);
    for (size_t i = 0; i < g.size(); ++i) g[i] = self.grad->get(i);
    return g;
}

Tensor grad_tensor(const TensorNode& self) {  // self.grad as a no-grad host tensor (for upload)
    NoGradGuard ng;
    Tensor t = Tensor::zeros(self.shape, TensorOpts{Dtype::kF64, false});
    for (int64_t i = 0; i < self.numel; ++i) t.set((size_t)i, self.grad->get((size_t)i));
    return t;
}

void need(bool ok, const std::string& msg) {
    if (!ok) throw ShapeError(msg);
}

// ---- in-process bootstrap of a peer group: the spt_allgather_fn of P threads
struct Bootstrap {
    int n;
    std::barrier<> bar;
    std::vector<std::vector<char>> slots;
    explicit Bootstrap(int n_) : n(n_), bar(n_), slots(n_) {}
};
struct Ctx {
    Bootstrap* b;
    int rank;
};

int32_t allgather_threads(const void* in, void* out, size_t bytes, void* user) {
    auto* c = static_cast<Ctx*>(user);
    Bootstrap& b = *c->b;
    b.slots[c->rank].assign((const char*)in, (const char*)in + bytes);
    b.bar.arrive_and_wait();
    for (int r = 0; r < b.n; ++r) std::memcpy((char*)out + (size_t)r * bytes, b.slots[r].data(), bytes);
    b.bar.arrive_and_wait();
    return 0;
}

// Symmetric communication buffers of one group, recycled instead of freed (see the file comment).  Every rank
// acquires / releases in the same order, so the pool stays symmetric.
struct SymPool {
    spt_comm* comm = nullptr;
    std::mutex mu;
    std::multimap<size_t, void*> free_;
    void* acquire(size_t bytes) {
        {
            std::lock_guard<std::mutex> g(mu);
            auto it = free_.find(bytes);
            if (it != free_.end()) {
                void* p = it->second;
                free_.erase(it);
                return p;
            }
        }
        void* p = nullptr;
        ck(spt_comm_alloc(comm, bytes, &p), "spt_comm_alloc");
        ck(spt_comm_connect(comm), "spt_comm_connect");  // collective: every rank maps the new allocation
        return p;
    }
    void release(size_t bytes, void* p) {
        std::lock_guard<std::mutex> g(mu);
        free_.emplace(bytes, p);
    }
};

struct GroupState {
    std::shared_ptr<Bootstrap> boot;
    Ctx ctx{};
    SymPool pool;
};

}  // namespace

struct GroupAccess {
    static GroupState& state(Group& g) { return *static_cast<GroupState*>(g.bootstrap_.get()); }
    static Group* make() { return new Group(); }
    static void set(Group& g, spt_comm* c, int rank, int size, int device, std::shared_ptr<void> st) {
        g.comm_ = c;
        g.rank_ = rank;
        g.size_ = size;
        g.device_ = device;
        g.bootstrap_ = std::move(st);
    }
};

std::vector<std::shared_ptr<Group>> Group::in_process(int nranks, std::vector<int> devices) {
    if (nranks < 1) throw ConfigError("group size must be >= 1");
    if (devices.empty()) devices = {0};
    auto boot = std::make_shared<Bootstrap>(nranks);
    std::vector<std::shared_ptr<GroupState>> states(nranks);
    std::vector<std::shared_ptr<Group>> groups(nranks);
    std::vector<spt_comm*> comms(nranks, nullptr);
    std::vector<std::thread> th;
    std::vector<spt_status> rc(nranks, SPT_OK);
    std::vector<std::string> err(nranks);
    for (int r = 0; r < nranks; ++r) {
        states[r] = std::make_shared<GroupState>();
        states[r]->boot = boot;
        states[r]->ctx = Ctx{boot.get(), r};
    }
    // spt_comm_init_peer exchanges handles collectively: one thread per rank
    for (int r = 0; r < nranks; ++r)
        th.emplace_back([&, r] {
            const int d = devices[(size_t)r % devices.size()];
            cudaSetDevice(d);
            rc[r] = spt_comm_init_peer(nranks, r, d, allgather_threads, &states[r]->ctx, &comms[r]);
            if (rc[r] != SPT_OK) err[r] = spt_last_error();
        });
    for (auto& t : th) t.join();
    for (int r = 0; r < nranks; ++r)
        if (rc[r] != SPT_OK) raise(rc[r], "spt_comm_init_peer (rank " + std::to_string(r) + "): " + err[r]);
    for (int r = 0; r < nranks; ++r) {
        states[r]->pool.comm = comms[r];
        groups[r] = std::shared_ptr<Group>(GroupAccess::make());
        GroupAccess::set(*groups[r], comms[r], r, nranks, devices[(size_t)r % devices.size()], states[r]);
    }
    return groups;
}

std::shared_ptr<Group> Group::single(int device) { return in_process(1, {device})[0]; }

Group::~Group() {
    if (!comm_) return;
    cudaSetDevice(device_);
    cudaDeviceSynchronize();
    spt_comm_destroy(comm_);  // frees the pooled symmetric buffers with the group
}

std::string Group::stats_json() const {
    std::string b(1 << 16, '\0');
    ck(spt_comm_stats_json(comm_, b.data(), b.size()), "spt_comm_stats_json");
    return b.c_str();
}

// ------------------------------------------------------------------------------------------ matmul
Tensor matmul(const Tensor& a, const Tensor& b, int device) {
    need(a.shape().size() == 2 && b.shape().size() == 2 && a.dim(1) == b.dim(0),
         "matmul: shapes " + detail::shape_str(a.shape()) + " and " + detail::shape_str(b.shape()) + " do not agree");
    const int64_t m = a.dim(0), k = a.dim(1), n = b.dim(1);
    need(n % 64 == 0 && k % 8 == 0, "matmul: the tcgen05 GEMM needs n % 64 == 0 and k % 8 == 0, got " +
                                         detail::shape_str(a.shape()) + " x " + detail::shape_str(b.shape()));
    const cudaStream_t st = stream_for(device);
    DevP A = upload_bf16(a, MemTag::kActivationCkpt, device);
    DevP B = upload_bf16(b, MemTag::kActivationCkpt, device);
    DevP C = dev((size_t)(m * n) * 4, MemTag::kWorkspace, device);
    ck(spt_gemm_bf16(A->p, k, 0, B->p, n, 1, C->p, n, 1, 0, nullptr, 0, m, n, k, 1.f, st), "matmul");
    const auto out = download_f32(C->p, (size_t)(m * n), st);
    NodePtr node = detail::make_op("gpu_matmul", {m, n}, a.dtype(), {a.node(), b.node()},
                                   [A, B, m, k, n, device](TensorNode& self) {
        need(m % 8 == 0 && k % 64 == 0, "matmul backward: needs m % 8 == 0 and k % 64 == 0");
        const cudaStream_t s = stream_for(device);
        DevP dC = upload_bf16(grad_tensor(self), MemTag::kWorkspace, device);
        const NodePtr& na = self.inputs[0];
        const NodePtr& nb = self.inputs[1];
        if (na->requires_grad) {  // dA = dC B^T  [m, k]
            DevP dA = dev((size_t)(m * k) * 4, MemTag::kWorkspace, device);
            ck(spt_gemm_bf16(dC->p, n, 0, B->p, n, 0, dA->p, k, 1, 0, nullptr, 0, m, k, n, 1.f, s), "matmul dA");
            na->accumulate_grad(download_f32(dA->p, (size_t)(m * k), s));
        }
        if (nb->requires_grad) {  // dB = A^T dC  [k, n]
            DevP dB = dev((size_t)(k * n) * 4, MemTag::kWorkspace, device);
            ck(spt_gemm_bf16(A->p, k, 1, dC->p, n, 1, dB->p, n, 1, 0, nullptr, 0, k, n, m, 1.f, s), "matmul dB");
            nb->accumulate_grad(download_f32(dB->p, (size_t)(k * n), s));
        }
    });
    set_values(node, out);
    return Tensor(node);
}

// ------------------------------------------------------------------------------------------ rmsnorm
Tensor rmsnorm(const Tensor& x, const Tensor& g, double eps, int device) {
    need(x.shape().size() == 2 && g.numel() == x.dim(1), "rmsnorm: x [n, h] and g [h]");
    const int64_t n = x.dim(0), h = x.dim(1);
    const cudaStream_t st = stream_for(device);
    DevP X = upload_bf16(x, MemTag::kActivationCkpt, device);
    DevP G = upload_bf16(g, MemTag::kWeights, device);
    DevP Y = dev((size_t)(n * h) * 2, MemTag::kWorkspace, device);
    DevP R = dev((size_t)n * 4, MemTag::kActivationCkpt, device);
    ck(spt_rmsnorm_fwd(X->p, G->p, Y->p, (float*)R->p, n, h, (float)eps, st), "rmsnorm");
    const auto out = download_bf16(Y->p, (size_t)(n * h), st);
    NodePtr node = detail::make_op("gpu_rmsnorm", {n, h}, x.dtype(), {x.node(), g.node()},
                                   [X, G, R, n, h, device](TensorNode& self) {
        const cudaStream_t s = stream_for(device);
        DevP dY = upload_bf16(grad_tensor(self), MemTag::kWorkspace, device);
        DevP dX = dev((size_t)(n * h) * 2, MemTag::kWorkspace, device);
        DevP dG = dev((size_t)h * 4, MemTag::kWorkspace, device);
        DevP ws = dev(spt_rmsnorm_bwd_workspace(n, h), MemTag::kWorkspace, device);
        cu(cudaMemsetAsync(dG->p, 0, (size_t)h * 4, s), "memset");
        ck(spt_rmsnorm_bwd(X->p, G->p, (const float*)R->p, dY->p, nullptr, dX->p, (float*)dG->p, ws->p, n, h, s),
           "rmsnorm backward");
        if (self.inputs[0]->requires_grad) self.inputs[0]->accumulate_grad(download_bf16(dX->p, (size_t)(n * h), s));
        if (self.inputs[1]->requires_grad) self.inputs[1]->accumulate_grad(download_f32(dG->p, (size_t)h, s));
    });
    set_values(node, out);
    return Tensor(node);
}

// ------------------------------------------------------------------------------------------ tiled_mlp
Tensor tiled_mlp(const Tensor& x, const Tensor& wg, const Tensor& wu, const Tensor& wd, int num_tiles, int device) {
    need(x.shape().size() == 2, "tiled_mlp: x [s, h]");
    const int64_t s = x.dim(0), h = x.dim(1), I = wg.dim(0);
    need(wg.dim(1) == h && wu.dim(0) == I && wu.dim(1) == h && wd.dim(0) == h && wd.dim(1) == I,
         "tiled_mlp: wg / wu [I, h], wd [h, I]");
    need(h % 64 == 0 && I % 32 == 0, "tiled_mlp: hidden % 64 == 0 and intermediate % 32 == 0");
    const int64_t tiles = num_tiles > 0 ? num_tiles : std::max<int64_t>(1, (s + h - 1) / h);
    const int64_t tile_n = (s + tiles - 1) / tiles;
    const cudaStream_t st = stream_for(device);
    // gate / up rows interleaved in blocks of 32 (the fused SwiGLU epilogue's layout, sptrain_b200.h)
    std::vector<uint16_t> gu((size_t)(2 * I * h));
    const auto g16 = bf16_of(wg), u16 = bf16_of(wu);
    for (int64_t r = 0; r < I; ++r) {
        const int64_t blk = r / 32, off = r % 32;
        std::memcpy(&gu[(size_t)((64 * blk + off) * h)], &g16[(size_t)(r * h)], (size_t)h * 2);
        std::memcpy(&gu[(size_t)((64 * blk + 32 + off) * h)], &u16[(size_t)(r * h)], (size_t)h * 2);
    }
    DevP X = upload_bf16(x, MemTag::kActivationCkpt, device);
    DevP WGU = dev(gu.size() * 2, MemTag::kWeights, device);
    h2d(WGU->p, gu.data(), gu.size() * 2, st);
    DevP WD = upload_bf16(wd, MemTag::kWeights, device);
    DevP Y = dev((size_t)(s * h) * 2, MemTag::kWorkspace, device);
    {
        DevP ws = dev(spt_mlp_workspace(tile_n, I), MemTag::kWorkspace, device);
        ck(spt_mlp_fwd(X->p, WGU->p, WD->p, nullptr, Y->p, s, h, I, tile_n, ws->p, st), "tiled_mlp");
        sync(st);
    }
    const auto out = download_bf16(Y->p, (size_t)(s * h), st);
    NodePtr node = detail::make_op("gpu_tiled_mlp", {s, h}, x.dtype(), {x.node(), wg.node(), wu.node(), wd.node()},
                                   [X, WGU, WD, s, h, I, tile_n, device](TensorNode& self) {
        const cudaStream_t q = stream_for(device);
        DevP dY = upload_bf16(grad_tensor(self), MemTag::kWorkspace, device);
        DevP dX = dev((size_t)(s * h) * 2, MemTag::kWorkspace, device);
        DevP dGU = dev((size_t)(2 * I * h) * 4, MemTag::kWorkspace, device);
        DevP dD = dev((size_t)(h * I) * 4, MemTag::kWorkspace, device);
        DevP ws = dev(spt_mlp_workspace(tile_n, I), MemTag::kWorkspace, device);
        ck(spt_mlp_bwd(X->p, WGU->p, WD->p, dY->p, dX->p, (float*)dGU->p, (float*)dD->p, 0, s, h, I, tile_n, ws->p, q),
           "tiled_mlp backward");
        if (self.inputs[0]->requires_grad) self.inputs[0]->accumulate_grad(download_bf16(dX->p, (size_t)(s * h), q));
        const auto dgu = download_f32(dGU->p, (size_t)(2 * I * h), q);
        std::vector<double> dg((size_t)(I * h)), du((size_t)(I * h));
        for (int64_t r = 0; r < I; ++r) {
            const int64_t blk = r / 32, off = r % 32;
            std::copy_n(&dgu[(size_t)((64 * blk + off) * h)], h, &dg[(size_t)(r * h)]);
            std::copy_n(&dgu[(size_t)((64 * blk + 32 + off) * h)], h, &du[(size_t)(r * h)]);
        }
        if (self.inputs[1]->requires_grad) self.inputs[1]->accumulate_grad(dg);
        if (self.inputs[2]->requires_grad) self.inputs[2]->accumulate_grad(du);
        if (self.inputs[3]->requires_grad) self.inputs[3]->accumulate_grad(download_f32(dD->p, (size_t)(h * I), q));
    });
    set_values(node, out);
    return Tensor(node);
}

// ------------------------------------------------------------------------------------------ tiled_logits_loss
std::pair<Tensor, int64_t> tiled_logits_loss(const Tensor& hidden, const Tensor& w_lm,
                                             const std::vector<int64_t>& shift_labels, int64_t tile_len, int device) {
    need(hidden.shape().size() == 2 && w_lm.shape().size() == 2 && w_lm.dim(1) == hidden.dim(1),
         "tiled_logits_loss: hidden [s, h], W_lm [V, h]");
    const int64_t s = hidden.dim(0), h = hidden.dim(1), V = w_lm.dim(0);
    need((int64_t)shift_labels.size() == s, "tiled_logits_loss: one label per token");
    need(V % 64 == 0 && h % 64 == 0, "tiled_logits_loss: vocab and hidden must be multiples of 64");
    // tile_len * V * 4 <= 1 GiB by default (the paper's ~1 GiB logits shards, SPEC.md:423 budget)
    const int64_t tile = tile_len > 0 ? std::min(tile_len, s)
                                      : std::min<int64_t>(s, std::max<int64_t>(128, (1ll << 30) / (V * 4) / 128 * 128));
    const cudaStream_t st = stream_for(device);
    DevP X = upload_bf16(hidden, MemTag::kActivationCkpt, device);
    DevP W = upload_bf16(w_lm, MemTag::kWeights, device);
    DevP LAB = dev((size_t)s * 8, MemTag::kWorkspace, device);
    h2d(LAB->p, shift_labels.data(), (size_t)s * 8, st);
    struct Sc {
        double loss_sum;
        int64_t count;
        float scale;
        int32_t err;
    };
    DevP SC = dev(sizeof(Sc), MemTag::kWorkspace, device);
    const Sc sc0{0.0, 0, 1.f, 0};  // grads of the loss SUM (scale 1): the caller divides by the count
    h2d(SC->p, &sc0, sizeof(Sc), st);
    auto* scd = static_cast<Sc*>(SC->p);
    DevP dX = dev((size_t)(s * h) * 2, MemTag::kActivationCkpt, device);  // kept for the backward
    DevP dW = dev((size_t)(V * h) * 4, MemTag::kGrads, device);
    {
        DevP ws = dev(spt_flce_workspace(tile, V), MemTag::kLogits, device);  // the only [tile, V] buffer
        ck(spt_label_stats((const int64_t*)LAB->p, s, V, &scd->count, &scd->err, st), "label_stats");
        ck(spt_flce(X->p, W->p, (const int64_t*)LAB->p, s, h, V, tile, &scd->scale, &scd->loss_sum, dX->p,
                    (float*)dW->p, 0, &scd->err, ws->p, st),
           "tiled_logits_loss");
        sync(st);
    }
    Sc sc{};
    cu(cudaMemcpyAsync(&sc, SC->p, sizeof(Sc), cudaMemcpyDeviceToHost, st), "D2H");
    sync(st);
    if (sc.err != 0) throw ValidationError("tiled_logits_loss: label outside [0, " + std::to_string(V) + ") U {-100}");
    NodePtr node = detail::make_op("gpu_tiled_logits_loss", {}, hidden.dtype(), {hidden.node(), w_lm.node()},
                                   [dX, dW, s, h, V, device](TensorNode& self) {
        const cudaStream_t q = stream_for(device);
        const double g = self.grad->get(0);
        if (self.inputs[0]->requires_grad) {
            auto d = download_bf16(dX->p, (size_t)(s * h), q);
            for (double& v : d) v *= g;
            self.inputs[0]->accumulate_grad(d);
        }
        if (self.inputs[1]->requires_grad) {
            auto d = download_f32(dW->p, (size_t)(V * h), q);
            for (double& v : d) v *= g;
            self.inputs[1]->accumulate_grad(d);
        }
    });
    node->value->set(0, sc.loss_sum);
    return {Tensor(node), sc.count};
}

// ------------------------------------------------------------------------------------------ ulysses_attention
Tensor ulysses_attention(Group& group, const Tensor& qkv, int q_heads, int kv_heads, int head_dim,
                         const std::vector<int64_t>* position_ids_full) {
    const int P = group.size();
    const int device = group.device();
    spt_head_shard_plan plan{};
    ck(spt_plan_head_shards(q_heads, kv_heads, P, &plan), "plan_head_shards");
    const int64_t W = (int64_t)(q_heads + 2 * kv_heads) * head_dim;
    need(qkv.shape().size() == 2 && qkv.dim(1) == W,
         "ulysses_attention: qkv [s_loc, (Hq + 2 Hkv) * d], got " + detail::shape_str(qkv.shape()));
    const int64_t s_loc = qkv.dim(0), s = s_loc * P;
    need(s % 128 == 0, "ulysses_attention: the global sequence must be a multiple of 128 (pad_to_multiple)");
    need(!position_ids_full || (int64_t)position_ids_full->size() == s,
         "ulysses_attention: position_ids_full covers the whole sequence");
    const int hq = plan.q_heads_per_rank, hkv = plan.kv_heads_per_rank, hl = hq + 2 * hkv;
    const float scl = 1.f / std::sqrt((float)head_dim);
    const cudaStream_t st = stream_for(device);
    auto& pool = GroupAccess::state(group).pool;
    auto sym = [&pool](size_t bytes) {  // symmetric buffer, back to the pool when the last user drops it
        void* p = pool.acquire(bytes);
        return std::shared_ptr<void>(p, [&pool, bytes](void* q) { pool.release(bytes, q); });
    };
    spt_comm* comm = group.handle();
    DevP X = upload_bf16(qkv, MemTag::kWorkspace, device);
    auto qkv_head = sym((size_t)(s * hl * head_dim) * 2);
    LedgerReg reg_qkv(current_ledger(), Tier::kDevice, MemTag::kCommBuffer, (size_t)(s * hl * head_dim) * 2);
    const void* xs[1] = {X->p};
    void* outs[1] = {qkv_head.get()};
    ck(spt_seq_to_head(comm, &plan, 0, xs, s_loc, head_dim, outs, nullptr, st), "seq_to_head");
    DevP seg;
    if (position_ids_full) {
        DevP pos = dev((size_t)s * 8, MemTag::kWorkspace, device);
        h2d(pos->p, position_ids_full->data(), (size_t)s * 8, st);
        seg = dev((size_t)s * 4 + 16, MemTag::kActivationCkpt, device);
        int32_t* err = (int32_t*)((char*)seg->p + (size_t)s * 4);
        cu(cudaMemsetAsync(err, 0, 4, st), "memset");
        ck(spt_segment_starts((const int64_t*)pos->p, s, (int32_t*)seg->p, err, st), "segment_starts");
        int32_t herr = 0;
        cu(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st), "D2H");
        sync(st);
        if (herr) throw ValidationError("position_ids: not zero-based ascending runs (SPEC.md:245-247)");
    }
    auto o_head = sym((size_t)(s * hq * head_dim) * 2);
    LedgerReg reg_o(current_ledger(), Tier::kDevice, MemTag::kCommBuffer, (size_t)(s * hq * head_dim) * 2);
    DevP LSE = dev((size_t)(hq * s) * 4, MemTag::kActivationCkpt, device);
    const int32_t* segp = seg ? (const int32_t*)seg->p : nullptr;
    ck(spt_attn_fwd(qkv_head.get(), s, hq, hkv, head_dim, segp, scl, o_head.get(), (float*)LSE->p, st), "attention");
    DevP O = dev((size_t)(s_loc * q_heads * head_dim) * 2, MemTag::kWorkspace, device);
    const void* os[1] = {o_head.get()};
    void* oo[1] = {O->p};
    ck(spt_head_to_seq(comm, &plan, 0, os, s_loc, head_dim, oo, nullptr, st), "head_to_seq");
    const auto out = download_bf16(O->p, (size_t)(s_loc * q_heads * head_dim), st);
    auto regs = std::make_shared<std::pair<LedgerReg, LedgerReg>>(std::move(reg_qkv), std::move(reg_o));
    Group* gp = &group;
    NodePtr node = detail::make_op(
        "gpu_ulysses_attention", {s_loc, (int64_t)q_heads * head_dim}, qkv.dtype(), {qkv.node()},
        [gp, plan, qkv_head, o_head, LSE, seg, regs, s_loc, s, hq, hkv, hl, W, q_heads, head_dim, scl,
         device](TensorNode& self) {
            Group& g = *gp;
            auto& pl = GroupAccess::state(g).pool;
            auto symb = [&pl](size_t bytes) {
                void* p = pl.acquire(bytes);
                return std::shared_ptr<void>(p, [&pl, bytes](void* q) { pl.release(bytes, q); });
            };
            const cudaStream_t q = stream_for(device);
            spt_comm* c = g.handle();
            DevP dO = upload_bf16(grad_tensor(self), MemTag::kWorkspace, device);
            auto do_head = symb((size_t)(s * hq * head_dim) * 2);
            const void* xs1[1] = {dO->p};
            void* o1[1] = {do_head.get()};
            ck(spt_seq_to_head(c, &plan, 1, xs1, s_loc, head_dim, o1, nullptr, q), "seq_to_head (dO)");
            auto dqkv_head = symb((size_t)(s * hl * head_dim) * 2);
            DevP ws = dev(spt_attn_bwd_workspace(s, hq, hkv, head_dim), MemTag::kWorkspace, device);
            ck(spt_attn_bwd(qkv_head.get(), o_head.get(), (const float*)LSE->p, do_head.get(), s, hq, hkv, head_dim,
                            seg ? (const int32_t*)seg->p : nullptr, scl, dqkv_head.get(), ws->p, q),
               "attention backward");
            DevP dX = dev((size_t)(s_loc * W) * 2, MemTag::kWorkspace, device);
            const void* xs2[1] = {dqkv_head.get()};
            void* o2[1] = {dX->p};
            ck(spt_head_to_seq(c, &plan, 1, xs2, s_loc, head_dim, o2, nullptr, q), "head_to_seq (dqkv)");
            self.inputs[0]->accumulate_grad(download_bf16(dX->p, (size_t)(s_loc * W), q));
            ck(spt_comm_check(c), "peer group");
        });
    set_values(node, out);
    ck(spt_comm_check(comm), "peer group");
    return Tensor(node);
}

// ------------------------------------------------------------------------------------------ host glue
Tensor add(const Tensor& a, const Tensor& b) {
    need(a.numel() == b.numel(), "add: shapes " + detail::shape_str(a.shape()) + " and " + detail::shape_str(b.shape()));
    NodePtr node = detail::make_op("add", a.shape(), a.dtype(), {a.node(), b.node()}, [](TensorNode& self) {
        const auto g = grad_of(self);
        for (int i = 0; i < 2; ++i)
            if (self.inputs[i]->requires_grad) self.inputs[i]->accumulate_grad(g);
    });
    for (int64_t i = 0; i < a.numel(); ++i) node->value->set((size_t)i, a.at((size_t)i) + b.at((size_t)i));
    return Tensor(node);
}

Tensor scale(const Tensor& a, double c) {
    NodePtr node = detail::make_op("scale", a.shape(), a.dtype(), {a.node()}, [c](TensorNode& self) {
        auto g = grad_of(self);
        for (double& v : g) v *= c;
        if (self.inputs[0]->requires_grad) self.inputs[0]->accumulate_grad(g);
    });
    for (int64_t i = 0; i < a.numel(); ++i) node->value->set((size_t)i, a.at((size_t)i) * c);
    return Tensor(node);
}

}  // namespace sptrain::gpu
