// The reference's C++ API end to end: a program written against /root/reference/proj/include/sptrain
// (Tensor / TensorNode / detail::make_op, MemoryLedger / LedgerScope, backward / checkpoint / finite_diff_grad)
// linked with the reference's own tensor.cpp / ledger.cpp, this repo's autograd.cpp and the sptrain::gpu ops.
//
//   --cpu                       autograd engine checks on host ops (SPEC.md:26-121 examples and properties)
//   --gpu IN OUT [ckpt]         one Llama-shaped layer + lm_head step built from sptrain::gpu ops on one rank,
//                               optionally the decoder layer under sptrain::checkpoint; writes loss, count,
//                               grads, d x and the ledger's summary_json for the Python checker
//   --gpu-sp P IN OUT           the same step with P SP ranks as P host threads (one rank per thread,
//                               SPEC.md:110) on the peer transport; weight grads summed over ranks in rank order
// Exit code 0 = pass (the Python test compares the GPU outputs against the numpy oracle).
#include <sptrain/autograd.hpp>
#include <sptrain/gpu.hpp>
#include <sptrain/ledger.hpp>
#include <sptrain/tensor.hpp>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

using namespace sptrain;

static int fails = 0;
#define EXPECT(c)                                                    \
    do {                                                             \
        if (!(c)) {                                                  \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                                 \
        }                                                            \
    } while (0)

// ------------------------------------------------------------------------------------ host test ops
static Tensor hmatmul(const Tensor& a, const Tensor& b) {
    const int64_t m = a.dim(0), k = a.dim(1), n = b.dim(1);
    NodePtr node = detail::make_op("matmul", {m, n}, a.dtype(), {a.node(), b.node()}, [m, k, n](TensorNode& self) {
        const NodePtr &A = self.inputs[0], &B = self.inputs[1];
        std::vector<double> da((size_t)(m * k), 0.0), db((size_t)(k * n), 0.0);
        for (int64_t i = 0; i < m; ++i)
            for (int64_t j = 0; j < n; ++j) {
                const double g = self.grad->get((size_t)(i * n + j));
                for (int64_t t = 0; t < k; ++t) {
                    da[(size_t)(i * k + t)] += g * B->value->get((size_t)(t * n + j));
                    db[(size_t)(t * n + j)] += A->value->get((size_t)(i * k + t)) * g;
                }
            }
        if (A->requires_grad) A->accumulate_grad(da);
        if (B->requires_grad) B->accumulate_grad(db);
    });
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            double acc = 0;
            for (int64_t t = 0; t < k; ++t) acc += a.at((size_t)(i * k + t)) * b.at((size_t)(t * n + j));
            node->value->set((size_t)(i * n + j), acc);
        }
    return Tensor(node);
}

static Tensor htanh(const Tensor& x) {
    NodePtr node = detail::make_op("tanh", x.shape(), x.dtype(), {x.node()}, [](TensorNode& self) {
        std::vector<double> g((size_t)self.numel);
        for (size_t i = 0; i < g.size(); ++i) {
            const double y = self.value->get(i);
            g[i] = self.grad->get(i) * (1 - y * y);
        }
        self.inputs[0]->accumulate_grad(g);
    });
    for (int64_t i = 0; i < x.numel(); ++i) node->value->set((size_t)i, std::tanh(x.at((size_t)i)));
    return Tensor(node);
}

static Tensor hsum(const Tensor& x) {
    NodePtr node = detail::make_op("sum", {}, x.dtype(), {x.node()}, [](TensorNode& self) {
        const NodePtr& in = self.inputs[0];
        self.inputs[0]->accumulate_grad(std::vector<double>((size_t)in->numel, self.grad->get(0)));
    });
    double s = 0;
    for (int64_t i = 0; i < x.numel(); ++i) s += x.at((size_t)i);
    node->value->set(0, s);
    return Tensor(node);
}

static double max_rel(const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num += (a[i] - b[i]) * (a[i] - b[i]);
        den += b[i] * b[i];
    }
    return std::sqrt(num / (den > 0 ? den : 1));
}

static void cpu_tests() {
    std::mt19937_64 rng(7);
    MemoryLedger led;
    LedgerScope scope(led);
    Tensor x = Tensor::randn({3, 4}, rng, 1.0, {Dtype::kF64, true});
    Tensor w = Tensor::randn({4, 2}, rng, 1.0, {Dtype::kF64, true});
    auto f = [&](const Tensor& xx) {
        NoGradGuard ng;
        return hsum(htanh(hmatmul(xx, w))).item();
    };
    // tape gradient vs finite differences (rel < 1e-6 at 64-bit, eps 1e-5)
    Tensor loss = hsum(htanh(hmatmul(x, w)));
    backward(loss);
    const auto gx = x.grad_vector();
    EXPECT(max_rel(gx, finite_diff_grad(f, x, 1e-5).to_vector()) < 1e-6);
    // finite_diff_grad of sum x^2 at [1, 2] -> [2, 4]
    Tensor p = Tensor::from_values({2}, {1.0, 2.0});
    auto fd = finite_diff_grad([](const Tensor& t) { return t.at(0) * t.at(0) + t.at(1) * t.at(1); }, p, 1e-5);
    EXPECT(std::abs(fd.at(0) - 2.0) < 1e-8 && std::abs(fd.at(1) - 4.0) < 1e-8);
    // additive accumulation across backward passes
    Tensor loss2 = hsum(htanh(hmatmul(x, w)));
    backward(loss2);
    const auto gx2 = x.grad_vector();
    for (size_t i = 0; i < gx.size(); ++i) EXPECT(gx2[i] == 2 * gx[i]);
    // checkpoint == plain in values (bit-exact) and grads; offload parks x on the host tier
    for (auto mode : {CheckpointMode::kPlain, CheckpointMode::kOffload}) {
        x.zero_grad();
        w.zero_grad();
        Tensor h = Tensor::randn({3, 4}, rng, 1.0, {Dtype::kF64, true});
        Tensor plain = htanh(hmatmul(h, w));
        const auto pv = plain.to_vector();
        backward(hsum(plain));
        const auto gh = h.grad_vector(), gw = w.grad_vector();
        h.zero_grad();
        w.zero_grad();
        const uint64_t host0 = led.live_bytes(Tier::kHost);
        Tensor ck = checkpoint([&](const Tensor& t) { return htanh(hmatmul(t, w)); }, h, mode);
        EXPECT(ck.to_vector() == pv);
        if (mode == CheckpointMode::kOffload) EXPECT(led.live_bytes(Tier::kHost) == host0 + 3 * 4 * 8);
        backward(hsum(ck));
        EXPECT(led.live_bytes(Tier::kHost) == host0);
        EXPECT(max_rel(h.grad_vector(), gh) <= 1e-12 && max_rel(w.grad_vector(), gw) <= 1e-12);
        EXPECT(ck.buffer().released());  // autograd.hpp:29-30
    }
    // a non-reentrant region -> DeterminismError on replay (errors.hpp:36-40)
    int calls = 0;
    Tensor h = Tensor::randn({3, 4}, rng, 1.0, {Dtype::kF64, true});
    Tensor bad = checkpoint([&](const Tensor& t) { return htanh(hmatmul(calls++ ? hmatmul(t, Tensor::full({4, 4}, 0.5)) : t, w)); }, h);
    bool det = false;
    try {
        backward(hsum(bad));
    } catch (const DeterminismError&) {
        det = true;
    }
    EXPECT(det);
    // backward is deterministic: identical runs give bit-identical grads
    x.zero_grad();
    backward(hsum(htanh(hmatmul(x, w))));
    const auto r1 = x.grad_vector();
    x.zero_grad();
    backward(hsum(htanh(hmatmul(x, w))));
    EXPECT(x.grad_vector() == r1);
    // backward of a non-scalar without a seed -> ShapeError
    bool shape = false;
    try {
        backward(hmatmul(x, w));
    } catch (const ShapeError&) {
        shape = true;
    }
    EXPECT(shape);
}

// ------------------------------------------------------------------------------------ GPU layer step
struct Cfg {
    int64_t h = 0, hq = 0, hkv = 0, d = 0, I = 0, V = 0, N = 0;
};
struct Inputs {
    Cfg c;
    std::vector<float> x, g1, wqkvT, woT, g2, wg, wu, wd, g3, wlm;
    std::vector<int64_t> labels, pos;
};

static Inputs read_inputs(const char* path) {
    std::ifstream f(path, std::ios::binary);
    Inputs in;
    int64_t hdr[8];
    f.read((char*)hdr, sizeof(hdr));
    in.c = {hdr[0], hdr[1], hdr[2], hdr[3], hdr[4], hdr[5], hdr[6]};
    const bool packed = hdr[7] != 0;
    const Cfg& c = in.c;
    auto rd = [&](std::vector<float>& v, int64_t n) {
        v.resize((size_t)n);
        f.read((char*)v.data(), n * 4);
    };
    rd(in.x, c.N * c.h);
    rd(in.g1, c.h);
    rd(in.wqkvT, c.h * (c.hq + 2 * c.hkv) * c.d);
    rd(in.woT, c.hq * c.d * c.h);
    rd(in.g2, c.h);
    rd(in.wg, c.I * c.h);
    rd(in.wu, c.I * c.h);
    rd(in.wd, c.h * c.I);
    rd(in.g3, c.h);
    rd(in.wlm, c.V * c.h);
    in.labels.resize((size_t)c.N);
    f.read((char*)in.labels.data(), c.N * 8);
    if (packed) {
        in.pos.resize((size_t)c.N);
        f.read((char*)in.pos.data(), c.N * 8);
    }
    if (!f) throw std::runtime_error(std::string("short input file ") + path);
    return in;
}

static Tensor leaf(const std::vector<float>& v, std::vector<int64_t> shape, bool grad, int64_t off = 0) {
    Tensor t = Tensor::zeros(std::move(shape), {Dtype::kF64, grad});
    for (int64_t i = 0; i < t.numel(); ++i) t.set((size_t)i, v[(size_t)(off + i)]);
    return t;
}

struct Params {
    Tensor g1, wqkvT, woT, g2, wg, wu, wd, g3, wlm;
};

static Params make_params(const Inputs& in) {
    const Cfg& c = in.c;
    const int64_t qo = (c.hq + 2 * c.hkv) * c.d;
    return {leaf(in.g1, {c.h}, true),         leaf(in.wqkvT, {c.h, qo}, true), leaf(in.woT, {c.hq * c.d, c.h}, true),
            leaf(in.g2, {c.h}, true),         leaf(in.wg, {c.I, c.h}, true),   leaf(in.wu, {c.I, c.h}, true),
            leaf(in.wd, {c.h, c.I}, true),    leaf(in.g3, {c.h}, true),        leaf(in.wlm, {c.V, c.h}, true)};
}

// One rank's step: x [s_loc, h] (leaf) -> decoder layer -> final norm -> tiled logits/loss; returns loss_sum.
static std::pair<Tensor, int64_t> rank_step(gpu::Group& g, const Cfg& c, const Params& p, const Tensor& x,
                                            const std::vector<int64_t>& labels, const std::vector<int64_t>* pos,
                                            bool ckpt) {
    const int dev = g.device();
    auto layer = [&](const Tensor& xin) {
        Tensor xn1 = gpu::rmsnorm(xin, p.g1, 1e-5, dev);
        Tensor qkv = gpu::matmul(xn1, p.wqkvT, dev);
        Tensor attn = gpu::ulysses_attention(g, qkv, (int)c.hq, (int)c.hkv, (int)c.d, pos);
        Tensor x1 = gpu::add(xin, gpu::matmul(attn, p.woT, dev));
        Tensor xn2 = gpu::rmsnorm(x1, p.g2, 1e-5, dev);
        return gpu::add(x1, gpu::tiled_mlp(xn2, p.wg, p.wu, p.wd, 0, dev));
    };
    Tensor x2 = ckpt ? checkpoint(layer, x) : layer(x);
    Tensor z = gpu::rmsnorm(x2, p.g3, 1e-5, dev);
    return gpu::tiled_logits_loss(z, p.wlm, labels, 0, dev);
}

static void write_out(const char* path, const std::vector<std::pair<std::string, std::vector<double>>>& recs,
                      const std::string& ledger_json) {
    std::ofstream f(path, std::ios::binary);
    for (auto& r : recs) {
        const int64_t nl = (int64_t)r.first.size(), n = (int64_t)r.second.size();
        f.write((const char*)&nl, 8);
        f.write(r.first.data(), nl);
        f.write((const char*)&n, 8);
        f.write((const char*)r.second.data(), n * 8);
    }
    std::ofstream(std::string(path) + ".ledger.json") << ledger_json;
}

static void gpu_step(int P, const char* in_path, const char* out_path, bool ckpt) {
    // one MemoryLedger per rank thread, declared first: it must outlive every buffer registered in it (the
    // replicated weights' grads are created lazily inside the rank threads)
    std::vector<std::unique_ptr<MemoryLedger>> leds;
    for (int r = 0; r < P; ++r) leds.push_back(std::make_unique<MemoryLedger>());
    const Inputs in = read_inputs(in_path);
    const Cfg& c = in.c;
    const int64_t s_loc = c.N / P;
    int64_t total_count = 0;
    for (int64_t l : in.labels) total_count += l != -100;
    auto groups = gpu::Group::in_process(P, {0});
    std::vector<Params> params;
    for (int r = 0; r < P; ++r) params.push_back(make_params(in));  // weights replicated on every rank
    std::vector<Tensor> xs(P);
    std::vector<double> loss_sum(P);
    std::vector<int64_t> counts(P);
    std::vector<std::string> ledgers(P), errs(P);
    std::vector<std::thread> th;
    for (int r = 0; r < P; ++r)
        th.emplace_back([&, r] {
            try {
                MemoryLedger& led = *leds[r];
                LedgerScope scope(led);
                xs[r] = leaf(in.x, {s_loc, c.h}, true, r * s_loc * c.h);
                std::vector<int64_t> lab(in.labels.begin() + r * s_loc, in.labels.begin() + (r + 1) * s_loc);
                auto [ls, cnt] = rank_step(*groups[r], c, params[r], xs[r], lab, in.pos.empty() ? nullptr : &in.pos, ckpt);
                loss_sum[r] = ls.item();
                counts[r] = cnt;
                // global mean loss: d loss / d loss_sum = 1 / global count
                Tensor loss = gpu::scale(ls, 1.0 / (double)total_count);
                backward(loss);
                ledgers[r] = led.summary_json();
            } catch (const std::exception& e) {
                errs[r] = e.what();
            }
        });
    for (auto& t : th) t.join();
    for (int r = 0; r < P; ++r)
        if (!errs[r].empty()) throw std::runtime_error("rank " + std::to_string(r) + ": " + errs[r]);
    double ls = 0;
    int64_t cnt = 0;
    for (int r = 0; r < P; ++r) {  // all_reduce_sum of (loss_sum, count), rank order
        ls += loss_sum[r];
        cnt += counts[r];
    }
    EXPECT(cnt == total_count);
    std::vector<std::pair<std::string, std::vector<double>>> recs;
    recs.push_back({"loss", {ls / (double)cnt}});
    recs.push_back({"count", {(double)cnt}});
    const char* names[] = {"g1", "wqkvT", "woT", "g2", "wg", "wu", "wd", "g3", "wlm"};
    for (int k = 0; k < 9; ++k) {  // SP-group weight-grad all-reduce, rank-ascending
        std::vector<double> acc;
        for (int r = 0; r < P; ++r) {
            const Params& p = params[r];
            const Tensor* t[] = {&p.g1, &p.wqkvT, &p.woT, &p.g2, &p.wg, &p.wu, &p.wd, &p.g3, &p.wlm};
            const auto g = t[k]->grad_vector();
            if (acc.empty()) acc = g;
            else
                for (size_t i = 0; i < g.size(); ++i) acc[i] += g[i];
        }
        recs.push_back({names[k], acc});
    }
    std::vector<double> dx;
    for (int r = 0; r < P; ++r) {
        const auto g = xs[r].grad_vector();
        dx.insert(dx.end(), g.begin(), g.end());
    }
    recs.push_back({"dx", dx});
    write_out(out_path, recs, ledgers[0]);
    std::printf("rank-0 comm stats: %s\n", groups[0]->stats_json().c_str());
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "--cpu";
    try {
        if (mode == "--cpu") {
            cpu_tests();
        } else if (mode == "--gpu" && argc >= 4) {
            gpu_step(1, argv[2], argv[3], argc >= 5 && std::string(argv[4]) == "ckpt");
        } else if (mode == "--gpu-sp" && argc >= 5) {
            gpu_step(std::atoi(argv[2]), argv[3], argv[4], argc >= 6 && std::string(argv[5]) == "ckpt");
        } else {
            std::printf("usage: %s --cpu | --gpu IN OUT [ckpt] | --gpu-sp P IN OUT [ckpt]\n", argv[0]);
            return 2;
        }
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 1;
    }
    std::printf("%s\n", fails ? "FAILED" : "ok");
    return fails ? 1 : 0;
}
