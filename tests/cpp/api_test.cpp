// C++ host-API test (include/sptrain/b200.hpp over the C-ABI).  `--cpu`: host logic against the SPEC/PAPER
// golden vectors and the errors.hpp exception mapping; `--gpu`: a tiny layer step through UlyssesLayerStep
// (SP=1 vs SP=2 loopback, determinism, checkpointed 2-layer stack with offload).  Exit code 0 = pass.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "sptrain/b200.hpp"

namespace sb = sptrain::b200;

static int fails = 0;
#define EXPECT(c)                                                        \
    do {                                                                 \
        if (!(c)) {                                                      \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
            ++fails;                                                     \
        }                                                                \
    } while (0)

static void cpu_tests() {
    // head plans
    auto p = sb::plan_head_shards(32, 8, 8);
    EXPECT(p.q_heads_per_rank == 4 && p.kv_heads_per_rank == 1 && p.kv_replication == 1);
    p = sb::plan_head_shards(32, 8, 32);
    EXPECT(p.q_heads_per_rank == 1 && p.kv_heads_per_rank == 1 && p.kv_replication == 4);
    p = sb::plan_head_shards(32, 4, 8);
    EXPECT(p.q_heads_per_rank == 4 && p.kv_heads_per_rank == 1 && p.kv_replication == 2);
    p = sb::plan_head_shards(8, 2, 1);
    EXPECT(p.q_heads_per_rank == 8 && p.kv_heads_per_rank == 2 && p.kv_replication == 1);
    EXPECT((sb::heads_of(sb::plan_head_shards(32, 4, 8), 3, 1) == std::vector<int>{1}));
    bool thrown = false;
    try {
        sb::plan_head_shards(9, 1, 8);  // "q_heads not divisible by SP degree"
    } catch (const sptrain::ValidationError& e) {
        thrown = std::string(e.what()).find("divisible") != std::string::npos;
    }
    EXPECT(thrown);
    // pre-shift + shard: [1..8] -> [2..8,-100], shards [2,3,4,5] [6,7,8,-100]
    std::vector<int64_t> lab = {1, 2, 3, 4, 5, 6, 7, 8};
    auto sh = sb::preshift_labels(lab);
    EXPECT((sh == std::vector<int64_t>{2, 3, 4, 5, 6, 7, 8, -100}));
    sb::Batch b{lab, {0, 1, 2, 3, 4, 5, 6, 7}, sh};
    EXPECT((sb::shard_sequence(b, 2, 0).shift_labels == std::vector<int64_t>{2, 3, 4, 5}));
    EXPECT((sb::shard_sequence(b, 2, 1).shift_labels == std::vector<int64_t>{6, 7, 8, -100}));
    // pad s=7, P=4 -> 8 with one -100
    sb::Batch b7{{1, 2, 3, 4, 5, 6, 7}, {0, 1, 2, 3, 4, 5, 6}, sb::preshift_labels({1, 2, 3, 4, 5, 6, 7})};
    auto pb = sb::pad_to_multiple(b7, 4);
    EXPECT(pb.input_ids.size() == 8 && pb.shift_labels[7] == -100 && pb.shift_labels[6] == -100);
    // block-causal packed [0,1,0,1]: position 2 sees {2}, position 3 sees {2,3}
    EXPECT((sb::block_causal_starts({0, 1, 0, 1}) == std::vector<int64_t>{0, 0, 2, 2}));
    // exception taxonomy (errors.hpp): ShapeError is-a ValidationError
    bool shape_is_validation = false;
    try {
        sb::check(SPT_ERR_SHAPE);
    } catch (const sptrain::ValidationError&) {
        shape_is_validation = true;
    }
    EXPECT(shape_is_validation);
#ifdef SPTRAIN_B200_REFERENCE_ERRORS
    std::printf("errors: reference sptrain/errors.hpp\n");
#else
    std::printf("errors: b200.hpp declarations\n");
#endif
}

static uint16_t bf16(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFF + ((u >> 16) & 1);
    return (uint16_t)(u >> 16);
}

static void gpu_tests() {
    const sb::ModelShape m{256, 8, 2, 32, 1024, 2048};
    const int64_t N = 512;
    std::mt19937 rng(7);
    std::normal_distribution<float> nd(0.f, 1.f);
    auto mk = [&](size_t n, float sd, float mean) {
        std::vector<uint16_t> v(n);
        for (auto& x : v) x = bf16(mean + sd * nd(rng));
        return v;
    };
    const int64_t qkv = (int64_t)(m.q_heads + 2 * m.kv_heads) * m.head_dim, qd = (int64_t)m.q_heads * m.head_dim;
    struct W {
        std::string n;
        std::vector<uint16_t> v;
    };
    std::vector<W> ws = {{"g1", mk(m.hidden, 0.05f, 1.f)},
                         {"wqkv", mk(qkv * m.hidden, 0.02f, 0.f)},
                         {"wo", mk(m.hidden * qd, 0.02f, 0.f)},
                         {"g2", mk(m.hidden, 0.05f, 1.f)},
                         {"wg", mk((size_t)m.intermediate * m.hidden, 0.02f, 0.f)},
                         {"wu", mk((size_t)m.intermediate * m.hidden, 0.02f, 0.f)},
                         {"wd", mk((size_t)m.hidden * m.intermediate, 0.02f, 0.f)},
                         {"g3", mk(m.hidden, 0.05f, 1.f)},
                         {"wlm", mk((size_t)m.vocab * m.hidden, 0.02f, 0.f)}};
    auto x = mk((size_t)N * m.hidden, 1.f, 0.f);
    std::vector<int64_t> lab(N);
    for (int64_t i = 0; i < N; ++i) lab[i] = (i * 7919) % m.vocab;
    lab = sb::preshift_labels(lab);
    float loss1 = 0.f, loss2 = 0.f;
    int64_t cnt = 0;
    for (int P : {1, 2}) {
        auto grp = sb::ProcessGroup::loopback(P);
        sb::UlyssesLayerStep eng(m, N, grp);
        for (auto& w : ws) eng.set_param(w.n, w.v.data(), (int64_t)w.v.size(), true);  // size-checked form
        if (P == 1) {  // a W_o of the wrong element count is a ShapeError, not an out-of-bounds read
            bool threw = false;
            try {
                eng.set_param("wo", ws[2].v.data(), (int64_t)ws[2].v.size() - 1, true);
            } catch (const sptrain::ShapeError&) {
                threw = true;
            }
            EXPECT(threw);
            EXPECT(eng.param_numel("wlm") == (int64_t)m.vocab * m.hidden);
        }
        auto a = eng.step(x.data(), lab.data());
        auto b = eng.step(x.data(), lab.data());
        EXPECT(std::isfinite(a.first) && a.first == b.first);  // deterministic
        EXPECT(a.second == N - 1);
        (P == 1 ? loss1 : loss2) = a.first;
        cnt = a.second;
        auto g = eng.grad("wo", (size_t)m.hidden * qd);
        double nrm = 0;
        for (float v : g) nrm += (double)v * v;
        EXPECT(nrm > 0 && std::isfinite(nrm));
    }
    EXPECT(std::fabs(loss1 - loss2) <= 1e-3f * std::fabs(loss1));  // SP=2 == SP=1
    {  // 2-layer stack, checkpoints offloaded to pinned host memory
        auto grp = sb::ProcessGroup::loopback(2);
        sb::StepOptions o;
        o.n_layers = 2;
        o.ckpt_offload = true;
        sb::UlyssesLayerStep eng(m, N, grp, o);
        for (int l = 0; l < 2; ++l)
            for (auto& w : ws)
                if (w.n != "g3" && w.n != "wlm") eng.set_param("layers." + std::to_string(l) + "." + w.n, w.v.data());
        eng.set_param("g3", ws[7].v.data());
        eng.set_param("wlm", ws[8].v.data());
        auto a = eng.step(x.data(), lab.data());
        EXPECT(std::isfinite(a.first) && a.second == cnt);
        EXPECT(eng.memory_json().find("\"ckpt_offload\":true") != std::string::npos);
    }
    std::printf("gpu: loss SP1 %.6f SP2 %.6f\n", loss1, loss2);
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::string(argv[1]) == "--gpu";
    try {
        cpu_tests();
        if (gpu) gpu_tests();
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 2;
    }
    std::printf(fails ? "FAILED (%d)\n" : "ok\n", fails);
    return fails ? 1 : 0;
}
