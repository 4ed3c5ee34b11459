// Host-only logic of the path (no GPU): head-shard plans, label pre-shift / padding, block-causal
// run validation and the all-to-all schedule.  These mirror SPEC.md operations one-to-one.
#include <string>
#include <vector>

#include "common.h"
#include "plan.h"

namespace spt {

// SPEC.md:296-305 (rules: PAPER.md:326-358; limits: PAPER.md:946-957)
spt_head_shard_plan plan_head_shards(int hq, int hkv, int p) {
    SPT_CHECK(hq >= 1 && hkv >= 1 && p >= 1, SPT_ERR_VALIDATION, "head counts and SP degree must be >= 1");
    SPT_CHECK(hq % hkv == 0, SPT_ERR_VALIDATION,
              "q_heads (" + std::to_string(hq) + ") not divisible by kv_heads (" + std::to_string(hkv) + ")");
    if (hq % p != 0) {
        std::string ok;
        for (int d = 1; d <= hq; ++d)
            if (hq % d == 0) ok += (ok.empty() ? "" : ", ") + std::to_string(d);
        SPT_THROW(SPT_ERR_VALIDATION, "q_heads not divisible by SP degree: q_heads=" + std::to_string(hq) +
                                          ", sp=" + std::to_string(p) + "; you'd need SP to be one of [" + ok + "]");
    }
    spt_head_shard_plan pl{p, hq, hkv, hq / p, 0, 1};
    if (hkv >= p) {
        SPT_CHECK(hkv % p == 0, SPT_ERR_VALIDATION,
                  "kv_heads (" + std::to_string(hkv) + ") >= SP (" + std::to_string(p) + ") but not divisible by it");
        pl.kv_heads_per_rank = hkv / p;
    } else {
        SPT_CHECK(p % hkv == 0, SPT_ERR_VALIDATION,
                  "SP (" + std::to_string(p) + ") not a multiple of kv_heads (" + std::to_string(hkv) + ")");
        pl.kv_heads_per_rank = 1;
        pl.kv_replication = p / hkv;
    }
    return pl;
}

std::vector<int> heads_of(const spt_head_shard_plan& pl, int rank, int kind) {
    std::vector<int> out;
    if (kind == 0) {
        for (int a = 0; a < pl.q_heads_per_rank; ++a) out.push_back(rank * pl.q_heads_per_rank + a);
    } else if (pl.kv_replication > 1) {
        out.push_back(rank / pl.kv_replication);  // r > 1 -> head floor(rank / r)
    } else {
        for (int a = 0; a < pl.kv_heads_per_rank; ++a) out.push_back(rank * pl.kv_heads_per_rank + a);
    }
    return out;
}

// Fused-QKV pack table: for destination j, slots [q heads | k heads | v heads] of the local payload,
// as indices into the source token row [Hq | Hkv | Hkv] heads.
std::vector<int32_t> qkv_pack_map(const spt_head_shard_plan& pl) {
    std::vector<int32_t> m;
    for (int j = 0; j < pl.sp_degree; ++j) {
        for (int h : heads_of(pl, j, 0)) m.push_back(h);
        for (int h : heads_of(pl, j, 1)) m.push_back(pl.q_heads + h);
        for (int h : heads_of(pl, j, 1)) m.push_back(pl.q_heads + pl.kv_heads + h);
    }
    return m;
}

std::vector<int32_t> q_pack_map(const spt_head_shard_plan& pl) {
    std::vector<int32_t> m;
    for (int j = 0; j < pl.sp_degree; ++j)
        for (int h : heads_of(pl, j, 0)) m.push_back(h);
    return m;
}

// Unpack gather table for head_to_seq of a payload whose per-rank slots are `slots(j)`:
// out head h <- list of (rank j * heads_in + slot a) with slots(j)[a] == h, in rank order.
static std::vector<int32_t> gather_table(const spt_head_shard_plan& pl, int heads_out, int heads_in,
                                         const std::vector<std::vector<int>>& slots, int* max_src) {
    std::vector<std::vector<int32_t>> lists(heads_out);
    for (int j = 0; j < pl.sp_degree; ++j)
        for (int a = 0; a < (int)slots[j].size(); ++a) lists[slots[j][a]].push_back(j * heads_in + a);
    int ms = 1;
    for (auto& l : lists) {
        SPT_CHECK(!l.empty(), SPT_ERR_INTERNAL, "head_to_seq: head without a source");
        ms = std::max<int>(ms, (int)l.size());
    }
    std::vector<int32_t> t((size_t)heads_out * ms, -1);
    for (int h = 0; h < heads_out; ++h)
        for (size_t e = 0; e < lists[h].size(); ++e) t[(size_t)h * ms + e] = lists[h][e];
    *max_src = ms;
    return t;
}

std::vector<int32_t> o_gather_map(const spt_head_shard_plan& pl, int* max_src) {
    std::vector<std::vector<int>> slots;
    for (int j = 0; j < pl.sp_degree; ++j) slots.push_back(heads_of(pl, j, 0));
    return gather_table(pl, pl.q_heads, pl.q_heads_per_rank, slots, max_src);
}

std::vector<int32_t> qkv_gather_map(const spt_head_shard_plan& pl, int* max_src) {
    std::vector<std::vector<int>> slots;
    for (int j = 0; j < pl.sp_degree; ++j) {
        std::vector<int> s = heads_of(pl, j, 0);
        for (int h : heads_of(pl, j, 1)) s.push_back(pl.q_heads + h);
        for (int h : heads_of(pl, j, 1)) s.push_back(pl.q_heads + pl.kv_heads + h);
        slots.push_back(s);
    }
    const int heads_in = pl.q_heads_per_rank + 2 * pl.kv_heads_per_rank;
    return gather_table(pl, pl.q_heads + 2 * pl.kv_heads, heads_in, slots, max_src);
}

}  // namespace spt

using namespace spt;

extern "C" spt_status spt_plan_head_shards(int32_t q_heads, int32_t kv_heads, int32_t sp_degree,
                                           spt_head_shard_plan* out) {
    return capi_guard([&] {
        SPT_CHECK(out != nullptr, SPT_ERR_VALIDATION, "null output");
        *out = plan_head_shards(q_heads, kv_heads, sp_degree);
    });
}

extern "C" spt_status spt_plan_heads_of(const spt_head_shard_plan* plan, int32_t rank, int32_t kind,
                                        int32_t* out_heads, int32_t capacity, int32_t* n_out) {
    return capi_guard([&] {
        SPT_CHECK(plan && rank >= 0 && rank < plan->sp_degree, SPT_ERR_VALIDATION, "bad plan/rank");
        auto v = heads_of(*plan, rank, kind);
        SPT_CHECK((int)v.size() <= capacity, SPT_ERR_SHAPE, "capacity too small");
        for (size_t i = 0; i < v.size(); ++i) out_heads[i] = v[i];
        *n_out = (int32_t)v.size();
    });
}

// SPEC.md:512-519
extern "C" spt_status spt_preshift_labels(const int64_t* labels, int64_t s, int64_t* out) {
    return capi_guard([&] {
        SPT_CHECK(s >= 0, SPT_ERR_SHAPE, "negative length");
        if (s == 0) return;
        for (int64_t i = 0; i + 1 < s; ++i) out[i] = labels[i + 1];
        out[s - 1] = -100;
    });
}

// SPEC.md:531-535, :553
extern "C" spt_status spt_pad_to_multiple(int64_t* input_ids, int64_t* position_ids, int64_t* shift_labels, int64_t s,
                                          int32_t sp_degree, int64_t cap, int64_t* padded_len) {
    return capi_guard([&] {
        SPT_CHECK(sp_degree >= 1 && s >= 0, SPT_ERR_VALIDATION, "bad arguments");
        const int64_t pad = (sp_degree - s % sp_degree) % sp_degree;
        *padded_len = s + pad;
        if (cap < s + pad) return;
        for (int64_t i = 0; i < pad; ++i) {
            if (input_ids) input_ids[s + i] = 0;
            if (position_ids) position_ids[s + i] = i;  // isolated run starting at 0
            if (shift_labels) shift_labels[s + i] = -100;
        }
    });
}

// SPEC.md:243-251
extern "C" spt_status spt_block_causal_starts(const int64_t* position_ids, int64_t s, int64_t* starts_out) {
    return capi_guard([&] {
        for (int64_t t = 0; t < s; ++t) {
            const int64_t p = position_ids[t];
            const bool ok = t == 0 ? p == 0 : (p == 0 || p == position_ids[t - 1] + 1);
            SPT_CHECK(ok, SPT_ERR_VALIDATION, "position_ids not zero-based ascending runs at index " + std::to_string(t));
            starts_out[t] = t - p;
        }
    });
}

// All-to-all element counts per peer (actual GQA payloads per SURVEY App. B #2)
extern "C" spt_status spt_a2a_counts(const spt_head_shard_plan* plan, int64_t s_loc, int32_t head_dim,
                                     int32_t direction, int64_t* send_counts, int64_t* recv_counts) {
    return capi_guard([&] {
        SPT_CHECK(plan != nullptr, SPT_ERR_VALIDATION, "null plan");
        const int64_t qkv_loc = plan->q_heads_per_rank + 2 * plan->kv_heads_per_rank;
        const int64_t q_loc = plan->q_heads_per_rank;
        const int64_t per = (direction == 0 || direction == 3) ? qkv_loc : q_loc;
        SPT_CHECK(direction >= 0 && direction <= 3, SPT_ERR_VALIDATION, "direction in [0,3]");
        for (int j = 0; j < plan->sp_degree; ++j) {
            send_counts[j] = s_loc * per * head_dim;
            recv_counts[j] = s_loc * per * head_dim;
        }
    });
}
