#pragma once

#include <cstdint>
#include <vector>

#include "../../include/sptrain_b200.h"

namespace spt {

spt_head_shard_plan plan_head_shards(int hq, int hkv, int p);
std::vector<int> heads_of(const spt_head_shard_plan& pl, int rank, int kind);
std::vector<int32_t> qkv_pack_map(const spt_head_shard_plan& pl);
std::vector<int32_t> q_pack_map(const spt_head_shard_plan& pl);
std::vector<int32_t> o_gather_map(const spt_head_shard_plan& pl, int* max_src);
std::vector<int32_t> qkv_gather_map(const spt_head_shard_plan& pl, int* max_src);

}  // namespace spt
