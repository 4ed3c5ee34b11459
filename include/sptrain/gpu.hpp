// sptrain::gpu — the B200 hot path as operations on the reference's own Tensor type.
//
// For a program written against the reference C++ API (/root/reference/proj/include/sptrain/{tensor,ledger,
// autograd,errors}.hpp): every function below builds an ordinary graph node with detail::make_op
// (tensor.hpp:152-157), so sptrain::backward / sptrain::checkpoint (autograd.hpp:14-32; defined in
// paper_2506_13996_b200/sptrain_ext/autograd.cpp) differentiate through it, and its backward_fn calls the
// C-ABI *_bwd kernels.  Values cross the boundary as the reference's host Tensors (f64 / f32, tensor.hpp:22):
// inputs are rounded to bf16 on upload (the GPU path's storage type), outputs and gradients come back fp32-
// accumulated and widened.  Device memory an op keeps for its backward (the saved activations of the inner
// attention, the fused logits/loss gradients) is registered with the caller's ambient MemoryLedger on
// Tier::kDevice (LedgerScope, ledger.hpp:120-152) under the op's MemTag, so summary_json reports real HBM.
//
// Threading follows the reference (ledger.cpp thread_local scopes): one SP rank per host thread,
// each with its own Group.  Group::in_process(P) creates the P peer-transport groups of one process (ranks
// share one or several GPUs; the seq_to_head / head_to_seq kernels store into / load from the other ranks'
// buffers directly).
//
// Shape limits of the kernels behind these ops are reported as ShapeError: matmul needs n % 64 == 0 and
// k % 8 == 0 (backward also m % 8 == 0, k % 64 == 0); attention needs head_dim in {32, 64, 128} and the
// global sequence a multiple of 128; hidden sizes % 64 == 0; intermediate % 32 == 0; vocab % 64 == 0.
#pragma once

#include <sptrain/autograd.hpp>
#include <sptrain/tensor.hpp>

#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

#include "../sptrain_b200.h"

namespace sptrain::gpu {

// One SP rank's process group handle (peer transport, or loopback for P = 1 / the single-thread case).
class Group {
public:
    // P groups for P threads of this process (rank r uses groups[r] on `devices[r % devices.size()]`).
    static std::vector<std::shared_ptr<Group>> in_process(int nranks, std::vector<int> devices = {0});
    // A single-rank group on `device` (SP = 1).
    static std::shared_ptr<Group> single(int device = 0);
    ~Group();
    int rank() const { return rank_; }
    int size() const { return size_; }
    int device() const { return device_; }
    spt_comm* handle() const { return comm_; }
    std::string stats_json() const;

private:
    Group() = default;
    spt_comm* comm_ = nullptr;
    int rank_ = 0, size_ = 1, device_ = 0;
    std::shared_ptr<void> bootstrap_;
    friend struct GroupAccess;
};

// SPEC.md:49-57 matmul(a [m,k], b [k,n]) -> [m,n] on tcgen05 (bf16 operands, fp32 accumulate).
Tensor matmul(const Tensor& a, const Tensor& b, int device = 0);
// SPEC.md:259 RMSNorm over the last dim: y = x * rsqrt(mean(x^2) + eps) * g; x [n, h], g [h].
Tensor rmsnorm(const Tensor& x, const Tensor& g, double eps = 1e-5, int device = 0);
// SPEC.md:395-403 tiled_mlp: y = W_d (silu(W_g x) * W_u x), x [s, h], wg / wu [I, h], wd [h, I]; num_tiles 0 ->
// ceil(s / h).  Per-tile recompute in the backward, parameter grads summed in ascending tile order.
Tensor tiled_mlp(const Tensor& x, const Tensor& wg, const Tensor& wu, const Tensor& wd, int num_tiles = 0,
                 int device = 0);
// SPEC.md:405-413 tiled_logits_loss: (loss_sum as a scalar Tensor, valid_count) of cross_entropy(hidden W_lm^T,
// shift_labels) with -100 ignored; no [s, V] logits ever live (tiles of tile_len tokens; 0 -> auto).  Labels
// outside [0, V) U {-100} -> ValidationError.
std::pair<Tensor, int64_t> tiled_logits_loss(const Tensor& hidden, const Tensor& w_lm,
                                             const std::vector<int64_t>& shift_labels, int64_t tile_len = 0,
                                             int device = 0);
// SPEC.md:333-341 ulysses_attention for this rank: qkv [s_loc, (Hq + 2 Hkv) * d] (this rank's sequence shard of
// the fused projection: q heads, k heads, v heads) -> [s_loc, Hq * d].  seq_to_head (with kv replication when
// Hkv < P) -> causal GQA attention over the full sequence (block-causal from position_ids_full when given,
// SPEC.md:243-251) -> head_to_seq.  Every rank of `group` calls it at the same program point.
Tensor ulysses_attention(Group& group, const Tensor& qkv, int q_heads, int kv_heads, int head_dim,
                         const std::vector<int64_t>* position_ids_full = nullptr);

// Small host-side glue ops with the SPEC's conventions (for composing a layer in tests / drivers).
Tensor add(const Tensor& a, const Tensor& b);
Tensor scale(const Tensor& a, double c);

}  // namespace sptrain::gpu
