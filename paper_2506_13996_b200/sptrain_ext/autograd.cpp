// The reference's backward engine, recompute-on-backward checkpointing and finite-difference oracle:
// /root/reference/proj/include/sptrain/autograd.hpp declares them (autograd.hpp:14-37) but the reference ships no
// definition ("autograd.hpp is unresolved at link time").  This file defines them over the
// reference's own Tensor / TensorNode / ledger (tensor.hpp, ledger.hpp), so a program written against the
// reference API links and runs, with the GPU ops of sptrain/gpu.hpp as graph nodes.
//
// Semantics (SPEC.md:26-121 core_autograd):
//   * backward(root, seed): nodes reachable from root are visited in exact reverse creation order (a reverse
//     topological order: an op is always created after its inputs, tensor.cpp next_seq); each non-leaf node's
//     backward_fn reads self.grad and accumulates into its inputs (tensor.hpp:86-91).  Gradient accumulation
//     into leaves is additive across calls.  Intermediate grads are released once consumed.
//   * checkpoint(region, x, mode): forward runs the region without recording and keeps only x (on the host
//     tier while parked with kOffload, autograd.hpp:20-24); backward replays the region on an alias of x,
//     checks the replay is bit-identical to the recorded output (DeterminismError otherwise, errors.hpp:36-40,
//     SPEC.md:82-83), differentiates through the replayed subgraph and reclaims the output's storage.
//   * finite_diff_grad(f, x, eps): central differences.
#include <sptrain/autograd.hpp>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <unordered_set>
#include <vector>

namespace sptrain {

namespace {

void collect(const NodePtr& root, std::vector<TensorNode*>& out) {
    std::unordered_set<TensorNode*> seen;
    std::vector<TensorNode*> stack{root.get()};
    while (!stack.empty()) {
        TensorNode* n = stack.back();
        stack.pop_back();
        if (!n || !seen.insert(n).second) continue;
        out.push_back(n);
        for (const NodePtr& in : n->inputs)
            if (in && in->requires_grad) stack.push_back(in.get());
    }
    std::sort(out.begin(), out.end(), [](TensorNode* a, TensorNode* b) { return a->seq > b->seq; });
}

bool same_bits(const DataBuffer& a, const DataBuffer& b) {
    if (a.dtype() != b.dtype() || a.size() != b.size()) return false;
    if (a.dtype() == Dtype::kF64)
        return std::memcmp(a.f64().data(), b.f64().data(), a.size() * sizeof(double)) == 0;
    return std::memcmp(a.f32().data(), b.f32().data(), a.size() * sizeof(float)) == 0;
}

}  // namespace

void backward(const Tensor& root, std::span<const double> seed) {
    if (!root.defined()) throw ValidationError("backward of an undefined tensor");
    if (!root.requires_grad()) throw ValidationError("backward of a tensor that does not require grad");
    if (static_cast<int64_t>(seed.size()) != root.numel())
        throw ShapeError("backward seed has " + std::to_string(seed.size()) + " values for a tensor of " +
                         std::to_string(root.numel()));
    std::vector<TensorNode*> order;
    collect(root.node(), order);
    root.node()->accumulate_grad(seed);
    for (TensorNode* n : order) {
        if (n->is_leaf || !n->grad || !n->backward_fn) continue;
        n->backward_fn(*n);
        if (n != root.node().get()) n->grad.reset();  // consumed: an intermediate grad is never read again
    }
}

void backward(const Tensor& root) {
    if (root.defined() && root.numel() != 1)
        throw ShapeError("backward(root) needs a scalar root; got " + detail::shape_str(root.shape()));
    const double one = 1.0;
    backward(root, std::span<const double>(&one, 1));
}

Tensor checkpoint(const RegionFn& region, const Tensor& x, CheckpointMode mode) {
    Tensor recorded;
    {
        NoGradGuard no_grad;  // forward without recording: only x survives
        recorded = region(x);
    }
    NodePtr xin = x.node();
    auto node = std::make_shared<TensorNode>();
    node->shape = recorded.shape();
    node->numel = recorded.numel();
    node->dtype = recorded.dtype();
    node->tag = recorded.node()->tag;
    node->value = recorded.node()->value;  // the region's output storage, no copy
    node->op_name = "checkpoint";
    node->seq = detail::next_seq();
    if (!(grad_enabled() && xin->requires_grad)) return Tensor(node);
    node->requires_grad = true;
    node->is_leaf = false;
    node->inputs = {xin};
    if (mode == CheckpointMode::kOffload) xin->value->move_tier(Tier::kHost);  // parked until backward
    node->backward_fn = [region, xin, mode](TensorNode& self) {
        if (mode == CheckpointMode::kOffload) xin->value->move_tier(Tier::kDevice);
        Tensor xa = Tensor::alias_leaf(Tensor(xin), true);
        Tensor replay = region(xa);
        if (!same_bits(*replay.node()->value, *self.value))
            throw DeterminismError(std::string("checkpoint replay of region (output ") +
                                   detail::shape_str(self.shape) + ") is not bit-identical to its recorded forward");
        if (replay.requires_grad()) {
            std::vector<double> g(static_cast<std::size_t>(self.numel));
            for (std::size_t i = 0; i < g.size(); ++i) g[i] = self.grad->get(i);
            backward(replay, g);
        }
        if (xa.has_grad()) {
            const std::vector<double> gx = xa.grad_vector();
            xin->accumulate_grad(gx);
        }
        self.value->release_storage();  // autograd.hpp:29-30: the output's storage is reclaimed in backward
    };
    return Tensor(node);
}

Tensor finite_diff_grad(const std::function<double(const Tensor&)>& f, const Tensor& x, double eps) {
    NoGradGuard no_grad;
    Tensor g = Tensor::zeros(x.shape(), TensorOpts{Dtype::kF64, false});
    Tensor xp = Tensor::zeros(x.shape(), TensorOpts{x.dtype(), false});
    for (int64_t i = 0; i < x.numel(); ++i) xp.set(static_cast<std::size_t>(i), x.at(static_cast<std::size_t>(i)));
    for (int64_t i = 0; i < x.numel(); ++i) {
        const std::size_t k = static_cast<std::size_t>(i);
        const double x0 = x.at(k);
        xp.set(k, x0 + eps);
        const double fp = f(xp);
        xp.set(k, x0 - eps);
        const double fm = f(xp);
        xp.set(k, x0);
        g.set(k, (fp - fm) / (2.0 * eps));
    }
    return g;
}

}  // namespace sptrain
