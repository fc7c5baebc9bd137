// autograd.cpp — the tape and the backward engine.
//
// PAPER.md:158-159 (§4.3): the graph is rebuilt on every run by operator
// overloading; reverse mode computes the gradient of a scalar output.
// version counters detect saved tensors mutated before
// backward (checked at unpack time) — a user error, no copies.
// PAPER.md:177 (§5.1): the evaluator runs entirely in C++ (no GIL).
//
// Engine: dependency counts over the reachable
// graph; ready nodes issued in reverse creation order (max sequence number
// first — a valid reverse-topological order that emits each layer's weight
// gradient as early as possible, which is what lets DDP buckets fire while
// the rest of backward runs); pending input-gradients are summed in place
// (fan-out), leaf gradients accumulate with +=; saved tensors and pending
// buffers are released the moment their node has run, so their blocks go
// back to the stream pool immediately.
#include <algorithm>
#include <map>
#include <queue>
#include <unordered_map>
#include <unordered_set>

#include "kernels.h"
#include "runtime.h"

namespace be {

void node_retain(Node* n) { n->refcount.fetch_add(1, std::memory_order_relaxed); }
void release_saved(Node* n) {
  for (SavedVar& s : n->saved)
    if (s.storage) { s.storage->drop(); s.storage = nullptr; }
  n->saved.clear();
}
void node_drop(Node* n) {
  // iterative to avoid deep recursion on long chains
  std::vector<Node*> stack{n};
  std::vector<Tensor*> leaves;
  while (!stack.empty()) {
    Node* x = stack.back();
    stack.pop_back();
    if (x->refcount.fetch_sub(1, std::memory_order_acq_rel) != 1) continue;
    for (Edge& e : x->edges) {
      if (e.kind == Edge::NODE) stack.push_back(e.node);
      else if (e.kind == Edge::LEAF) leaves.push_back(e.leaf);
    }
    release_saved(x);
    delete x;
  }
  for (Tensor* t : leaves) tensor_drop(t);
}

void save(Node* n, Tensor* t) {
  SavedVar s;
  if (t) {
    s.storage = t->storage;
    t->storage->retain();
    s.offset = t->offset;
    s.rank = t->rank;
    for (int i = 0; i < t->rank; ++i) { s.shape[i] = t->shape[i]; s.strides[i] = t->strides[i]; }
    s.dtype = t->dtype;
    s.version = t->version();
    s.defined = true;
  }
  n->saved.push_back(s);
}

Tensor* unpack(Node* n, int i, TRef& holder) {
  BE_REQUIRE(i < (int)n->saved.size(), BE_E_DOUBLE_BACKWARD,
             std::string("saved tensors of ") + n->name + " were already freed (retain_graph=0)");
  SavedVar& s = n->saved[i];
  if (!s.defined) return nullptr;
  BE_REQUIRE(s.storage != nullptr, BE_E_DOUBLE_BACKWARD,
             std::string("saved tensors of ") + n->name + " were already freed (retain_graph=0)");
  if (s.storage->version.load() != s.version)
    fail(BE_E_VERSION, std::string("one of the tensors saved by ") + n->name +
                           " was modified in place after it was saved (version " + std::to_string(s.version) +
                           " -> " + std::to_string(s.storage->version.load()) + ")");
  Tensor* t = new Tensor();
  t->storage = s.storage;
  s.storage->retain();
  t->offset = s.offset;
  t->rank = s.rank;
  for (int k = 0; k < s.rank; ++k) { t->shape[k] = s.shape[k]; t->strides[k] = s.strides[k]; }
  t->dtype = s.dtype;
  holder = TRef(t);
  return t;
}

// ------------------------------------------------------------------ GradSink
bool GradSink::needs(int i) const { return node->edges[i].kind != Edge::NONE; }

Tensor* GradSink::dest(int i, float* beta) {
  if (node->edges[i].kind == Edge::NONE) return nullptr;
  bool existing = false;
  Tensor* t = acquire(i, &existing);
  slots[i].target = t;
  slots[i].used = true;
  *beta = existing ? 1.f : 0.f;
  return t;
}

Tensor* GradSink::dest_fresh(int i) {
  if (node->edges[i].kind == Edge::NONE) return nullptr;
  bool existing = false;
  Tensor* t = acquire(i, &existing);
  slots[i].target = t;
  slots[i].used = true;
  if (!existing) return t;
  TRef tmp = new_tensor(t->shape, t->rank, t->dtype);
  slots[i].tmp = tmp.release();
  return slots[i].tmp;
}

void GradSink::give(int i, TRef t) {
  if (node->edges[i].kind == Edge::NONE) return;
  if (t->refcount.load() == 1 && adopt(i, t.get())) {
    Tensor* raw = t.release();  // ownership moved to the engine
    finalize(i, raw);
    return;
  }
  float beta = 0.f;
  Tensor* d = dest(i, &beta);
  k::axpby(t->data(), t->dtype, d->data(), d->dtype, d->numel(), 1.f, beta, ctx().stream);
  commit(i);
}

void GradSink::commit(int i) {
  Slot& s = slots[i];
  if (!s.used) return;
  if (s.tmp) {
    k::axpby(s.tmp->data(), s.tmp->dtype, s.target->data(), s.target->dtype, s.target->numel(), 1.f, 1.f,
             ctx().stream);
    tensor_drop(s.tmp);
    s.tmp = nullptr;
  }
  finalize(i, s.target);
  s.used = false;
}

// ------------------------------------------------------------------ engine
namespace {
struct PKey {
  Node* n;
  int k;
  bool operator==(const PKey& o) const { return n == o.n && k == o.k; }
};
struct PKeyHash {
  size_t operator()(const PKey& p) const { return std::hash<void*>()(p.n) * 31 + p.k; }
};
struct BySeq {
  bool operator()(Node* a, Node* b) const { return a->seq < b->seq; }
};

void accumulate_leaf(Tensor* leaf, Tensor* g) {
  cudaStream_t s = ctx().stream;
  if (!leaf->grad) {
    TRef ng = ddp_active() ? TRef(ddp_grad_view(leaf)) : TRef();
    if (!ng) ng = new_tensor(leaf->shape, leaf->rank, BE_F32);
    k::axpby(g->data(), g->dtype, ng->data(), BE_F32, leaf->numel(), 1.f, 0.f, s);
    leaf->grad = ng.release();
  } else {
    k::axpby(g->data(), g->dtype, leaf->grad->data(), leaf->grad->dtype, leaf->numel(), 1.f, 1.f, s);
    leaf->grad->bump_version();
  }
  if (ddp_active()) ddp_on_leaf_grad_ready(leaf);
  else if (opt_param(leaf)) opt_on_grad_final(leaf);
}
}  // namespace

void run_backward(Tensor* root, Tensor* upstream, bool retain) {
  BE_REQUIRE(root->requires_grad, BE_E_ARG, "backward: root does not require grad");
  cudaStream_t s = ctx().stream;
  TRef seed;
  bool ones = false;
  if (upstream) {
    BE_REQUIRE(upstream->numel() == root->numel(), BE_E_SHAPE, "backward: upstream shape mismatch");
    seed = TRef(upstream, false);
  } else {
    BE_REQUIRE(root->numel() == 1, BE_E_NO_UPSTREAM, "backward: non-scalar root needs an upstream gradient");
    seed = new_tensor(root->shape, root->rank, root->dtype == BE_BF16 ? BE_BF16 : BE_F32);
    k::fill(seed->data(), 1, seed->dtype, 1.0, s);
    ones = true;
  }
  if (ddp_active()) ddp_begin_backward();
  if (!root->grad_fn) {  // leaf root
    accumulate_leaf(root, seed.get());
    opt_end_backward();
    return;
  }
  // 1. dependency counts (+ per-leaf use counts for the overlapped optimizer:
  // a registered parameter's gradient is final once every edge to it is done)
  const bool opt = opt_active() && !ddp_active();
  std::unordered_map<Node*, int> deps;
  std::unordered_map<Tensor*, int> leaf_uses;
  std::vector<Node*> stack{root->grad_fn};
  std::unordered_set<Node*> seen{root->grad_fn};
  while (!stack.empty()) {
    Node* n = stack.back();
    stack.pop_back();
    BE_REQUIRE(!n->consumed, BE_E_DOUBLE_BACKWARD,
               std::string("backward through ") + n->name + " a second time without retain_graph");
    for (Edge& e : n->edges) {
      if (opt && e.kind == Edge::LEAF && opt_param(e.leaf)) leaf_uses[e.leaf]++;
      if (e.kind != Edge::NODE) continue;
      deps[e.node]++;
      if (seen.insert(e.node).second) stack.push_back(e.node);
    }
  }
  std::vector<Tensor*> final_leaves;             // completed by the current node's VJP
  std::vector<Tensor*> ddp_leaves;               // DDP: grads landed in the current node's VJP
  std::unordered_set<Tensor*> partial_leaves;    // got a gradient, some edges never ran
  // 2. reverse-topological sweep
  std::unordered_map<PKey, Tensor*, PKeyHash> pending;  // owned refs
  pending[{root->grad_fn, root->output_nr}] = seed.release();
  std::priority_queue<Node*, std::vector<Node*>, BySeq> ready;
  ready.push(root->grad_fn);
  root->grad_fn->upstream_is_ones = ones;
  std::vector<Node*> to_release;
  try {
    while (!ready.empty()) {
      Node* n = ready.top();
      ready.pop();
      GradSink sink;
      sink.node = n;
      sink.retain = retain;
      sink.upstream.assign(n->outs.size(), nullptr);
      bool any = false;
      for (int k2 = 0; k2 < (int)n->outs.size(); ++k2) {
        auto it = pending.find({n, k2});
        if (it != pending.end()) { sink.upstream[k2] = it->second; any = true; }
      }
      sink.slots.assign(n->edges.size(), GradSink::Slot());
      sink.acquire = [&](int i, bool* existing) -> Tensor* {
        Edge& e = n->edges[i];
        if (e.kind == Edge::LEAF) {
          Tensor* leaf = e.leaf;
          if (leaf->grad) { *existing = true; return leaf->grad; }
          TRef g = ddp_active() ? TRef(ddp_grad_view(leaf)) : TRef();
          if (!g) g = new_tensor(leaf->shape, leaf->rank, BE_F32);
          leaf->grad = g.release();
          *existing = false;
          return leaf->grad;
        }
        PKey key{e.node, e.output_nr};
        auto it = pending.find(key);
        if (it != pending.end()) { *existing = true; return it->second; }
        const OutMeta& m = e.node->outs[e.output_nr];
        TRef g = new_tensor(m.shape, m.rank, m.dtype);
        Tensor* raw = g.release();
        pending[key] = raw;
        *existing = false;
        return raw;
      };
      sink.adopt = [&](int i, Tensor* t) -> bool {
        Edge& e = n->edges[i];
        if (e.kind == Edge::LEAF) {
          Tensor* leaf = e.leaf;
          if (leaf->grad || ddp_active() || t->dtype != BE_F32 || !t->is_contiguous() ||
              t->numel() != leaf->numel())
            return false;
          t->rank = leaf->rank;
          int64_t st = 1;
          for (int d = leaf->rank - 1; d >= 0; --d) { t->shape[d] = leaf->shape[d]; t->strides[d] = st; st *= leaf->shape[d]; }
          leaf->grad = t;
          return true;
        }
        PKey key{e.node, e.output_nr};
        if (pending.count(key)) return false;
        const OutMeta& m = e.node->outs[e.output_nr];
        int64_t mn = 1;
        for (int d = 0; d < m.rank; ++d) mn *= m.shape[d];
        if (m.dtype != t->dtype || !t->is_contiguous() || mn != t->numel()) return false;
        t->rank = m.rank;
        int64_t st = 1;
        for (int d = m.rank - 1; d >= 0; --d) { t->shape[d] = m.shape[d]; t->strides[d] = st; st *= m.shape[d]; }
        pending[key] = t;
        return true;
      };
      sink.fuse = [&](int i, k::SgdFuse* f) -> bool {
        if (!opt) return false;
        Edge& e = n->edges[i];
        if (e.kind != Edge::LEAF || !opt_param(e.leaf) || e.leaf->grad) return false;
        auto it = leaf_uses.find(e.leaf);
        if (it == leaf_uses.end() || it->second != 1) return false;  // more contributions to come
        return opt_fuse_desc(e.leaf, f);
      };
      sink.fused = [&](int i) {
        Edge& e = n->edges[i];
        --leaf_uses[e.leaf];
        opt_fused_done(e.leaf);
      };
      sink.finalize = [&](int i, Tensor* t) {
        Edge& e = n->edges[i];
        if (e.kind == Edge::LEAF) {
          t->bump_version();
          if (ddp_active()) ddp_leaves.push_back(e.leaf);
          else if (opt && opt_param(e.leaf)) {
            partial_leaves.insert(e.leaf);
            if (--leaf_uses[e.leaf] == 0) { final_leaves.push_back(e.leaf); partial_leaves.erase(e.leaf); }
          }
        }
      };
      if (any) {
        for (size_t k2 = 0; k2 < n->saved.size(); ++k2) {  // version check at unpack
          SavedVar& sv = n->saved[k2];
          if (sv.defined && sv.storage && sv.storage->version.load() != sv.version)
            fail(BE_E_VERSION, std::string("one of the tensors saved by ") + n->name +
                                   " was modified in place after it was saved");
        }
        n->vjp(n, sink);
        // updates are enqueued only after every kernel of this VJP (which may
        // still read the parameter or its bf16 shadow after committing dW)
        for (Tensor* leaf : final_leaves) opt_on_grad_final(leaf);
        final_leaves.clear();
        // likewise DDP bucket launches (their allreduce may be followed by
        // the overlapped update of the bucket's parameters)
        for (Tensor* leaf : ddp_leaves) ddp_on_leaf_grad_ready(leaf);
        ddp_leaves.clear();
      }
      n->upstream_is_ones = false;
      for (int k2 = 0; k2 < (int)n->outs.size(); ++k2) {
        auto it = pending.find({n, k2});
        if (it != pending.end()) { tensor_drop(it->second); pending.erase(it); }
      }
      if (!retain) { release_saved(n); n->consumed = true; }
      for (Edge& e : n->edges) {
        if (e.kind != Edge::NODE) continue;
        if (--deps[e.node] == 0) ready.push(e.node);
      }
    }
  } catch (...) {
    for (auto& kv : pending) tensor_drop(kv.second);
    throw;
  }
  for (auto& kv : pending) tensor_drop(kv.second);
  for (Tensor* leaf : partial_leaves) opt_on_grad_final(leaf);
  opt_end_backward();
}

}  // namespace be

using namespace be;
extern "C" {

be_status be_backward(be_tensor root, be_tensor upstream, int retain_graph) {
  BE_API_BEGIN
  Tensor* r = check_handle(root);
  Tensor* u = upstream ? check_handle(upstream) : nullptr;
  run_backward(r, u, retain_graph != 0);
  BE_API_END
}

be_status be_grad(be_tensor leaf, be_tensor* out) {
  BE_API_BEGIN
  Tensor* t = check_handle(leaf);
  if (t->grad) { t->grad->retain(); *out = reinterpret_cast<be_tensor>(t->grad); }
  else *out = nullptr;
  BE_API_END
}

be_status be_zero_grad(const be_tensor* params, int n) {
  BE_API_BEGIN
  for (int i = 0; i < n; ++i) {
    Tensor* t = check_handle(params[i]);
    if (t->grad) { tensor_drop(t->grad); t->grad = nullptr; }
  }
  BE_API_END
}

be_status be_detach(be_tensor h, be_tensor* out) {
  BE_API_BEGIN
  Tensor* t = check_handle(h);
  TRef v = make_view(t, t->shape, t->rank, t->strides, t->offset);
  *out = reinterpret_cast<be_tensor>(v.release());
  BE_API_END
}

}  // extern "C"
