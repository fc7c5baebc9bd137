// ops.cpp — be_op dispatch for the dense / elementwise / loss operators and
// their vector-Jacobian products, the fused SGD step and be_gemm.
//
// Each forward op (§5.2) checks shapes on the host,
// allocates its output from the caching allocator on the compute stream,
// enqueues its kernel(s) and returns; when grad mode is on and an input
// requires grad it records a Node with version-pinned saved tensors
// (PAPER.md:158-162).  The VJPs follow the definitions in oracle/ops.py
// (they share no code with it): Linear dX = dY·Wᵀ, dW = Xᵀ·dY, db = Σ_n dY
// (Listing 1); softmax-CE dz = (softmax − onehot)/B
// (SPEC S:615).
#include "ops_common.h"

namespace be {

// ------------------------------------------------------------------ helpers
Node* new_node(const char* name, int op, VjpFn vjp, std::initializer_list<Tensor*> inputs) {
  if (!grad_enabled()) return nullptr;
  bool any = false;
  for (Tensor* t : inputs) any |= (t && t->requires_grad);
  if (!any) return nullptr;
  Node* n = new Node();
  n->name = name;
  n->op = op;
  n->vjp = vjp;
  n->seq = ctx().seq.fetch_add(1);
  for (Tensor* t : inputs) {
    Edge e;
    if (t && t->requires_grad) {
      if (t->grad_fn) { e.kind = Edge::NODE; e.node = t->grad_fn; node_retain(t->grad_fn); e.output_nr = t->output_nr; }
      else { e.kind = Edge::LEAF; e.leaf = t; t->retain(); }
    }
    n->edges.push_back(e);
  }
  return n;
}

void set_output(Node* n, Tensor* out, int k) {
  if ((int)n->outs.size() <= k) n->outs.resize(k + 1);
  OutMeta& m = n->outs[k];
  m.rank = out->rank;
  for (int i = 0; i < out->rank; ++i) m.shape[i] = out->shape[i];
  m.dtype = out->dtype;
  if (out->grad_fn) node_drop(out->grad_fn);
  out->grad_fn = n;
  node_retain(n);
  out->output_nr = k;
  out->requires_grad = true;
}

void finish_node(Node* n) {
  if (n) node_drop(n);  // outputs hold the references
}

// bf16 shadow of an fp32 parameter (refreshed when the master changed).
Tensor* weight_operand(Tensor* w) {
  if (ctx().compute == BE_F32 || w->dtype == BE_BF16) return w;
  BE_REQUIRE(w->dtype == BE_F32, BE_E_DTYPE, "weights must be f32 or bf16");
  BE_REQUIRE(w->is_contiguous(), BE_E_NONCONTIG, "weights must be contiguous");
  if (!w->shadow) {
    TRef s = new_tensor(w->shape, w->rank, BE_BF16);
    w->shadow = s.release();
    w->shadow_version = ~0ull;
  }
  if (w->shadow_version != w->version()) {
    k::cast(w->data(), BE_F32, w->shadow->data(), BE_BF16, w->numel(), ctx().stream);
    w->shadow->bump_version();
    w->shadow_version = w->version();
  }
  return w->shadow;
}

// Differentiable cast (recorded on the tape when x requires grad).
static void vjp_cast(Node* n, GradSink& sink) {
  Tensor* g = sink.upstream[0];
  if (!g) return;
  float beta;
  Tensor* d = sink.dest(0, &beta);
  if (!d) return;
  k::axpby(g->data(), g->dtype, d->data(), d->dtype, d->numel(), 1.f, beta, ctx().stream);
  sink.commit(0);
}
TRef cast_op(Tensor* x, be_dtype dt) {
  if (x->dtype == dt) return TRef(x, false);
  BE_REQUIRE(x->is_contiguous(), BE_E_NONCONTIG, "cast needs a contiguous tensor");
  TRef y = new_tensor(x->shape, x->rank, dt);
  k::cast(x->data(), x->dtype, y->data(), dt, x->numel(), ctx().stream);
  Node* n = (dt == BE_F32 || dt == BE_BF16) ? new_node("cast", BE_OP_CAST, vjp_cast, {x}) : nullptr;
  if (n) { set_output(n, y.get(), 0); finish_node(n); }
  return y;
}
// Activation operand in the compute dtype.
TRef act_operand(Tensor* x) {
  be_dtype want = ctx().compute;
  if (x->dtype == want) return TRef(x, false);
  return cast_op(x, want);
}
TRef contiguous_like(Tensor* g, be_dtype dt) {  // copy/cast to a fresh contiguous tensor
  BE_REQUIRE(g->is_contiguous(), BE_E_NONCONTIG, "expected contiguous gradient");
  if (g->dtype == dt) return TRef(g, false);
  TRef y = new_tensor(g->shape, g->rank, dt);
  k::cast(g->data(), g->dtype, y->data(), dt, g->numel(), ctx().stream);
  return y;
}

// ------------------------------------------------------------------ LINEAR
// y[B,out] = act(x[B,in]·W[in,out] + b)   (Listing 1 LinearLayer)
static void vjp_linear(Node* n, GradSink& sink) {
  cudaStream_t s = ctx().stream;
  Tensor* g0 = sink.upstream[0];
  TRef hx, hw, hy;
  Tensor* x = unpack(n, 0, hx);
  Tensor* w = unpack(n, 1, hw);  // operand-precision weight (shadow in bf16 mode)
  Tensor* y = unpack(n, 2, hy);  // saved only with act
  const int act = (int)n->iattr[0];
  const bool has_b = n->iattr[1] != 0;
  const int64_t B = x->shape[0], IN = x->shape[1], OUT = w->shape[1];
  const be_dtype opd = x->dtype;
  // dz = g ⊙ 1[y>0] (act) and db = Σ_rows dz, fused in one pass
  TRef gz = contiguous_like(g0, opd);
  TRef dz;
  if (act) dz = new_tensor({B, OUT}, opd);
  else dz = gz;
  if (has_b && sink.needs(2)) {
    float bb;
    Tensor* db = sink.dest(2, &bb);
    k::relu_bwd_colsum(gz->data(), act ? y->data() : nullptr, dz->data(), B, OUT, opd, db->ptr<float>(), bb, act, s);
    sink.commit(2);
  } else if (act) {
    k::relu_bwd(gz->data(), y->data(), dz->data(), B * OUT, opd, 0.f, s);
  }
  gz = TRef();
  // dW[in,out] = xᵀ·dz  (A = xᵀ MN-major, B = dzᵀ MN-major), fp32
  k::GemmDesc gw;
  gw.M = (int)IN; gw.N = (int)OUT; gw.K = (int)B;
  gw.A = x->data(); gw.lda = IN; gw.a_kmajor = false;
  gw.B = dz->data(); gw.ldb = OUT; gw.b_kmajor = false;
  gw.ab = opd; gw.ldd = OUT;
  // overlapped SGD: when this is the weight's only gradient contribution, the
  // wgrad GEMM applies the update in its epilogue (no dW tensor, no separate
  // SGD pass) — after dX, which still reads the pre-update weight
  k::SgdFuse fz;
  bool fuse = sink.needs(1) && opd == BE_BF16 && k::gemm_tc_ok(gw) && sink.fuse(1, &fz);
  if (fuse) {
    gw.upd = &fz;
    fuse = k::gemm_update_ok(gw);
    gw.upd = nullptr;
  }
  if (sink.needs(1) && !fuse) {
    float bw;
    Tensor* dw = sink.dest(1, &bw);
    gw.D = dw->data(); gw.d = dw->dtype; gw.beta = bw;
    k::gemm(gw, s);
    sink.commit(1);
  }
  if (sink.needs(0)) {  // dX[B,in] = dz·Wᵀ  (A = dz K-major, B = W K-major)
    float bx;
    Tensor* dx = sink.dest(0, &bx);
    TRef dxc;
    Tensor* dxt = dx;
    if (dx->dtype != opd) { dxc = new_tensor(dx->shape, dx->rank, opd); dxt = dxc.get(); }
    k::GemmDesc gd;
    gd.M = (int)B; gd.N = (int)IN; gd.K = (int)OUT;
    gd.A = dz->data(); gd.lda = OUT; gd.a_kmajor = true;
    gd.B = w->data(); gd.ldb = OUT; gd.b_kmajor = true;
    gd.ab = opd; gd.D = dxt->data(); gd.ldd = IN; gd.d = dxt->dtype; gd.beta = dxc ? 0.f : bx;
    k::gemm(gd, s);
    if (dxc) k::axpby(dxc->data(), opd, dx->data(), dx->dtype, dx->numel(), 1.f, bx, s);
    sink.commit(0);
  }
  if (fuse) {
    gw.upd = &fz;
    k::gemm(gw, s);
    sink.fused(1);
  }
}

static void op_linear(const be_tensor* in, int n_in, const void* attrs, be_tensor* out, int n_out) {
  BE_REQUIRE(n_in == 2 || n_in == 3, BE_E_ARG, "linear: 2 or 3 inputs");
  Tensor* x0 = check_handle(in[0]);
  Tensor* w0 = check_handle(in[1]);
  Tensor* b = n_in == 3 && in[2] ? check_handle(in[2]) : nullptr;
  be_linear_attrs a{0, 0};
  if (attrs) a = *reinterpret_cast<const be_linear_attrs*>(attrs);
  BE_REQUIRE(x0->rank == 2 && w0->rank == 2, BE_E_SHAPE, "linear: x[B,in], w[in,out]");
  BE_REQUIRE(x0->shape[1] == w0->shape[0], BE_E_SHAPE, "linear: inner dimensions differ");
  BE_REQUIRE(!b || (b->rank == 1 && b->shape[0] == w0->shape[1] && b->dtype == BE_F32), BE_E_SHAPE,
             "linear: bias must be f32 [out]");
  BE_REQUIRE(x0->is_contiguous(), BE_E_NONCONTIG, "linear: x must be contiguous");
  TRef x = act_operand(x0);
  Tensor* w = weight_operand(w0);
  const int64_t B = x->shape[0], IN = x->shape[1], OUT = w->shape[1];
  const be_dtype od = (a.out_f32 || ctx().compute == BE_F32) ? BE_F32 : BE_BF16;
  TRef y = new_tensor({B, OUT}, od);
  k::GemmDesc gd;
  gd.M = (int)B; gd.N = (int)OUT; gd.K = (int)IN;
  gd.A = x->data(); gd.lda = IN; gd.a_kmajor = true;
  gd.B = w->data(); gd.ldb = OUT; gd.b_kmajor = false;
  gd.ab = x->dtype; gd.D = y->data(); gd.ldd = OUT; gd.d = od;
  gd.bias = b ? b->ptr<float>() : nullptr; gd.act = a.act;
  k::gemm(gd, ctx().stream);
  Node* n = new_node("linear", BE_OP_LINEAR, vjp_linear, {x.get(), w0, b});
  if (n) {
    save(n, x.get());
    save(n, w);
    save(n, a.act ? y.get() : nullptr);
    n->iattr[0] = a.act;
    n->iattr[1] = b != nullptr;
    set_output(n, y.get(), 0);
    finish_node(n);
  }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

// ------------------------------------------------------------------ MATMUL
static void vjp_matmul(Node* n, GradSink& sink) {
  cudaStream_t s = ctx().stream;
  TRef ha, hb;
  Tensor* a = unpack(n, 0, ha);
  Tensor* b = unpack(n, 1, hb);
  const int64_t M = a->shape[0], K = a->shape[1], N = b->shape[1];
  TRef g = contiguous_like(sink.upstream[0], a->dtype);
  if (sink.needs(1)) {  // dB[K,N] = Aᵀ·G
    float be_;
    Tensor* db = sink.dest(1, &be_);
    TRef tmp;
    Tensor* d = db;
    if (db->dtype != BE_F32 && db->dtype != BE_BF16) fail(BE_E_DTYPE, "matmul grad dtype");
    k::GemmDesc gd;
    gd.M = (int)K; gd.N = (int)N; gd.K = (int)M;
    gd.A = a->data(); gd.lda = K; gd.a_kmajor = false;
    gd.B = g->data(); gd.ldb = N; gd.b_kmajor = false;
    gd.ab = a->dtype; gd.D = d->data(); gd.ldd = N; gd.d = d->dtype; gd.beta = be_;
    k::gemm(gd, s);
    sink.commit(1);
  }
  if (sink.needs(0)) {  // dA[M,K] = G·Bᵀ
    float be_;
    Tensor* da = sink.dest(0, &be_);
    k::GemmDesc gd;
    gd.M = (int)M; gd.N = (int)K; gd.K = (int)N;
    gd.A = g->data(); gd.lda = N; gd.a_kmajor = true;
    gd.B = b->data(); gd.ldb = N; gd.b_kmajor = true;
    gd.ab = a->dtype; gd.D = da->data(); gd.ldd = K; gd.d = da->dtype; gd.beta = be_;
    k::gemm(gd, s);
    sink.commit(0);
  }
}
static void op_matmul(const be_tensor* in, int n_in, const void*, be_tensor* out, int) {
  BE_REQUIRE(n_in == 2, BE_E_ARG, "matmul: 2 inputs");
  Tensor* a0 = check_handle(in[0]);
  Tensor* b0 = check_handle(in[1]);
  BE_REQUIRE(a0->rank == 2 && b0->rank == 2 && a0->shape[1] == b0->shape[0], BE_E_SHAPE,
             "matmul: [M,K]·[K,N] required");
  BE_REQUIRE(a0->dtype == b0->dtype, BE_E_DTYPE, "matmul: dtypes differ");
  BE_REQUIRE(a0->dtype == BE_F32 || a0->dtype == BE_BF16, BE_E_UNSUPPORTED, "matmul: f32 or bf16 only");
  BE_REQUIRE(a0->is_contiguous() && b0->is_contiguous(), BE_E_NONCONTIG, "matmul: contiguous inputs");
  const int64_t M = a0->shape[0], K = a0->shape[1], N = b0->shape[1];
  TRef y = new_tensor({M, N}, a0->dtype);
  k::GemmDesc gd;
  gd.M = (int)M; gd.N = (int)N; gd.K = (int)K;
  gd.A = a0->data(); gd.lda = K; gd.a_kmajor = true;
  gd.B = b0->data(); gd.ldb = N; gd.b_kmajor = false;
  gd.ab = a0->dtype; gd.D = y->data(); gd.ldd = N; gd.d = a0->dtype;
  if (K == 0) k::fill(y->data(), M * N, y->dtype, 0.0, ctx().stream);
  else k::gemm(gd, ctx().stream);
  Node* n = new_node("matmul", BE_OP_MATMUL, vjp_matmul, {a0, b0});
  if (n) { save(n, a0); save(n, b0); set_output(n, y.get(), 0); finish_node(n); }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

// ------------------------------------------------------------------ ADD (broadcast), ADD_RELU, MUL, RELU
// Reduce g (out shape) onto an input of shape `ish` (right-aligned broadcast,
// SPEC S:83-91): sum over broadcast dims.  Supported reductions:
// identity, and summing leading dims down to a trailing block (row-vector
// bias) — both as column sums over a [rows, cols] view.
static void unbroadcast_into(Tensor* g, Tensor* d, float beta) {
  cudaStream_t s = ctx().stream;
  const int64_t n_out = g->numel(), n_in = d->numel();
  if (n_out == n_in) { k::axpby(g->data(), g->dtype, d->data(), d->dtype, n_in, 1.f, beta, s); return; }
  // trailing-block broadcast: input shape equals the last dims of out (leading dims size-1 or absent)
  BE_REQUIRE(d->dtype == BE_F32, BE_E_UNSUPPORTED, "broadcast grad must be f32");
  BE_REQUIRE(n_in > 0 && n_out % n_in == 0, BE_E_UNSUPPORTED, "unsupported broadcast pattern in backward");
  k::colsum(g->data(), n_out / n_in, n_in, g->dtype, d->ptr<float>(), beta, s);
}
static bool trailing_block(const Tensor* out, const Tensor* in) {
  // in's non-1 dims must equal out's trailing dims
  int64_t n = in->numel();
  int64_t acc = 1;
  for (int i = out->rank - 1; i >= 0; --i) {
    if (acc == n) break;
    acc *= out->shape[i];
  }
  if (acc != n) return false;
  int j = in->rank - 1;
  int i = out->rank - 1;
  int64_t prod = 1;
  while (prod < n && i >= 0) {
    while (j >= 0 && in->shape[j] == 1) --j;
    if (j < 0 || in->shape[j] != out->shape[i]) return false;
    prod *= out->shape[i];
    --i; --j;
  }
  return true;
}
static void vjp_add(Node* n, GradSink& sink) {
  Tensor* g = sink.upstream[0];
  const int act = (int)n->iattr[0];
  if (act && g->is_contiguous()) {
    // fused: both inputs receive dy·1[y>0] from one pass when shapes match
    TRef hy;
    Tensor* y = unpack(n, 0, hy);
    const int64_t ne = g->numel();
    float b0 = 0.f, b1 = 0.f;
    Tensor* d0 = sink.needs(0) ? sink.dest(0, &b0) : nullptr;
    Tensor* d1 = sink.needs(1) ? sink.dest(1, &b1) : nullptr;
    const bool ok0 = !d0 || (d0->numel() == ne && d0->dtype == g->dtype && d0->is_contiguous());
    const bool ok1 = !d1 || (d1->numel() == ne && d1->dtype == g->dtype && d1->is_contiguous() && d1 != d0);
    if (ok0 && ok1) {
      k::relu_bwd2(g->data(), y->data(), d0 ? d0->data() : nullptr, b0, d1 ? d1->data() : nullptr, b1, ne, g->dtype,
                   ctx().stream);
      if (d0) sink.commit(0);
      if (d1) sink.commit(1);
      return;
    }
    // general path below (broadcast or aliasing): destinations already acquired
    TRef dz = new_tensor(g->shape, g->rank, g->dtype);
    k::relu_bwd(g->data(), y->data(), dz->data(), ne, g->dtype, 0.f, ctx().stream);
    if (d0) { unbroadcast_into(dz.get(), d0, b0); sink.commit(0); }
    if (d1) {
      float bb = b1;
      if (d1 == d0) bb = 1.f;  // same tensor added twice
      unbroadcast_into(dz.get(), d1, bb);
      sink.commit(1);
    }
    return;
  }
  TRef dz;
  if (act) {
    TRef hy;
    Tensor* y = unpack(n, 0, hy);
    dz = new_tensor(g->shape, g->rank, g->dtype);
    k::relu_bwd(g->data(), y->data(), dz->data(), g->numel(), g->dtype, 0.f, ctx().stream);
  } else {
    dz = TRef(g, false);
  }
  for (int i = 0; i < 2; ++i) {
    if (!sink.needs(i)) continue;
    float beta;
    Tensor* d = sink.dest(i, &beta);
    unbroadcast_into(dz.get(), d, beta);
    sink.commit(i);
  }
}
static void broadcast_shape(Tensor* a, Tensor* b, int64_t* shape, int* rank) {
  int r = std::max(a->rank, b->rank);
  for (int i = 0; i < r; ++i) {
    int ia = a->rank - r + i, ib = b->rank - r + i;
    int64_t da = ia >= 0 ? a->shape[ia] : 1, db = ib >= 0 ? b->shape[ib] : 1;
    BE_REQUIRE(da == db || da == 1 || db == 1, BE_E_BROADCAST,
               "broadcast: dims " + std::to_string(da) + " and " + std::to_string(db) + " are incompatible");
    shape[i] = std::max(da, db);
    if (da == 0 || db == 0) shape[i] = 0;
  }
  *rank = r;
}
static void op_add(const be_tensor* in, int n_in, const void* attrs, be_tensor* out, int, int force_act) {
  BE_REQUIRE(n_in == 2, BE_E_ARG, "add: 2 inputs");
  Tensor* a = check_handle(in[0]);
  Tensor* b = check_handle(in[1]);
  BE_REQUIRE(a->dtype == b->dtype, BE_E_DTYPE, "add: dtypes differ");
  BE_REQUIRE(a->dtype == BE_F32 || a->dtype == BE_BF16, BE_E_UNSUPPORTED, "add: f32/bf16");
  int act = force_act;
  if (attrs && !force_act) act = *reinterpret_cast<const int*>(attrs);
  int64_t shape[6];
  int rank;
  broadcast_shape(a, b, shape, &rank);
  TRef y = new_tensor(shape, rank, a->dtype);
  const int64_t n = y->numel();
  if (a->numel() == n && b->numel() == n && a->is_contiguous() && b->is_contiguous()) {
    k::add_same(a->data(), b->data(), y->data(), n, a->dtype, act, ctx().stream);
  } else {
    k::BcastDesc d;
    d.rank = rank;
    for (int i = 0; i < rank; ++i) {
      d.shape[i] = shape[i];
      int ia = a->rank - rank + i, ib = b->rank - rank + i;
      d.sa[i] = (ia >= 0 && a->shape[ia] != 1) ? a->strides[ia] : 0;
      d.sb[i] = (ib >= 0 && b->shape[ib] != 1) ? b->strides[ib] : 0;
    }
    k::add_bcast(a->data(), b->data(), y->data(), d, a->dtype, act, ctx().stream);
  }
  Node* node = new_node(act ? "add_relu" : "add", BE_OP_ADD, vjp_add, {a, b});
  if (node) {
    for (Tensor* t : {a, b})
      if (t->requires_grad && t->numel() != n)
        BE_REQUIRE(trailing_block(y.get(), t), BE_E_UNSUPPORTED, "add: broadcast pattern has no backward kernel");
    save(node, act ? y.get() : nullptr);
    node->iattr[0] = act;
    set_output(node, y.get(), 0);
    finish_node(node);
  }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

static void vjp_mul(Node* n, GradSink& sink) {
  Tensor* g = sink.upstream[0];
  TRef ha, hb;
  Tensor* a = unpack(n, 0, ha);
  Tensor* b = unpack(n, 1, hb);
  for (int i = 0; i < 2; ++i) {
    if (!sink.needs(i)) continue;
    float beta;
    Tensor* d = sink.dest(i, &beta);
    BE_REQUIRE(d->dtype == g->dtype, BE_E_DTYPE, "mul backward dtype");
    k::mul_acc(g->data(), (i == 0 ? b : a)->data(), d->data(), g->numel(), g->dtype, beta, ctx().stream);
    sink.commit(i);
  }
}
static void op_mul(const be_tensor* in, int n_in, const void*, be_tensor* out, int) {
  BE_REQUIRE(n_in == 2, BE_E_ARG, "mul: 2 inputs");
  Tensor* a = check_handle(in[0]);
  Tensor* b = check_handle(in[1]);
  BE_REQUIRE(a->dtype == b->dtype, BE_E_DTYPE, "mul: dtypes differ");
  BE_REQUIRE(a->numel() == b->numel() && a->rank == b->rank, BE_E_SHAPE, "mul: same shapes required");
  BE_REQUIRE(a->is_contiguous() && b->is_contiguous(), BE_E_NONCONTIG, "mul: contiguous");
  TRef y = new_tensor(a->shape, a->rank, a->dtype);
  k::mul_same(a->data(), b->data(), y->data(), a->numel(), a->dtype, ctx().stream);
  Node* n = new_node("mul", BE_OP_MUL, vjp_mul, {a, b});
  if (n) { save(n, a); save(n, b); set_output(n, y.get(), 0); finish_node(n); }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

static void vjp_relu(Node* n, GradSink& sink) {
  Tensor* g = sink.upstream[0];
  TRef hy;
  Tensor* y = unpack(n, 0, hy);
  float beta;
  Tensor* d = sink.dest(0, &beta);
  if (!d) return;
  k::relu_bwd(g->data(), y->data(), d->data(), g->numel(), g->dtype, beta, ctx().stream);
  sink.commit(0);
}
static void op_relu(const be_tensor* in, int n_in, const void*, be_tensor* out, int) {
  BE_REQUIRE(n_in == 1, BE_E_ARG, "relu: 1 input");
  Tensor* x = check_handle(in[0]);
  BE_REQUIRE(x->is_contiguous(), BE_E_NONCONTIG, "relu: contiguous");
  BE_REQUIRE(x->dtype == BE_F32 || x->dtype == BE_BF16, BE_E_DTYPE, "relu: float dtype");
  TRef y = new_tensor(x->shape, x->rank, x->dtype);
  k::relu_fwd(x->data(), y->data(), x->numel(), x->dtype, ctx().stream);
  Node* n = new_node("relu", BE_OP_RELU, vjp_relu, {x});
  if (n) { save(n, y.get()); set_output(n, y.get(), 0); finish_node(n); }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

// ------------------------------------------------------------------ losses
// SOFTMAX_XENT: loss = mean_i(LSE(z_i) − z_i[y_i]); dz computed in the same
// pass and saved, so backward with the implicit upstream 1 is free.
static void vjp_loss(Node* n, GradSink& sink) {
  if (!sink.needs(0)) return;
  TRef hdz;
  Tensor* dz = unpack(n, 0, hdz);
  if (sink.upstream_ones()) {
    if (!sink.retain) {
      // the saved dz IS the gradient; the engine adopts it (its saved slot is
      // released right after this node), so no kernel runs here
      sink.give(0, std::move(hdz));
    } else {
      float beta;
      Tensor* d = sink.dest(0, &beta);
      k::axpby(dz->data(), dz->dtype, d->data(), d->dtype, d->numel(), 1.f, beta, ctx().stream);
      sink.commit(0);
    }
    return;
  }
  TRef gf = contiguous_like(sink.upstream[0], BE_F32);
  Tensor* d = sink.dest_fresh(0);
  k::scale_dev(dz->data(), dz->dtype, d->data(), d->dtype, dz->numel(), gf->ptr<float>(), ctx().stream);
  sink.commit(0);
}
static void op_softmax_xent(const be_tensor* in, int n_in, const void*, be_tensor* out, int n_out) {
  BE_REQUIRE(n_in == 2, BE_E_ARG, "softmax_xent: logits, labels");
  Tensor* z = check_handle(in[0]);
  Tensor* y = check_handle(in[1]);
  BE_REQUIRE(z->rank == 2 && y->rank == 1 && y->shape[0] == z->shape[0], BE_E_SHAPE,
             "softmax_xent: logits[B,C], labels[B]");
  BE_REQUIRE(y->dtype == BE_I32, BE_E_DTYPE, "softmax_xent: labels must be i32");
  BE_REQUIRE(z->dtype == BE_F32 || z->dtype == BE_BF16, BE_E_DTYPE, "softmax_xent: float logits");
  BE_REQUIRE(z->strides[1] == 1, BE_E_NONCONTIG, "softmax_xent: row-contiguous logits");
  const int64_t B = z->shape[0], C = z->shape[1];
  BE_REQUIRE(B > 0, BE_E_EMPTY_REDUCTION, "softmax_xent: empty batch");
  cudaStream_t s = ctx().stream;
  TRef loss = new_tensor(nullptr, 0, BE_F32);
  TRef dz = new_tensor({B, C}, z->dtype);
  TRef rows = new_tensor({B}, BE_F32);
  TRef am;
  if (n_out > 1) am = new_tensor({B}, BE_I32);
  k::softmax_xent(z->data(), z->dtype, z->strides[0], y->ptr<int32_t>(), B, C, rows->ptr<float>(),
                  loss->ptr<float>(), dz->data(), dz->dtype, am ? am->ptr<int32_t>() : nullptr, s);
  Node* n = new_node("softmax_xent", BE_OP_SOFTMAX_XENT, vjp_loss, {z});
  if (n) { save(n, dz.get()); set_output(n, loss.get(), 0); finish_node(n); }
  out[0] = reinterpret_cast<be_tensor>(loss.release());
  if (n_out > 1) out[1] = reinterpret_cast<be_tensor>(am.release());
}
static void op_bce(const be_tensor* in, int n_in, const void*, be_tensor* out, int) {
  BE_REQUIRE(n_in == 2, BE_E_ARG, "bce_logits: z, labels");
  Tensor* z = check_handle(in[0]);
  Tensor* y = check_handle(in[1]);
  const int64_t B = z->shape[0];
  BE_REQUIRE(z->numel() == B && y->numel() == B && y->dtype == BE_I32, BE_E_SHAPE, "bce_logits: z[B,1], labels i32[B]");
  BE_REQUIRE(z->is_contiguous(), BE_E_NONCONTIG, "bce_logits: contiguous");
  BE_REQUIRE(B > 0, BE_E_EMPTY_REDUCTION, "bce_logits: empty batch");
  TRef loss = new_tensor(nullptr, 0, BE_F32);
  TRef dz = new_tensor(z->shape, z->rank, z->dtype);
  TRef rows = new_tensor({B}, BE_F32);
  k::bce_logits(z->data(), z->dtype, y->ptr<int32_t>(), B, rows->ptr<float>(), loss->ptr<float>(), dz->data(),
                dz->dtype, ctx().stream);
  Node* n = new_node("bce_logits", BE_OP_BCE_LOGITS, vjp_loss, {z});
  if (n) { save(n, dz.get()); set_output(n, loss.get(), 0); finish_node(n); }
  out[0] = reinterpret_cast<be_tensor>(loss.release());
}

// ------------------------------------------------------------------ SUM / MEAN / RESHAPE / CAST / CONCAT
static void vjp_sum(Node* n, GradSink& sink) {
  Tensor* g = sink.upstream[0];
  TRef gf = contiguous_like(g, BE_F32);
  float beta;
  Tensor* d = sink.dest(0, &beta);
  if (!d) return;
  const float scale = n->op == BE_OP_MEAN ? 1.f / (float)std::max<int64_t>(1, d->numel()) : 1.f;
  k::broadcast_scalar(gf->ptr<float>(), d->data(), d->dtype, d->numel(), scale, beta, ctx().stream);
  sink.commit(0);
}
static void op_sum(int op, const be_tensor* in, int n_in, be_tensor* out) {
  BE_REQUIRE(n_in == 1, BE_E_ARG, "sum/mean: 1 input");
  Tensor* x = check_handle(in[0]);
  BE_REQUIRE(x->is_contiguous(), BE_E_NONCONTIG, "sum/mean: contiguous");
  BE_REQUIRE(x->dtype == BE_F32 || x->dtype == BE_BF16, BE_E_DTYPE, "sum/mean: float");
  const int64_t n = x->numel();
  BE_REQUIRE(op == BE_OP_SUM || n > 0, BE_E_EMPTY_REDUCTION, "mean of an empty tensor");
  TRef y = new_tensor(nullptr, 0, BE_F32);
  TRef scratch = new_tensor({1024}, BE_F32);
  k::reduce_sum(x->data(), n, x->dtype, y->ptr<float>(), op == BE_OP_MEAN ? 1.f / (float)n : 1.f,
                scratch->ptr<float>(), ctx().stream);
  Node* nd = new_node(op == BE_OP_SUM ? "sum" : "mean", op, vjp_sum, {x});
  if (nd) { set_output(nd, y.get(), 0); finish_node(nd); }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

static void vjp_reshape(Node* n, GradSink& sink) {
  Tensor* g = sink.upstream[0];
  float beta;
  Tensor* d = sink.dest(0, &beta);
  if (!d) return;
  k::axpby(g->data(), g->dtype, d->data(), d->dtype, d->numel(), 1.f, beta, ctx().stream);
  sink.commit(0);
}
static void op_reshape(const be_tensor* in, int n_in, const void* attrs, be_tensor* out) {
  BE_REQUIRE(n_in == 1 && attrs, BE_E_ARG, "reshape: 1 input + be_shape_attrs");
  Tensor* x = check_handle(in[0]);
  const be_shape_attrs* a = reinterpret_cast<const be_shape_attrs*>(attrs);
  BE_REQUIRE(x->is_contiguous(), BE_E_NONCONTIG, "reshape of a non-contiguous tensor");
  int64_t shape[6];
  int64_t known = 1;
  int neg = -1;
  for (int i = 0; i < a->rank; ++i) {
    shape[i] = a->shape[i];
    if (shape[i] == -1) { BE_REQUIRE(neg < 0, BE_E_SHAPE, "reshape: one -1 at most"); neg = i; }
    else known *= shape[i];
  }
  if (neg >= 0) shape[neg] = known ? x->numel() / known : 0;
  int64_t n = 1;
  for (int i = 0; i < a->rank; ++i) n *= shape[i];
  BE_REQUIRE(n == x->numel(), BE_E_SHAPE, "reshape: element count differs");
  TRef y = make_view(x, shape, a->rank, nullptr, x->offset);
  Node* nd = new_node("reshape", BE_OP_RESHAPE, vjp_reshape, {x});
  if (nd) { set_output(nd, y.get(), 0); finish_node(nd); }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

static void vjp_concat(Node* n, GradSink& sink) {
  Tensor* g = sink.upstream[0];
  const int64_t rows = g->shape[0], ld = g->shape[1];
  int64_t col = 0;
  for (int i = 0; i < (int)n->edges.size(); ++i) {
    const int64_t w = n->iattr[i];
    if (sink.needs(i)) {
      float beta;
      Tensor* d = sink.dest(i, &beta);
      k::slice_cols(g->data(), ld, col, w, rows, d->data(), g->dtype, beta, ctx().stream);
      sink.commit(i);
    }
    col += w;
  }
}
static void op_concat(const be_tensor* in, int n_in, be_tensor* out) {
  BE_REQUIRE(n_in >= 1 && n_in <= 8, BE_E_ARG, "concat: 1..8 inputs");
  std::vector<Tensor*> xs;
  std::vector<const void*> ptrs;
  std::vector<int64_t> widths;
  int64_t total = 0;
  for (int i = 0; i < n_in; ++i) {
    Tensor* x = check_handle(in[i]);
    BE_REQUIRE(x->rank == 2 && x->is_contiguous(), BE_E_SHAPE, "concat: contiguous 2-D inputs");
    BE_REQUIRE(x->shape[0] == check_handle(in[0])->shape[0], BE_E_SHAPE, "concat: row counts differ");
    BE_REQUIRE(x->dtype == check_handle(in[0])->dtype, BE_E_DTYPE, "concat: dtypes differ");
    xs.push_back(x);
    ptrs.push_back(x->data());
    widths.push_back(x->shape[1]);
    total += x->shape[1];
  }
  const int64_t rows = xs[0]->shape[0];
  TRef y = new_tensor({rows, total}, xs[0]->dtype);
  k::concat_cols(ptrs.data(), widths.data(), n_in, rows, y->data(), y->dtype, ctx().stream);
  Node* nd = nullptr;
  if (grad_enabled()) {
    bool any = false;
    for (Tensor* x : xs) any |= x->requires_grad;
    if (any) {
      nd = new Node();
      nd->name = "concat";
      nd->op = BE_OP_CONCAT;
      nd->vjp = vjp_concat;
      nd->seq = ctx().seq.fetch_add(1);
      for (Tensor* x : xs) {
        Edge e;
        if (x->requires_grad) {
          if (x->grad_fn) { e.kind = Edge::NODE; e.node = x->grad_fn; node_retain(x->grad_fn); e.output_nr = x->output_nr; }
          else { e.kind = Edge::LEAF; e.leaf = x; x->retain(); }
        }
        nd->edges.push_back(e);
      }
      for (int i = 0; i < n_in; ++i) nd->iattr[i] = widths[i];
    }
  }
  if (nd) { set_output(nd, y.get(), 0); finish_node(nd); }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

// ------------------------------------------------------------------ dispatch
void op_cnn(int op, const be_tensor* in, int n_in, const void* attrs, be_tensor* out, int n_out);

}  // namespace be

using namespace be;
extern "C" {

be_status be_op(int op_id, const be_tensor* in, int n_in, const void* attrs, be_tensor* out, int n_out) {
  BE_API_BEGIN
  BE_REQUIRE(ctx().inited, BE_E_NOT_INIT, "be_init() was not called");
  BE_REQUIRE(out != nullptr && n_out >= 1, BE_E_ARG, "be_op: need at least one output slot");
  for (int i = 0; i < n_out; ++i) out[i] = nullptr;
  switch (op_id) {
    case BE_OP_LINEAR: op_linear(in, n_in, attrs, out, n_out); break;
    case BE_OP_MATMUL: op_matmul(in, n_in, attrs, out, n_out); break;
    case BE_OP_ADD: op_add(in, n_in, attrs, out, n_out, 0); break;
    case BE_OP_ADD_RELU: op_add(in, n_in, attrs, out, n_out, 1); break;
    case BE_OP_MUL: op_mul(in, n_in, attrs, out, n_out); break;
    case BE_OP_RELU: op_relu(in, n_in, attrs, out, n_out); break;
    case BE_OP_SOFTMAX_XENT: op_softmax_xent(in, n_in, attrs, out, n_out); break;
    case BE_OP_BCE_LOGITS: op_bce(in, n_in, attrs, out, n_out); break;
    case BE_OP_SUM:
    case BE_OP_MEAN: op_sum(op_id, in, n_in, out); break;
    case BE_OP_RESHAPE: op_reshape(in, n_in, attrs, out); break;
    case BE_OP_CONCAT: op_concat(in, n_in, out); break;
    case BE_OP_CAST: {
      BE_REQUIRE(n_in == 1 && attrs, BE_E_ARG, "cast: 1 input + be_dtype");
      TRef y = cast_op(check_handle(in[0]), *reinterpret_cast<const be_dtype*>(attrs));
      out[0] = reinterpret_cast<be_tensor>(y.release());
      break;
    }
    case BE_OP_CONV2D:
    case BE_OP_MAXPOOL2D:
    case BE_OP_AVGPOOL_GLOBAL:
    case BE_OP_BATCHNORM2D:
    case BE_OP_EMBEDDING:
    case BE_OP_BN_CONV1X1: op_cnn(op_id, in, n_in, attrs, out, n_out); break;
    case BE_OP_DROPOUT:
    case BE_OP_CONV2D_DEPTHWISE: op_mobile(op_id, in, n_in, attrs, out, n_out); break;
    default: fail(BE_E_UNSUPPORTED, "unknown op id " + std::to_string(op_id));
  }
  BE_API_END
}

be_status be_fill_(be_tensor h, double v) {
  BE_API_BEGIN
  Tensor* t = check_handle(h);
  BE_REQUIRE(!(t->requires_grad && t->is_leaf() && grad_enabled()), BE_E_INPLACE_LEAF,
             "in-place write to a leaf that requires grad (use no-grad mode)");
  BE_REQUIRE(t->is_contiguous(), BE_E_NONCONTIG, "fill_: contiguous");
  k::fill(t->data(), t->numel(), t->dtype, v, ctx().stream);
  t->bump_version();
  BE_API_END
}

be_status be_copy_(be_tensor dst, be_tensor src) {
  BE_API_BEGIN
  Tensor* d = check_handle(dst);
  Tensor* s = check_handle(src);
  BE_REQUIRE(!(d->requires_grad && d->is_leaf() && grad_enabled()), BE_E_INPLACE_LEAF,
             "in-place write to a leaf that requires grad (use no-grad mode)");
  BE_REQUIRE(d->numel() == s->numel(), BE_E_SHAPE, "copy_: element counts differ");
  BE_REQUIRE(d->is_contiguous() && s->is_contiguous(), BE_E_NONCONTIG, "copy_: contiguous");
  k::cast(s->data(), s->dtype, d->data(), d->dtype, d->numel(), ctx().stream);
  d->bump_version();
  BE_API_END
}

be_status be_gemm(be_tensor A, int trans_a, be_tensor Bt, int trans_b, be_tensor D, be_tensor bias, int act,
                  float beta) {
  BE_API_BEGIN
  Tensor* a = check_handle(A);
  Tensor* b = check_handle(Bt);
  Tensor* d = check_handle(D);
  Tensor* bi = bias ? check_handle(bias) : nullptr;
  BE_REQUIRE(a->rank == 2 && b->rank == 2 && d->rank == 2, BE_E_SHAPE, "gemm: 2-D tensors");
  BE_REQUIRE(a->is_contiguous() && b->is_contiguous() && d->is_contiguous(), BE_E_NONCONTIG, "gemm: contiguous");
  BE_REQUIRE(a->dtype == b->dtype, BE_E_DTYPE, "gemm: A and B dtypes differ");
  const int64_t M = trans_a ? a->shape[1] : a->shape[0];
  const int64_t K = trans_a ? a->shape[0] : a->shape[1];
  const int64_t K2 = trans_b ? b->shape[1] : b->shape[0];
  const int64_t N = trans_b ? b->shape[0] : b->shape[1];
  BE_REQUIRE(K == K2 && d->shape[0] == M && d->shape[1] == N, BE_E_SHAPE, "gemm: shape mismatch");
  k::GemmDesc gd;
  gd.M = (int)M; gd.N = (int)N; gd.K = (int)K;
  gd.A = a->data(); gd.lda = a->shape[1]; gd.a_kmajor = !trans_a;
  gd.B = b->data(); gd.ldb = b->shape[1]; gd.b_kmajor = trans_b != 0;
  gd.ab = a->dtype; gd.D = d->data(); gd.ldd = N; gd.d = d->dtype; gd.beta = beta;
  gd.bias = bi ? bi->ptr<float>() : nullptr; gd.act = act;
  k::gemm(gd, ctx().stream);
  d->bump_version();
  BE_API_END
}

}  // extern "C"
