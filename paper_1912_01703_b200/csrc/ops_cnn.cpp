// ops_cnn.cpp — CNN / recommender operators: conv2d (as GEMMs on the tcgen05
// kernel), max / global-average pooling, batch norm (train), embedding.
//
// Conv2d (Listing 1 `nn.Conv2d`): NHWC
// activations x[N,H,W,C], KRSC weights w[K,R,S,C]:
//   fwd    Y[M=NPQ, K]   = cols(x)[M, RSC] · Wᵀ          (+bias, ReLU in the epilogue)
//   wgrad  dW[K, RSC]    = dYᵀ[K, M] · cols(x)[M, RSC]   (split-K, fp32)
//   dgrad  dcols[M, RSC] = dY[M, K] · W[K, RSC];  dx = col2im(dcols)
// 1×1 / stride-1 / pad-0 convolutions use x itself as the column matrix
// (no im2col, no col2im).  Operand majorness is chosen per GEMM so no
// transpose kernel ever runs.
#include "ops_common.h"

namespace be {

static k::ConvGeom conv_geom(const Tensor* x, const Tensor* w, int stride, int pad) {
  k::ConvGeom g;
  g.N = (int)x->shape[0]; g.H = (int)x->shape[1]; g.W = (int)x->shape[2]; g.C = (int)x->shape[3];
  g.K = (int)w->shape[0]; g.R = (int)w->shape[1]; g.S = (int)w->shape[2];
  g.stride = stride; g.pad = pad;
  g.P = (g.H + 2 * pad - g.R) / stride + 1;
  g.Q = (g.W + 2 * pad - g.S) / stride + 1;
  return g;
}
static bool is_pointwise(const k::ConvGeom& g) { return g.R == 1 && g.S == 1 && g.stride == 1 && g.pad == 0; }
static int64_t cols_ld(int64_t rsc, be_dtype dt) {
  const int64_t q = dt == BE_BF16 ? 8 : 4;  // 16-byte rows for TMA
  return (rsc + q - 1) / q * q;
}

// Column matrix of x (im2col or x itself); returns pointer + ld.
static TRef make_cols(Tensor* x, const k::ConvGeom& g, int64_t* ld) {
  const int64_t RSC = (int64_t)g.R * g.S * g.C;
  if (is_pointwise(g)) { *ld = g.C; return TRef(x, false); }
  const int64_t M = (int64_t)g.N * g.P * g.Q;
  *ld = cols_ld(RSC, x->dtype);
  TRef cols = new_tensor({M, *ld}, x->dtype);
  k::im2col(x->data(), cols->data(), *ld, g, x->dtype, ctx().stream);
  return cols;
}

static void vjp_conv(Node* n, GradSink& sink) {
  cudaStream_t s = ctx().stream;
  TRef hx, hw, hy;
  Tensor* x = unpack(n, 0, hx);
  Tensor* w = unpack(n, 1, hw);
  Tensor* y = unpack(n, 2, hy);
  const int stride = (int)n->iattr[0], pad = (int)n->iattr[1], act = (int)n->iattr[2];
  const bool has_b = n->iattr[3] != 0;
  const k::ConvGeom g = conv_geom(x, w, stride, pad);
  const be_dtype opd = x->dtype;
  const int64_t M = (int64_t)g.N * g.P * g.Q, K = g.K, RSC = (int64_t)g.R * g.S * g.C;
  TRef gz = contiguous_like(sink.upstream[0], opd);
  TRef dz;
  if (act) dz = new_tensor({M, K}, opd);
  else dz = gz;
  if (has_b && sink.needs(2)) {
    float bb;
    Tensor* db = sink.dest(2, &bb);
    k::relu_bwd_colsum(gz->data(), act ? y->data() : nullptr, dz->data(), M, K, opd, db->ptr<float>(), bb, act, s);
    sink.commit(2);
  } else if (act) {
    k::relu_bwd(gz->data(), y->data(), dz->data(), M * K, opd, 0.f, s);
  }
  gz = TRef();
  if (sink.needs(1)) {  // dW[K, RSC] = dzᵀ · cols
    float bw;
    Tensor* dw = sink.dest(1, &bw);
    k::GemmDesc gd;
    gd.M = (int)K; gd.N = (int)RSC; gd.K = (int)M;
    gd.A = dz->data(); gd.lda = K; gd.a_kmajor = false;
    gd.ab = opd; gd.D = dw->data(); gd.ldd = RSC; gd.d = dw->dtype; gd.beta = bw;
    gd.b_kmajor = false;
    TRef cols;
    // variant 0: B = im2col(x) read in place by TMA im2col; variant 1:
    // materialised columns + GEMM.  TMA im2col moves ~0.13 pixel/cycle/SM,
    // so which one wins depends on the shape: autotuned per shape.
    // variant 2: A = dY and B = x read as shifted 4-D tiles (blocks of whole
    // output rows; TMA zero-fills the padding) — tiled TMA, no im2col mode
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int variant = 1, gidx = -1;
    if (!is_pointwise(g) && opd == BE_BF16 && g.C % 64 == 0 && (K * 2) % 16 == 0) {
      char key[160];
      snprintf(key, sizeof(key), "conv_wgrad:%d,%d,%d,%d,%d,%d,%d,%d,%d", g.N, g.H, g.W, g.C, g.K, g.R, g.S,
               g.stride, g.pad);
      static const int shift_on = [] { const char* e = getenv("BE_WGRAD_SHIFT"); return e ? atoi(e) : 1; }();
      const bool shift_ok = shift_on && g.Q <= 64 && g.K % 8 == 0 && g.stride <= 2;
      // variant 3: shared input patch per tile, shifted UMMA operands (stride 1, C = K = 64)
      const bool patch_ok = shift_ok && g.stride == 1 && ((g.C == 64 && g.K % 64 == 0 && g.K <= 256) || (g.C == 128 && g.K == 128)) &&
                            dw->dtype == BE_F32 && g.R * g.S <= 64 && g.Q + g.S - 1 <= 128;
      static const int force = [] { const char* e = getenv("BE_WGRAD_VARIANT"); return e ? atoi(e) : -1; }();
      int nv = patch_ok ? 4 : (shift_ok ? 3 : 2);
      // last candidate: the im2col slice gathered into shared memory (conv_wgrad_gather)
      if (dw->dtype == BE_F32 && g.K % 128 == 0 && (RSC % 128) == 0 && (bw == 0.f || bw == 1.f)) gidx = nv++;
      if (force >= 0 && force < nv) variant = force;  // probes / tests
      else variant = tune_choose(key, nv, 0, &e0, &e1);
    }
    if (e0) cudaEventRecord(e0, s);
    if (g.C == 8 && opd == BE_BF16 && !e0 && k::conv_wgrad_stem(dz->data(), x->data(), dw->data(), dw->dtype, g, bw, s)) {
      sink.commit(1);
    } else if (variant == gidx && k::conv_wgrad_gather(dz->data(), x->data(), dw->data(), dw->dtype, g, bw, s)) {
      if (e1) cudaEventRecord(e1, s);
      sink.commit(1);
    } else if (variant == 3 && gidx != 3 &&
               k::conv_wgrad_patch(dz->data(), x->data(), dw->data(), dw->dtype, g, bw, s)) {
      if (e1) cudaEventRecord(e1, s);
      sink.commit(1);
    } else {
    if (variant == gidx) variant = 1;
    if (variant == 3) variant = 1;
    if (variant == 0 || variant == 2) {
      gd.conv_x = x->data();
      gd.conv_g = g;
      gd.conv_shift = variant == 2;
    } else {
      int64_t ldc;
      cols = make_cols(x, g, &ldc);
      gd.B = cols->data(); gd.ldb = ldc;
    }
    k::gemm(gd, s);
    if (e1) cudaEventRecord(e1, s);
    sink.commit(1);
    }
  }
  if (sink.needs(0)) {
    float bx;
    Tensor* dx = sink.dest(0, &bx);
    BE_REQUIRE(dx->dtype == opd, BE_E_DTYPE, "conv dgrad dtype");
    // stride-1 dgrad is itself a convolution: dX = conv(dY, W', pad R−1−pad),
    // W'[c,r,s,k] = W[k,R−1−r,S−1−s,c] → implicit GEMM, no dcols / col2im
    if (!is_pointwise(g) && g.stride == 1 && opd == BE_BF16 && g.K % 64 == 0 && g.C % 16 == 0 &&
        g.pad <= g.R - 1 && g.pad <= g.S - 1) {
      // W'[c, r, s, k] = W[k, R−1−r, S−1−s, c] read in place (MN-major B operand): no flipped copy
      const int bw[6] = {g.R - 1, -1, g.S - 1, -1, g.S, (int)RSC};
      k::ConvGeom gt;
      gt.N = g.N; gt.H = g.P; gt.W = g.Q; gt.C = g.K; gt.K = g.C; gt.R = g.R; gt.S = g.S;
      gt.stride = 1; gt.pad = g.R - 1 - g.pad;
      gt.P = (gt.H + 2 * gt.pad - gt.R) + 1;
      gt.Q = (gt.W + 2 * (g.S - 1 - g.pad) - gt.S) + 1;
      if (gt.P == g.H && gt.Q == g.W && g.R == g.S &&
          k::conv_implicit(dz->data(), w->data(), dx->data(), gt, opd, nullptr, 0, bx, s, nullptr, nullptr, bw)) {
        sink.commit(0);
        return;
      }
    }
    // stride ≥ 2: st² stride-1 phase convolutions stored straight into dx
    if (g.stride >= 2 && opd == BE_BF16 && k::conv_dgrad_phases(dz->data(), w->data(), dx->data(), g, bx, s)) {
      sink.commit(0);
      return;
    }
    k::GemmDesc gd;
    gd.M = (int)M; gd.N = (int)RSC; gd.K = (int)K;
    gd.A = dz->data(); gd.lda = K; gd.a_kmajor = true;
    gd.B = w->data(); gd.ldb = RSC; gd.b_kmajor = false;
    gd.ab = opd;
    if (is_pointwise(g)) {
      gd.D = dx->data(); gd.ldd = RSC; gd.d = opd; gd.beta = bx;
      k::gemm(gd, s);
    } else {
      const int64_t ldc = cols_ld(RSC, opd);
      TRef dcols = new_tensor({M, ldc}, opd);
      gd.D = dcols->data(); gd.ldd = ldc; gd.d = opd; gd.beta = 0.f;
      k::gemm(gd, s);
      k::col2im(dcols->data(), ldc, dx->data(), g, opd, bx, s);
    }
    sink.commit(0);
  }
}

static void op_conv(const be_tensor* in, int n_in, const void* attrs, be_tensor* out) {
  BE_REQUIRE(n_in == 2 || n_in == 3, BE_E_ARG, "conv2d: x, w[, b]");
  BE_REQUIRE(attrs, BE_E_ARG, "conv2d: be_conv_attrs required");
  const be_conv_attrs a = *reinterpret_cast<const be_conv_attrs*>(attrs);
  Tensor* x0 = check_handle(in[0]);
  Tensor* w0 = check_handle(in[1]);
  Tensor* b = n_in == 3 && in[2] ? check_handle(in[2]) : nullptr;
  BE_REQUIRE(x0->rank == 4 && w0->rank == 4, BE_E_SHAPE, "conv2d: x NHWC[N,H,W,C], w KRSC[K,R,S,C]");
  BE_REQUIRE(x0->shape[3] == w0->shape[3], BE_E_SHAPE, "conv2d: channel counts differ");
  BE_REQUIRE(a.stride >= 1 && a.pad >= 0, BE_E_ARG, "conv2d: stride >= 1, pad >= 0");
  BE_REQUIRE(x0->shape[1] + 2 * a.pad >= w0->shape[1] && x0->shape[2] + 2 * a.pad >= w0->shape[2], BE_E_SHAPE,
             "conv2d: kernel larger than padded input");
  BE_REQUIRE(!b || (b->rank == 1 && b->shape[0] == w0->shape[0] && b->dtype == BE_F32), BE_E_SHAPE,
             "conv2d: bias f32 [K]");
  BE_REQUIRE(x0->is_contiguous(), BE_E_NONCONTIG, "conv2d: contiguous input");
  TRef x = act_operand(x0);
  Tensor* w = weight_operand(w0);
  const k::ConvGeom g = conv_geom(x.get(), w, a.stride, a.pad);
  const int64_t M = (int64_t)g.N * g.P * g.Q, RSC = (int64_t)g.R * g.S * g.C;
  const be_dtype od = (a.out_f32 || ctx().compute == BE_F32) ? BE_F32 : BE_BF16;
  TRef y = new_tensor({g.N, g.P, g.Q, g.K}, od);
  // BN statistics from the epilogue: zeroed partial rows for up to 4·num_sms parts
  TRef stats;
  int parts = 0;
  static const bool stats_on = [] { const char* e = getenv("BE_BN_STATS"); return !(e && e[0] == '0'); }();
  // only where the epilogue has slack: reduction depth R·S·C ≥ output channels
  // (for K-light, N-heavy convs — the 1×1 expansions — the epilogue is the
  // bottleneck and the extra column reduction costs more than the BN pass it saves)
  static const bool stats_all = [] { const char* e = getenv("BE_BN_STATS_ALL"); return e && e[0] == '1'; }();
  if (stats_on && a.bn_stats && !b && !a.act && M > 0 && (RSC >= g.K || stats_all)) {
    const int64_t cap = (int64_t)ctx().num_sms * 4;
    stats = new_tensor({2 * cap * g.K}, BE_F32);
    BE_CHECK_CUDA(cudaMemsetAsync(stats->data(), 0, sizeof(float) * 2 * cap * g.K, ctx().stream));
  }
  float* sp = stats ? stats->ptr<float>() : nullptr;
  if (is_pointwise(g) || x->dtype != BE_BF16 ||
      !k::conv_implicit(x->data(), w->data(), y->data(), g, od, b ? b->ptr<float>() : nullptr, a.act, 0.f,
                        ctx().stream, sp, &parts)) {
    int64_t ldc;
    TRef cols = make_cols(x.get(), g, &ldc);
    k::GemmDesc gd;
    gd.M = (int)M; gd.N = g.K; gd.K = (int)RSC;
    gd.A = cols->data(); gd.lda = ldc; gd.a_kmajor = true;
    gd.B = w->data(); gd.ldb = RSC; gd.b_kmajor = true;
    gd.ab = x->dtype; gd.D = y->data(); gd.ldd = g.K; gd.d = od;
    gd.bias = b ? b->ptr<float>() : nullptr; gd.act = a.act;
    gd.stats = sp; gd.stats_parts = &parts;
    k::gemm(gd, ctx().stream);
  }
  if (parts > 0) {
    y->bn_stats = stats.release();
    y->bn_stats_parts = parts;
    y->bn_stats_version = y->version();
  }
  Node* n = new_node("conv2d", BE_OP_CONV2D, vjp_conv, {x.get(), w0, b});
  if (n) {
    save(n, x.get());
    save(n, w);
    save(n, a.act ? y.get() : nullptr);
    n->iattr[0] = a.stride; n->iattr[1] = a.pad; n->iattr[2] = a.act; n->iattr[3] = b != nullptr;
    set_output(n, y.get(), 0);
    finish_node(n);
  }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

// ------------------------------------------------------------------ pooling
static void vjp_maxpool(Node* n, GradSink& sink) {
  TRef ham;
  Tensor* am = unpack(n, 0, ham);
  k::ConvGeom g;
  g.N = (int)n->iattr[3]; g.H = (int)n->iattr[4]; g.W = (int)n->iattr[5]; g.C = (int)n->iattr[6];
  g.R = g.S = (int)n->iattr[0]; g.stride = (int)n->iattr[1]; g.pad = (int)n->iattr[2];
  g.P = (g.H + 2 * g.pad - g.R) / g.stride + 1;
  g.Q = (g.W + 2 * g.pad - g.S) / g.stride + 1;
  g.K = g.C;
  float beta;
  Tensor* dx = sink.dest(0, &beta);
  if (!dx) return;
  TRef gz = contiguous_like(sink.upstream[0], dx->dtype);
  k::maxpool_bwd(gz->data(), am->ptr<uint8_t>(), dx->data(), g, dx->dtype, beta, ctx().stream);
  sink.commit(0);
}
static void op_maxpool(const be_tensor* in, int n_in, const void* attrs, be_tensor* out, int n_out) {
  BE_REQUIRE(n_in == 1 && attrs, BE_E_ARG, "maxpool2d: x + be_pool_attrs");
  const be_pool_attrs a = *reinterpret_cast<const be_pool_attrs*>(attrs);
  Tensor* x = check_handle(in[0]);
  BE_REQUIRE(x->rank == 4 && x->is_contiguous(), BE_E_SHAPE, "maxpool2d: contiguous NHWC input");
  BE_REQUIRE(a.k >= 1 && a.k * a.k <= 255 && a.stride >= 1 && a.pad >= 0 && a.pad <= a.k / 2, BE_E_ARG,
             "maxpool2d: bad window");
  k::ConvGeom g;
  g.N = (int)x->shape[0]; g.H = (int)x->shape[1]; g.W = (int)x->shape[2]; g.C = (int)x->shape[3];
  g.R = g.S = a.k; g.stride = a.stride; g.pad = a.pad; g.K = g.C;
  g.P = (g.H + 2 * a.pad - a.k) / a.stride + 1;
  g.Q = (g.W + 2 * a.pad - a.k) / a.stride + 1;
  BE_REQUIRE(g.P > 0 && g.Q > 0, BE_E_SHAPE, "maxpool2d: window larger than input");
  TRef y = new_tensor({g.N, g.P, g.Q, g.C}, x->dtype);
  TRef am = new_tensor({g.N, g.P, g.Q, g.C}, BE_U8);
  k::maxpool_fwd(x->data(), y->data(), am->ptr<uint8_t>(), g, x->dtype, ctx().stream);
  Node* n = new_node("maxpool2d", BE_OP_MAXPOOL2D, vjp_maxpool, {x});
  if (n) {
    save(n, am.get());
    n->iattr[0] = a.k; n->iattr[1] = a.stride; n->iattr[2] = a.pad;
    n->iattr[3] = g.N; n->iattr[4] = g.H; n->iattr[5] = g.W; n->iattr[6] = g.C;
    set_output(n, y.get(), 0);
    finish_node(n);
  }
  out[0] = reinterpret_cast<be_tensor>(y.release());
  if (n_out > 1) out[1] = reinterpret_cast<be_tensor>(am.release());
}

static void vjp_avgpool(Node* n, GradSink& sink) {
  float beta;
  Tensor* dx = sink.dest(0, &beta);
  if (!dx) return;
  TRef gz = contiguous_like(sink.upstream[0], dx->dtype);
  const int N = (int)dx->shape[0], HW = (int)(dx->shape[1] * dx->shape[2]), C = (int)dx->shape[3];
  k::avgpool_bwd(gz->data(), dx->data(), N, HW, C, dx->dtype, beta, ctx().stream);
  sink.commit(0);
}
static void op_avgpool(const be_tensor* in, int n_in, be_tensor* out) {
  BE_REQUIRE(n_in == 1, BE_E_ARG, "avgpool_global: 1 input");
  Tensor* x = check_handle(in[0]);
  BE_REQUIRE(x->rank == 4 && x->is_contiguous(), BE_E_SHAPE, "avgpool_global: contiguous NHWC");
  const int N = (int)x->shape[0], HW = (int)(x->shape[1] * x->shape[2]), C = (int)x->shape[3];
  BE_REQUIRE(HW > 0, BE_E_EMPTY_REDUCTION, "avgpool_global: empty plane");
  TRef y = new_tensor({(int64_t)N, (int64_t)C}, x->dtype);
  k::avgpool_fwd(x->data(), y->data(), N, HW, C, x->dtype, ctx().stream);
  Node* n = new_node("avgpool_global", BE_OP_AVGPOOL_GLOBAL, vjp_avgpool, {x});
  if (n) { set_output(n, y.get(), 0); finish_node(n); }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

// ------------------------------------------------------------------ batch norm (train)
static void vjp_bn(Node* n, GradSink& sink) {
  cudaStream_t s = ctx().stream;
  TRef hx, hmean, hinv, hg, hy, hb;
  Tensor* x = unpack(n, 0, hx);
  Tensor* mean = unpack(n, 1, hmean);
  Tensor* inv = unpack(n, 2, hinv);
  Tensor* gamma = unpack(n, 3, hg);
  Tensor* y = unpack(n, 4, hy);
  Tensor* bshift = unpack(n, 5, hb);  // β: the ReLU mask is recomputed from x
  const int act = (int)n->iattr[0];
  const bool residual = n->iattr[1] != 0;
  const int C = (int)x->shape[3];
  const int64_t rows = x->numel() / C;
  TRef gz = contiguous_like(sink.upstream[0], x->dtype);
  // y = relu(bn(x) + r): g = dy·1[y > 0] is both r's gradient and the BN's
  // upstream; bn_bwd writes it (fused into its reduction pass)
  TRef gmask;
  if (residual && act) gmask = new_tensor(x->shape, x->rank, x->dtype);
  // dgamma / dbeta accumulate flags must agree: compute into temps when they differ
  float bg = 0.f, bb = 0.f;
  Tensor* dg = sink.needs(1) ? sink.dest(1, &bg) : nullptr;
  Tensor* db = sink.needs(2) ? sink.dest(2, &bb) : nullptr;
  TRef tg, tb;
  float gb_beta = 0.f;
  if (dg && db && bg == bb) gb_beta = bg;
  else {
    if (dg && bg != 0.f) { tg = new_tensor({C}, BE_F32); }
    if (db && bb != 0.f) { tb = new_tensor({C}, BE_F32); }
  }
  TRef part = new_tensor({(int64_t)k::bn_partial_floats(rows, C)}, BE_F32);
  float bx = 0.f;
  Tensor* dx = sink.needs(0) ? sink.dest(0, &bx) : nullptr;
  TRef dgs = dg ? TRef() : new_tensor({C}, BE_F32);
  TRef dbs = db ? TRef() : new_tensor({C}, BE_F32);
  float* dgp = tg ? tg->ptr<float>() : (dg ? dg->ptr<float>() : dgs->ptr<float>());
  float* dbp = tb ? tb->ptr<float>() : (db ? db->ptr<float>() : dbs->ptr<float>());
  const int bact = residual ? 0 : act;  // with a residual the mask is already in gz
  const bool bits = n->iattr[2] != 0;  // saved[4] is the 1-bit residual mask
  k::bn_bwd(gz->data(), x->data(), bact ? y->data() : nullptr, bact, dx ? dx->data() : nullptr, rows, C, x->dtype,
            mean->ptr<float>(), inv->ptr<float>(), gamma->ptr<float>(), dgp, dbp, gb_beta, bx, part->ptr<float>(), s,
            bact ? bshift->ptr<float>() : nullptr, gmask && !bits ? y->data() : nullptr,
            gmask ? gmask->data() : nullptr, gmask && bits ? y->ptr<uint8_t>() : nullptr);
  if (gmask) gz = std::move(gmask);  // sole reference: the shortcut adopts it without a copy
  if (tg) k::axpby(tg->data(), BE_F32, dg->data(), BE_F32, C, 1.f, 1.f, s);
  if (tb) k::axpby(tb->data(), BE_F32, db->data(), BE_F32, C, 1.f, 1.f, s);
  if (dx) sink.commit(0);
  if (dg) sink.commit(1);
  if (db) sink.commit(2);
  // the residual's gradient (last edge) is g itself: handed over without a copy
  // when nothing else has been accumulated for it yet
  if (residual && sink.needs((int)n->edges.size() - 1)) sink.give((int)n->edges.size() - 1, std::move(gz));
}
// ------------------------------------------------------------------ ResNet projection block output
// y = act(bn(x) + bn_r(x_r)) in ONE apply pass (be_bn_attrs.residual = 2; the
// residual branch's BN — the projection shortcut's, act 0 — is applied on the
// fly instead of being written and re-read as a residual tensor).  Both BNs
// keep their own statistics / running statistics.  Backward: the main BN's
// backward with the residual 1-bit mask writes g = dy·1[y > 0], which is then
// the upstream of the residual BN's backward (exactly the unfused pair's
// gradients: batchnorm2d(x_r) → batchnorm2d(x, residual) composed).
static void vjp_bn_add_bn(Node* n, GradSink& sink) {
  cudaStream_t s = ctx().stream;
  TRef hx, hmean, hinv, hg, hbits, hb, hxr, hmr, hir, hgr;
  Tensor* x = unpack(n, 0, hx);
  Tensor* mean = unpack(n, 1, hmean);
  Tensor* inv = unpack(n, 2, hinv);
  Tensor* gamma = unpack(n, 3, hg);
  Tensor* bits = unpack(n, 4, hbits);
  Tensor* beta = unpack(n, 5, hb);
  Tensor* xr = unpack(n, 6, hxr);
  Tensor* mr = unpack(n, 7, hmr);
  Tensor* ir = unpack(n, 8, hir);
  Tensor* gr = unpack(n, 9, hgr);
  (void)beta;
  const int act = (int)n->iattr[0];
  const int C = (int)x->shape[3];
  const int64_t rows = x->numel() / C;
  TRef gz = contiguous_like(sink.upstream[0], x->dtype);
  TRef gmask = act ? new_tensor(x->shape, x->rank, x->dtype) : TRef();
  // one BN backward: upstream u, input xb → dx into edge ex (gamma/beta edges eg, eb)
  auto bwd = [&](Tensor* u, Tensor* xb, Tensor* mb, Tensor* ib, Tensor* gb, int ex, int eg, int eb, bool first) {
    float bg = 0.f, bbt = 0.f;
    Tensor* dg = sink.needs(eg) ? sink.dest(eg, &bg) : nullptr;
    Tensor* db = sink.needs(eb) ? sink.dest(eb, &bbt) : nullptr;
    TRef tg, tb;
    float gb_beta = 0.f;
    if (dg && db && bg == bbt) gb_beta = bg;
    else {
      if (dg && bg != 0.f) tg = new_tensor({C}, BE_F32);
      if (db && bbt != 0.f) tb = new_tensor({C}, BE_F32);
    }
    TRef part = new_tensor({(int64_t)k::bn_partial_floats(rows, C)}, BE_F32);
    float bx = 0.f;
    Tensor* dx = sink.needs(ex) ? sink.dest(ex, &bx) : nullptr;
    TRef dgs = dg ? TRef() : new_tensor({C}, BE_F32);
    TRef dbs = db ? TRef() : new_tensor({C}, BE_F32);
    float* dgp = tg ? tg->ptr<float>() : (dg ? dg->ptr<float>() : dgs->ptr<float>());
    float* dbp = tb ? tb->ptr<float>() : (db ? db->ptr<float>() : dbs->ptr<float>());
    const bool mask = first && act;
    k::bn_bwd(u->data(), xb->data(), nullptr, 0, dx ? dx->data() : nullptr, rows, C, xb->dtype, mb->ptr<float>(),
              ib->ptr<float>(), gb->ptr<float>(), dgp, dbp, gb_beta, bx, part->ptr<float>(), s, nullptr, nullptr,
              mask ? gmask->data() : nullptr, mask ? bits->ptr<uint8_t>() : nullptr);
    if (tg) k::axpby(tg->data(), BE_F32, dg->data(), BE_F32, C, 1.f, 1.f, s);
    if (tb) k::axpby(tb->data(), BE_F32, db->data(), BE_F32, C, 1.f, 1.f, s);
    if (dx) sink.commit(ex);
    if (dg) sink.commit(eg);
    if (db) sink.commit(eb);
  };
  bwd(gz.get(), x, mean, inv, gamma, 0, 1, 2, true);
  if (gmask) gz = std::move(gmask);
  bwd(gz.get(), xr, mr, ir, gr, 3, 4, 5, false);
}

static void op_bn_add_bn(const be_tensor* in, int n_in, const be_bn_attrs& a, int nb, be_tensor* out) {
  Tensor* x = check_handle(in[0]);
  Tensor* gamma = check_handle(in[1]);
  Tensor* beta = check_handle(in[2]);
  Tensor* rm = nb == 5 && in[3] ? check_handle(in[3]) : nullptr;
  Tensor* rv = nb == 5 && in[4] ? check_handle(in[4]) : nullptr;
  Tensor* xr = check_handle(in[nb]);
  Tensor* gr = check_handle(in[nb + 1]);
  Tensor* br = check_handle(in[nb + 2]);
  Tensor* rmr = in[nb + 3] ? check_handle(in[nb + 3]) : nullptr;
  Tensor* rvr = in[nb + 4] ? check_handle(in[nb + 4]) : nullptr;
  BE_REQUIRE(a.act == 0 || a.act == 1, BE_E_ARG, "batchnorm2d (residual bn): act 0 or 1");
  BE_REQUIRE(x->rank == 4 && x->is_contiguous() && xr->rank == 4 && xr->is_contiguous(), BE_E_SHAPE,
             "batchnorm2d: contiguous NHWC inputs");
  for (int d = 0; d < 4; ++d) BE_REQUIRE(xr->shape[d] == x->shape[d], BE_E_SHAPE, "batchnorm2d: residual shape");
  BE_REQUIRE(xr->dtype == x->dtype && x->dtype == BE_BF16, BE_E_DTYPE, "batchnorm2d (residual bn): bf16 inputs");
  const int C = (int)x->shape[3];
  const int64_t rows = x->numel() / std::max(C, 1);
  BE_REQUIRE(rows > 0, BE_E_EMPTY_REDUCTION, "batchnorm2d: empty batch");
  BE_REQUIRE(gamma->numel() == C && beta->numel() == C && gr->numel() == C && br->numel() == C, BE_E_SHAPE,
             "batchnorm2d: gamma/beta f32 [C]");
  BE_REQUIRE(k::bn_mask_bits_ok(x->data(), x->data(), xr->data(), rows, C, x->dtype), BE_E_UNSUPPORTED,
             "batchnorm2d (residual bn): needs the stream path (C % 8 == 0, C <= 2048, 16-B aligned)");
  cudaStream_t s = ctx().stream;
  auto stats = [&](Tensor* t, Tensor* m, Tensor* v, TRef& mean, TRef& inv) {
    mean = new_tensor({C}, BE_F32); inv = new_tensor({C}, BE_F32);
    TRef part = new_tensor({(int64_t)k::bn_partial_floats(rows, C)}, BE_F32);
    if (t->bn_stats && t->bn_stats_version == t->version() && t->bn_stats->numel() >= 2LL * t->bn_stats_parts * C)
      k::bn_stats_from_partials(t->bn_stats->ptr<float>(), t->bn_stats_parts, rows, C, a.eps, mean->ptr<float>(),
                                inv->ptr<float>(), m ? m->ptr<float>() : nullptr, v ? v->ptr<float>() : nullptr,
                                a.momentum, s);
    else
      k::bn_stats(t->data(), rows, C, t->dtype, a.eps, mean->ptr<float>(), inv->ptr<float>(), part->ptr<float>(),
                  m ? m->ptr<float>() : nullptr, v ? v->ptr<float>() : nullptr, a.momentum, s);
    if (m) m->bump_version();
    if (v) v->bump_version();
  };
  TRef mr, ir, mean, inv;
  stats(xr, rmr, rvr, mr, ir);
  stats(x, rm, rv, mean, inv);
  TRef y = new_tensor(x->shape, x->rank, x->dtype);
  const bool want_grad = grad_enabled() && (x->requires_grad || gamma->requires_grad || beta->requires_grad ||
                                            xr->requires_grad || gr->requires_grad || br->requires_grad);
  TRef bits = a.act && want_grad ? new_tensor({rows * (C / 8)}, BE_U8) : TRef();
  k::bn_apply_stream2(reinterpret_cast<const uint16_t*>(x->data()), reinterpret_cast<uint16_t*>(y->data()), rows, C,
                      mean->ptr<float>(), inv->ptr<float>(), gamma->ptr<float>(), beta->ptr<float>(), a.act,
                      reinterpret_cast<const uint16_t*>(xr->data()), mr->ptr<float>(), ir->ptr<float>(),
                      gr->ptr<float>(), br->ptr<float>(), s, bits ? bits->ptr<uint8_t>() : nullptr);
  Node* n = new_node("batchnorm2d_add_bn", BE_OP_BATCHNORM2D, vjp_bn_add_bn, {x, gamma, beta, xr, gr, br});
  if (n) {
    save(n, x); save(n, mean.get()); save(n, inv.get()); save(n, gamma); save(n, bits ? bits.get() : nullptr);
    save(n, beta); save(n, xr); save(n, mr.get()); save(n, ir.get()); save(n, gr);
    n->iattr[0] = a.act;
    set_output(n, y.get(), 0);
    finish_node(n);
  }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

static void op_bn(const be_tensor* in, int n_in, const void* attrs, be_tensor* out) {
  be_bn_attrs a{1e-5f, 0.1f, 0, 0};
  if (attrs) a = *reinterpret_cast<const be_bn_attrs*>(attrs);
  BE_REQUIRE(a.residual >= 0 && a.residual <= 2, BE_E_ARG, "batchnorm2d: residual 0, 1 or 2");
  const int nb = n_in - (a.residual == 1 ? 1 : (a.residual == 2 ? 5 : 0));
  BE_REQUIRE(nb == 3 || nb == 5, BE_E_ARG, "batchnorm2d: x, gamma, beta[, running_mean, running_var][, residual]");
  Tensor* x = check_handle(in[0]);
  Tensor* gamma = check_handle(in[1]);
  Tensor* beta = check_handle(in[2]);
  Tensor* rm = nb == 5 && in[3] ? check_handle(in[3]) : nullptr;
  Tensor* rv = nb == 5 && in[4] ? check_handle(in[4]) : nullptr;
  if (a.residual == 2) { op_bn_add_bn(in, n_in, a, nb, out); return; }
  Tensor* res = a.residual ? check_handle(in[n_in - 1]) : nullptr;
  BE_REQUIRE(a.act >= 0 && a.act <= 2, BE_E_ARG, "batchnorm2d: act 0 (none), 1 (ReLU) or 2 (ReLU6)");
  BE_REQUIRE(!(res && a.act == 2), BE_E_UNSUPPORTED, "batchnorm2d: ReLU6 after a residual add");
  BE_REQUIRE(x->rank == 4 && x->is_contiguous(), BE_E_SHAPE, "batchnorm2d: contiguous NHWC input");
  if (res) {
    BE_REQUIRE(res->rank == 4 && res->is_contiguous(), BE_E_SHAPE, "batchnorm2d: contiguous residual");
    for (int d = 0; d < 4; ++d) BE_REQUIRE(res->shape[d] == x->shape[d], BE_E_SHAPE, "batchnorm2d: residual shape");
    BE_REQUIRE(res->dtype == x->dtype, BE_E_DTYPE, "batchnorm2d: residual dtype must match x");
  }
  const int C = (int)x->shape[3];
  const int64_t rows = x->numel() / std::max(C, 1);
  BE_REQUIRE(rows > 0, BE_E_EMPTY_REDUCTION, "batchnorm2d: empty batch");
  BE_REQUIRE(gamma->numel() == C && beta->numel() == C && gamma->dtype == BE_F32 && beta->dtype == BE_F32,
             BE_E_SHAPE, "batchnorm2d: gamma/beta f32 [C]");
  cudaStream_t s = ctx().stream;
  TRef mean = new_tensor({C}, BE_F32), inv = new_tensor({C}, BE_F32);
  TRef part = new_tensor({(int64_t)k::bn_partial_floats(rows, C)}, BE_F32);
  if (x->bn_stats && x->bn_stats_version == x->version() && x->bn_stats->numel() >= 2LL * x->bn_stats_parts * C) {
    // statistics already produced by the producing conv's epilogue
    k::bn_stats_from_partials(x->bn_stats->ptr<float>(), x->bn_stats_parts, rows, C, a.eps, mean->ptr<float>(),
                              inv->ptr<float>(), rm ? rm->ptr<float>() : nullptr, rv ? rv->ptr<float>() : nullptr,
                              a.momentum, s);
  } else {
    k::bn_stats(x->data(), rows, C, x->dtype, a.eps, mean->ptr<float>(), inv->ptr<float>(), part->ptr<float>(),
                rm ? rm->ptr<float>() : nullptr, rv ? rv->ptr<float>() : nullptr, a.momentum, s);
  }
  if (rm) rm->bump_version();
  if (rv) rv->bump_version();
  TRef y = new_tensor(x->shape, x->rank, x->dtype);
  // residual block output relu(bn(x) + r): the backward needs only the sign of
  // y — a 1-bit mask written by the apply pass (1/16 of y's bytes to re-read)
  const bool want_grad = grad_enabled() && (x->requires_grad || gamma->requires_grad || beta->requires_grad ||
                                            (res && res->requires_grad));
  TRef bits;
  if (res && a.act == 1 && want_grad && k::bn_mask_bits_ok(x->data(), y->data(), res->data(), rows, C, x->dtype))
    bits = new_tensor({rows * (C / 8)}, BE_U8);
  k::bn_apply(x->data(), y->data(), rows, C, x->dtype, mean->ptr<float>(), inv->ptr<float>(), gamma->ptr<float>(),
              beta->ptr<float>(), a.act, s, res ? res->data() : nullptr, bits ? bits->ptr<uint8_t>() : nullptr,
              /*early: the statistics kernels just launched write neither x nor res*/ 1);
  Node* n = res ? new_node("batchnorm2d", BE_OP_BATCHNORM2D, vjp_bn, {x, gamma, beta, res})
                : new_node("batchnorm2d", BE_OP_BATCHNORM2D, vjp_bn, {x, gamma, beta});
  if (n) {
    save(n, x); save(n, mean.get()); save(n, inv.get()); save(n, gamma);
    save(n, bits ? bits.get() : (a.act ? y.get() : nullptr));
    save(n, beta);
    n->iattr[0] = a.act;
    n->iattr[1] = res != nullptr;
    n->iattr[2] = bits ? 1 : 0;
    set_output(n, y.get(), 0);
    finish_node(n);
  }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

// ------------------------------------------------------------------ batch norm → 1×1 conv (fused apply)
// y = conv1x1(act(bn(x)), w) with the BN's normalise + activation applied to
// the GEMM's A tile in shared memory ("normalise + ReLU in the
// next conv's operand load") — the BN output is never written to HBM; the
// backward recomputes it inside the weight-gradient GEMM's B tile and the BN
// backward recomputes the activation mask from x (oracle: batchnorm2d → relu
// → conv2d composed, oracle/ops.py).
static void vjp_bn_conv(Node* n, GradSink& sink) {
  cudaStream_t s = ctx().stream;
  TRef hx, hmean, hinv, hg, hb, hw;
  Tensor* x = unpack(n, 0, hx);
  Tensor* mean = unpack(n, 1, hmean);
  Tensor* inv = unpack(n, 2, hinv);
  Tensor* gamma = unpack(n, 3, hg);
  Tensor* beta = unpack(n, 4, hb);
  Tensor* w = unpack(n, 5, hw);  // bf16 [K, 1, 1, C]
  const int act = (int)n->iattr[0];
  const int C = (int)x->shape[3], K = (int)w->shape[0];
  const int64_t rows = x->numel() / C;
  TRef gz = contiguous_like(sink.upstream[0], BE_BF16);
  // 1. dW[K, C] = dYᵀ · act(bn(x))  (the BN output rebuilt in the B tile)
  if (sink.needs(3)) {
    float bw;
    Tensor* dw = sink.dest(3, &bw);
    TRef tmp;
    if (bw != 0.f) tmp = new_tensor({(int64_t)K, (int64_t)C}, BE_F32);
    k::GemmDesc gd;
    gd.M = K; gd.N = C; gd.K = (int)rows;
    gd.A = gz->data(); gd.lda = K; gd.a_kmajor = false;
    gd.B = x->data(); gd.ldb = C; gd.b_kmajor = false;
    gd.ab = BE_BF16; gd.D = tmp ? tmp->data() : dw->data(); gd.ldd = C; gd.d = BE_F32;
    gd.xf_op = 2; gd.xf_act = act; gd.xf_C = C;
    gd.xf_mean = mean->ptr<float>(); gd.xf_invstd = inv->ptr<float>();
    gd.xf_gamma = gamma->ptr<float>(); gd.xf_beta = beta->ptr<float>();
    k::gemm(gd, s);
    if (tmp) k::axpby(tmp->data(), BE_F32, dw->data(), BE_F32, (int64_t)K * C, 1.f, 1.f, s);
    sink.commit(3);
  }
  if (!sink.needs(0) && !sink.needs(1) && !sink.needs(2)) return;
  // 2. dZ[rows, C] = dY · W  (gradient w.r.t. the BN output)
  TRef dz = new_tensor({rows, (int64_t)C}, BE_BF16);
  {
    k::GemmDesc gd;
    gd.M = (int)rows; gd.N = C; gd.K = K;
    gd.A = gz->data(); gd.lda = K; gd.a_kmajor = true;
    gd.B = w->data(); gd.ldb = C; gd.b_kmajor = false;
    gd.ab = BE_BF16; gd.D = dz->data(); gd.ldd = C; gd.d = BE_BF16;
    k::gemm(gd, s);
  }
  gz = TRef();
  // 3. the BN backward of dZ, activation mask recomputed from x (as vjp_bn)
  float bg = 0.f, bb = 0.f;
  Tensor* dg = sink.needs(1) ? sink.dest(1, &bg) : nullptr;
  Tensor* db = sink.needs(2) ? sink.dest(2, &bb) : nullptr;
  TRef tg, tb;
  float gb_beta = 0.f;
  if (dg && db && bg == bb) gb_beta = bg;
  else {
    if (dg && bg != 0.f) { tg = new_tensor({C}, BE_F32); }
    if (db && bb != 0.f) { tb = new_tensor({C}, BE_F32); }
  }
  TRef part = new_tensor({(int64_t)k::bn_partial_floats(rows, C)}, BE_F32);
  float bx = 0.f;
  Tensor* dx = sink.needs(0) ? sink.dest(0, &bx) : nullptr;
  TRef dgs = dg ? TRef() : new_tensor({C}, BE_F32);
  TRef dbs = db ? TRef() : new_tensor({C}, BE_F32);
  float* dgp = tg ? tg->ptr<float>() : (dg ? dg->ptr<float>() : dgs->ptr<float>());
  float* dbp = tb ? tb->ptr<float>() : (db ? db->ptr<float>() : dbs->ptr<float>());
  k::bn_bwd(dz->data(), x->data(), nullptr, act, dx ? dx->data() : nullptr, rows, C, BE_BF16, mean->ptr<float>(),
            inv->ptr<float>(), gamma->ptr<float>(), dgp, dbp, gb_beta, bx, part->ptr<float>(), s,
            act ? beta->ptr<float>() : nullptr);
  if (tg) k::axpby(tg->data(), BE_F32, dg->data(), BE_F32, C, 1.f, 1.f, s);
  if (tb) k::axpby(tb->data(), BE_F32, db->data(), BE_F32, C, 1.f, 1.f, s);
  if (dx) sink.commit(0);
  if (dg) sink.commit(1);
  if (db) sink.commit(2);
}
static void op_bn_conv(const be_tensor* in, int n_in, const void* attrs, be_tensor* out) {
  be_bn_attrs a{1e-5f, 0.1f, 1, 0};
  if (attrs) a = *reinterpret_cast<const be_bn_attrs*>(attrs);
  BE_REQUIRE(n_in == 4 || n_in == 6, BE_E_ARG, "bn_conv1x1: x, gamma, beta[, running_mean, running_var], w");
  BE_REQUIRE(!a.residual && a.act >= 0 && a.act <= 2, BE_E_ARG, "bn_conv1x1: act 0/1/2, no residual");
  Tensor* x = check_handle(in[0]);
  Tensor* gamma = check_handle(in[1]);
  Tensor* beta = check_handle(in[2]);
  Tensor* rm = n_in == 6 && in[3] ? check_handle(in[3]) : nullptr;
  Tensor* rv = n_in == 6 && in[4] ? check_handle(in[4]) : nullptr;
  Tensor* w0 = check_handle(in[n_in - 1]);
  BE_REQUIRE(x->rank == 4 && x->is_contiguous() && x->dtype == BE_BF16, BE_E_SHAPE,
             "bn_conv1x1: contiguous bf16 NHWC input (bf16 compute mode)");
  const int C = (int)x->shape[3];
  BE_REQUIRE(C % 8 == 0, BE_E_UNSUPPORTED, "bn_conv1x1: C % 8 == 0");
  BE_REQUIRE(w0->rank == 4 && w0->shape[1] == 1 && w0->shape[2] == 1 && w0->shape[3] == C, BE_E_SHAPE,
             "bn_conv1x1: weight KRSC [K, 1, 1, C]");
  BE_REQUIRE(gamma->numel() == C && beta->numel() == C && gamma->dtype == BE_F32 && beta->dtype == BE_F32,
             BE_E_SHAPE, "bn_conv1x1: gamma/beta f32 [C]");
  const int K = (int)w0->shape[0];
  BE_REQUIRE(K % 8 == 0, BE_E_UNSUPPORTED, "bn_conv1x1: K % 8 == 0");
  const int64_t rows = x->numel() / C;
  BE_REQUIRE(rows > 0, BE_E_EMPTY_REDUCTION, "bn_conv1x1: empty batch");
  cudaStream_t s = ctx().stream;
  TRef mean = new_tensor({C}, BE_F32), inv = new_tensor({C}, BE_F32);
  TRef part = new_tensor({(int64_t)k::bn_partial_floats(rows, C)}, BE_F32);
  k::bn_stats(x->data(), rows, C, x->dtype, a.eps, mean->ptr<float>(), inv->ptr<float>(), part->ptr<float>(),
              rm ? rm->ptr<float>() : nullptr, rv ? rv->ptr<float>() : nullptr, a.momentum, s);
  if (rm) rm->bump_version();
  if (rv) rv->bump_version();
  Tensor* w = weight_operand(w0);
  BE_REQUIRE(w->dtype == BE_BF16, BE_E_DTYPE, "bn_conv1x1: bf16 compute mode");
  TRef y = new_tensor({x->shape[0], x->shape[1], x->shape[2], (int64_t)K}, BE_BF16);
  k::GemmDesc gd;
  gd.M = (int)rows; gd.N = K; gd.K = C;
  gd.A = x->data(); gd.lda = C; gd.a_kmajor = true;
  gd.B = w->data(); gd.ldb = C; gd.b_kmajor = true;
  gd.ab = BE_BF16; gd.D = y->data(); gd.ldd = K; gd.d = BE_BF16;
  gd.xf_op = 1; gd.xf_act = a.act; gd.xf_C = C;
  gd.xf_mean = mean->ptr<float>(); gd.xf_invstd = inv->ptr<float>();
  gd.xf_gamma = gamma->ptr<float>(); gd.xf_beta = beta->ptr<float>();
  k::gemm(gd, s);
  Node* n = new_node("bn_conv1x1", BE_OP_BN_CONV1X1, vjp_bn_conv, {x, gamma, beta, w0});
  if (n) {
    save(n, x); save(n, mean.get()); save(n, inv.get()); save(n, gamma); save(n, beta); save(n, w);
    n->iattr[0] = a.act;
    set_output(n, y.get(), 0);
    finish_node(n);
  }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

// ------------------------------------------------------------------ embedding
static void vjp_embedding(Node* n, GradSink& sink) {
  TRef hids;
  Tensor* ids = unpack(n, 0, hids);
  if (!sink.needs(0)) return;
  float slr = 0.f;
  const bool sparse = sink.fuse_sparse(0, &slr);
  float beta = 0.f;
  Tensor* dt = sparse ? sink.leaf(0) : sink.dest(0, &beta);
  if (!dt) return;
  TRef gz = contiguous_like(sink.upstream[0], sink.upstream[0]->dtype);
  int64_t B = ids->numel();
  const int64_t D = dt->shape[1], V = dt->shape[0];
  // Sparse exchange (R > 1): every rank all-gathers the step's lookups — ids
  // and upstream rows, R·B·(4 + D·e) bytes instead of the V·D·4 dense
  // gradient — and applies the whole global batch's touched-row update in
  // the same (id, rank, position) order, so the replicas stay bitwise equal.
  const int R = sparse ? ddp_world() : 1;
  TRef all_ids, all_rows;
  float scale = 1.f;
  if (R > 1) {
    all_ids = new_tensor({R * B}, BE_I32);
    all_rows = new_tensor({R * B, D}, gz->dtype);
    ddp_allgather(ids->data(), all_ids->data(), (size_t)B * 4, ctx().stream);
    ddp_allgather(gz->data(), all_rows->data(), (size_t)(B * D) * dtype_size(gz->dtype), ctx().stream);
    ids = all_ids.get();
    gz = all_rows;
    B *= R;
    scale = 1.f / (float)R;
  }
  // the (id, position) sort issued at forward time on the sort stream (R = 1):
  // the compute stream waits for it here (its event is re-recorded after every
  // sort on an in-order stream, so the latest record covers this one)
  if (R == 1 && n->saved.size() > 1) {
    TRef hs;
    Tensor* pre = unpack(n, 1, hs);
    if (pre && n->iattr[0] == V) {
      BE_CHECK_CUDA(cudaStreamWaitEvent(ctx().stream, ctx().sort_done, 0));
      if (sparse) {
        k::embedding_sgd_sorted(gz->data(), gz->dtype, B, D, dt->ptr<float>(), slr, scale, pre->data(), ctx().stream);
        sink.fused_sparse(0);
        return;
      }
      k::embedding_bwd_sorted(gz->data(), gz->dtype, B, D, dt->ptr<float>(), V, beta, pre->data(), ctx().stream);
      sink.commit(0);
      return;
    }
  }
  // Tables looked up with the same ids (NeuMF: GMF and MLP tables of a side)
  // share one sort: a small cache keyed by the ids storage, its version and V
  // (several entries: backward visits the user and item tables interleaved).
  // Entries are valid only within ONE backward pass (ctx().bw_epoch): every
  // step sorts its ids afresh, so ids rewritten in place without a version
  // bump (zero-copy external buffers) can never meet a stale sort.
  struct Entry {
    Storage* st = nullptr;
    uint64_t version = 0, stamp = 0, epoch = 0;
    int64_t B = -1, V = -1, off = 0;
    TRef sorted;
  };
  static Entry cache[4];
  static uint64_t clock = 0;
  Entry* e = nullptr;
  for (Entry& c : cache)
    if (c.st == ids->storage && c.version == ids->version() && c.B == B && c.V == V && c.off == ids->offset &&
        c.epoch == ctx().bw_epoch && c.sorted)
      e = &c;
  if (!e) {
    e = &cache[0];
    for (Entry& c : cache)
      if (c.stamp < e->stamp) e = &c;  // least recently used
    const size_t sb = k::embedding_bwd_scratch(B);
    TRef scratch = new_tensor({(int64_t)((sb + 3) / 4)}, BE_F32);
    k::embedding_sort(ids->ptr<int32_t>(), B, V, scratch->data(), ctx().stream);
    if (e->st) e->st->drop();
    e->st = ids->storage;
    e->st->retain();
    e->version = ids->version();
    e->B = B;
    e->V = V;
    e->off = ids->offset;
    e->epoch = ctx().bw_epoch;
    e->sorted = scratch;
  }
  e->stamp = ++clock;
  if (sparse) {
    k::embedding_sgd_sorted(gz->data(), gz->dtype, B, D, dt->ptr<float>(), slr, scale, e->sorted->data(),
                            ctx().stream);
    sink.fused_sparse(0);
    return;
  }
  k::embedding_bwd_sorted(gz->data(), gz->dtype, B, D, dt->ptr<float>(), V, beta, e->sorted->data(), ctx().stream);
  sink.commit(0);
}
static void op_embedding(const be_tensor* in, int n_in, be_tensor* out) {
  BE_REQUIRE(n_in == 2, BE_E_ARG, "embedding: table, ids");
  Tensor* t = check_handle(in[0]);
  Tensor* ids = check_handle(in[1]);
  BE_REQUIRE(t->rank == 2 && t->dtype == BE_F32 && t->is_contiguous(), BE_E_SHAPE, "embedding: f32 table [V,D]");
  BE_REQUIRE(ids->dtype == BE_I32 && ids->is_contiguous(), BE_E_DTYPE, "embedding: i32 ids");
  const int64_t B = ids->numel(), D = t->shape[1];
  const be_dtype od = ctx().compute;
  TRef y = new_tensor({B, D}, od);
  k::embedding_fwd(t->ptr<float>(), D, ids->ptr<int32_t>(), B, y->data(), od, ctx().stream);
  Node* n = new_node("embedding", BE_OP_EMBEDDING, vjp_embedding, {t});
  if (n) {
    save(n, ids);
    // the backward's (id, position) sort depends only on ids: issue it now on a
    // low-priority side stream so it overlaps the rest of the step instead of
    // sitting on the backward's critical path (single replica: with R > 1 the
    // backward sorts the all-gathered lookups)
    static const int pre_on = [] { const char* e = getenv("BE_EMB_PRESORT"); return e ? atoi(e) : 1; }();
    if (pre_on && ddp_world() == 1 && B > 0 && B < (1LL << 31)) {
      Context& c = ctx();
      if (!c.sort_stream) {
        int least = 0, greatest = 0;
        BE_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        BE_CHECK_CUDA(cudaStreamCreateWithPriority(&c.sort_stream, cudaStreamNonBlocking, least));
        BE_CHECK_CUDA(cudaEventCreateWithFlags(&c.sort_done, cudaEventDisableTiming));
      }
      const size_t sb = k::embedding_bwd_scratch(B);
      TRef scratch = new_tensor({(int64_t)((sb + 3) / 4)}, BE_F32);
      cudaEvent_t ready;
      BE_CHECK_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
      BE_CHECK_CUDA(cudaEventRecord(ready, c.stream));  // ids written, scratch allocated
      BE_CHECK_CUDA(cudaStreamWaitEvent(c.sort_stream, ready, 0));
      BE_CHECK_CUDA(cudaEventDestroy(ready));
      k::embedding_sort(ids->ptr<int32_t>(), B, t->shape[0], scratch->data(), c.sort_stream);
      BE_CHECK_CUDA(cudaEventRecord(c.sort_done, c.sort_stream));
      if (scratch->storage->block) c.alloc.record_stream(scratch->storage->block, c.sort_stream);
      if (ids->storage->block) c.alloc.record_stream(ids->storage->block, c.sort_stream);
      save(n, scratch.get());
      n->iattr[0] = t->shape[0];
    }
    set_output(n, y.get(), 0);
    finish_node(n);
  }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

void op_cnn(int op, const be_tensor* in, int n_in, const void* attrs, be_tensor* out, int n_out) {
  switch (op) {
    case BE_OP_CONV2D: op_conv(in, n_in, attrs, out); break;
    case BE_OP_MAXPOOL2D: op_maxpool(in, n_in, attrs, out, n_out); break;
    case BE_OP_AVGPOOL_GLOBAL: op_avgpool(in, n_in, out); break;
    case BE_OP_BATCHNORM2D: op_bn(in, n_in, attrs, out); break;
    case BE_OP_EMBEDDING: op_embedding(in, n_in, out); break;
    case BE_OP_BN_CONV1X1: op_bn_conv(in, n_in, attrs, out); break;
    default: fail(BE_E_UNSUPPORTED, "op_cnn: unknown op");
  }
}

}  // namespace be

using namespace be;
extern "C" be_status be_debug_im2col_offsets(const int64_t* geom, int64_t* out) {
  BE_API_BEGIN
  BE_REQUIRE(ctx().inited, BE_E_NOT_INIT, "be_init() was not called");
  k::ConvGeom g;
  g.N = (int)geom[0]; g.C = (int)geom[1]; g.H = (int)geom[2]; g.W = (int)geom[3];
  g.R = (int)geom[4]; g.S = (int)geom[5]; g.stride = (int)geom[6]; g.pad = (int)geom[7];
  g.P = (g.H + 2 * g.pad - g.R) / g.stride + 1;
  g.Q = (g.W + 2 * g.pad - g.S) / g.stride + 1;
  g.K = 1;
  const int64_t total = (int64_t)g.N * g.P * g.Q * g.R * g.S * g.C;
  TRef buf = new_tensor({std::max<int64_t>(total, 1)}, BE_I64);
  k::im2col_offsets(g, buf->ptr<int64_t>(), ctx().stream);
  if (total) BE_CHECK_CUDA(cudaMemcpyAsync(out, buf->data(), total * 8, cudaMemcpyDeviceToHost, ctx().stream));
  BE_CHECK_CUDA(cudaStreamSynchronize(ctx().stream));
  BE_API_END
}
