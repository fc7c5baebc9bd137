// ops_mobile.cpp — be_op dispatch and VJPs for the Table 1 CNN extras
// (VGG-19, MobileNet): inverted dropout with a counter-based
// mask and depthwise convolution.  Definitions follow
// oracle/ops.py (dropout, conv2d_depthwise); no code is shared with it.
#include "ops_common.h"

namespace be {

// ------------------------------------------------------------------ dropout
// The mask is regenerated from (seed, offset, element index) in the backward
// pass: nothing but the three scalars is saved.
static void vjp_dropout(Node* n, GradSink& sink) {
  float beta;
  Tensor* dx = sink.dest(0, &beta);
  if (!dx) return;
  TRef gz = contiguous_like(sink.upstream[0], dx->dtype);
  double p;
  memcpy(&p, n->attrs, sizeof(p));
  k::dropout_apply(gz->data(), dx->data(), dx->numel(), dx->dtype, (uint64_t)n->iattr[0], (uint64_t)n->iattr[1], p,
                   beta, ctx().stream);
  sink.commit(0);
}
static void op_dropout(const be_tensor* in, int n_in, const void* attrs, be_tensor* out) {
  BE_REQUIRE(n_in == 1 && attrs, BE_E_ARG, "dropout: x + be_dropout_attrs");
  const be_dropout_attrs a = *reinterpret_cast<const be_dropout_attrs*>(attrs);
  BE_REQUIRE(a.p >= 0.0 && a.p <= 1.0, BE_E_ARG, "dropout: p must be in [0, 1]");
  Tensor* x = check_handle(in[0]);
  BE_REQUIRE(x->is_contiguous(), BE_E_NONCONTIG, "dropout: contiguous input");
  BE_REQUIRE(x->dtype == BE_F32 || x->dtype == BE_BF16, BE_E_DTYPE, "dropout: float dtype");
  TRef y = new_tensor(x->shape, x->rank, x->dtype);
  const bool identity = !a.training || a.p == 0.0;
  if (identity) {
    if (x->numel()) BE_CHECK_CUDA(cudaMemcpyAsync(y->data(), x->data(), (size_t)x->numel() * dtype_size(x->dtype), cudaMemcpyDeviceToDevice,
                                                  ctx().stream));
  } else {
    k::dropout_apply(x->data(), y->data(), x->numel(), x->dtype, a.seed, a.offset, a.p, 0.f, ctx().stream);
  }
  Node* n = new_node("dropout", BE_OP_DROPOUT, vjp_dropout, {x});
  if (n) {
    const double p = identity ? 0.0 : a.p;
    memcpy(n->attrs, &p, sizeof(p));
    n->iattr[0] = (int64_t)a.seed;
    n->iattr[1] = (int64_t)a.offset;
    set_output(n, y.get(), 0);
    finish_node(n);
  }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

// ------------------------------------------------------------------ depthwise conv
static k::ConvGeom dw_geom(const Tensor* x, const Tensor* w, int stride, int pad) {
  k::ConvGeom g;
  g.N = (int)x->shape[0]; g.H = (int)x->shape[1]; g.W = (int)x->shape[2]; g.C = (int)x->shape[3];
  g.R = (int)w->shape[0]; g.S = (int)w->shape[1]; g.K = g.C;
  g.stride = stride; g.pad = pad;
  g.P = (g.H + 2 * pad - g.R) / stride + 1;
  g.Q = (g.W + 2 * pad - g.S) / stride + 1;
  return g;
}
static void vjp_dwconv(Node* n, GradSink& sink) {
  cudaStream_t s = ctx().stream;
  TRef hx, hw;
  Tensor* x = unpack(n, 0, hx);
  Tensor* w = unpack(n, 1, hw);
  const k::ConvGeom g = dw_geom(x, w, (int)n->iattr[0], (int)n->iattr[1]);
  TRef gz = contiguous_like(sink.upstream[0], x->dtype);
  if (sink.needs(1)) {
    float bw;
    Tensor* dw = sink.dest(1, &bw);
    TRef part = new_tensor({(int64_t)k::dw_wgrad_partial_floats(g, ctx().num_sms)}, BE_F32);
    k::dw_conv_wgrad(gz->data(), x->data(), dw->ptr<float>(), part->ptr<float>(), g, x->dtype, bw, ctx().num_sms, s);
    sink.commit(1);
  }
  if (sink.needs(0)) {
    float bx;
    Tensor* dx = sink.dest(0, &bx);
    k::dw_conv_dgrad(gz->data(), w->ptr<float>(), dx->data(), g, dx->dtype, bx, s);
    sink.commit(0);
  }
}
static void op_dwconv(const be_tensor* in, int n_in, const void* attrs, be_tensor* out) {
  BE_REQUIRE(n_in == 2 && attrs, BE_E_ARG, "conv2d_depthwise: x, w + be_dwconv_attrs");
  const be_dwconv_attrs a = *reinterpret_cast<const be_dwconv_attrs*>(attrs);
  Tensor* x = check_handle(in[0]);
  Tensor* w = check_handle(in[1]);
  BE_REQUIRE(x->rank == 4 && x->is_contiguous(), BE_E_SHAPE, "conv2d_depthwise: contiguous NHWC input");
  BE_REQUIRE(x->dtype == BE_F32 || x->dtype == BE_BF16, BE_E_DTYPE, "conv2d_depthwise: float input");
  BE_REQUIRE(w->rank == 3 && w->is_contiguous() && w->dtype == BE_F32, BE_E_SHAPE,
             "conv2d_depthwise: weight f32 RSC [R,S,C]");
  BE_REQUIRE(w->shape[2] == x->shape[3], BE_E_SHAPE, "conv2d_depthwise: weight channels != input channels");
  BE_REQUIRE(x->shape[3] % 8 == 0, BE_E_UNSUPPORTED, "conv2d_depthwise: C % 8 == 0 (16-B channel vectors)");
  BE_REQUIRE(w->shape[0] == 3 && w->shape[1] == 3, BE_E_UNSUPPORTED, "conv2d_depthwise: 3x3 filters");
  BE_REQUIRE(a.stride >= 1 && a.pad >= 0 && a.pad < 3, BE_E_ARG, "conv2d_depthwise: bad stride/pad");
  const k::ConvGeom g = dw_geom(x, w, a.stride, a.pad);
  BE_REQUIRE(g.P > 0 && g.Q > 0, BE_E_SHAPE, "conv2d_depthwise: filter larger than padded input");
  TRef y = new_tensor({g.N, g.P, g.Q, g.C}, x->dtype);
  k::dw_conv_fwd(x->data(), w->ptr<float>(), y->data(), g, x->dtype, ctx().stream);
  Node* n = new_node("conv2d_depthwise", BE_OP_CONV2D_DEPTHWISE, vjp_dwconv, {x, w});
  if (n) {
    save(n, x);
    save(n, w);
    n->iattr[0] = a.stride;
    n->iattr[1] = a.pad;
    set_output(n, y.get(), 0);
    finish_node(n);
  }
  out[0] = reinterpret_cast<be_tensor>(y.release());
}

void op_mobile(int op, const be_tensor* in, int n_in, const void* attrs, be_tensor* out, int) {
  switch (op) {
    case BE_OP_DROPOUT: op_dropout(in, n_in, attrs, out); break;
    case BE_OP_CONV2D_DEPTHWISE: op_dwconv(in, n_in, attrs, out); break;
    default: fail(BE_E_UNSUPPORTED, "op_mobile: unknown op");
  }
}

}  // namespace be
