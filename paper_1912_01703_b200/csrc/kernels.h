// kernels.h — host-side launchers of the sm_100a kernels (internal API).
// Every launcher enqueues on the given stream and returns immediately.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/be.h"

namespace be { namespace k {

struct ConvGeom {
  int N, H, W, C, K, R, S, stride, pad, P, Q;
};

// ------------------------------------------------------------------ GEMM
// D[M,N] = act(A[M,K]·B[N,K]ᵀ + bias[N]) + beta·D   (fp32 accumulate)
// A element (m,k) at A[m*lda + k] if a_kmajor else A[k*lda + m];
// B element (n,k) at B[n*ldb + k] if b_kmajor else B[k*ldb + n].
// ab = BE_BF16 (kind::f16) or BE_F32 (3xTF32 on kind::tf32).
struct GemmDesc {
  int M = 0, N = 0, K = 0;
  const void* A = nullptr; int64_t lda = 0; bool a_kmajor = true;
  const void* B = nullptr; int64_t ldb = 0; bool b_kmajor = true;
  be_dtype ab = BE_BF16;
  void* D = nullptr; int64_t ldd = 0; be_dtype d = BE_F32;
  float beta = 0.f;
  const float* bias = nullptr;
  int act = 0;  // 0 none, 1 relu
  // conv wgrad: B (MN-major, [K = pixels, N = R·S·C]) is im2col(conv_x) read in
  // place by TMA im2col (bf16, C % 64 == 0); B / ldb are then ignored
  const void* conv_x = nullptr;
  ConvGeom conv_g{};
  // with conv_x: read A (= dY, [N·P·Q, K_out]) and B (= x) as shifted 4-D
  // tiles instead of an im2col map (needs Q ≤ 64, C % 64 == 0, K_out % 8 == 0)
  bool conv_shift = false;
  // fused SGD epilogue: when set, D is not written; the accumulator is the
  // gradient g of the parameter P[M, N] (row-major, ld = ldd) and the epilogue
  // applies the SGD update to P, its momentum V and its bf16 shadow directly
  const struct SgdFuse* upd = nullptr;
  // batch-norm statistics of the stored output (no bias / act / beta): per
  // column Σ and Σx² partials [parts][N] then [parts][N] written into `stats`
  // (zeroed by the caller, room for 4·num_sms parts); *stats_parts = parts
  // when the launched kernel produced them (left untouched otherwise)
  float* stats = nullptr;
  int* stats_parts = nullptr;
  // operand transform (batch-norm apply fused into the GEMM's operand load):
  // xf_op 1: A[m, k] ← act(γ_k·(A − μ_k)·is_k + β_k) (A K-major, bf16);
  // xf_op 2: the same on B[n, k] per channel n (B MN-major, bf16);
  // channels ≥ xf_C read 0 parameters.  1-CTA bf16 kernel only.
  int xf_op = 0, xf_act = 0, xf_C = 0;
  const float *xf_mean = nullptr, *xf_invstd = nullptr, *xf_gamma = nullptr, *xf_beta = nullptr;
};
struct SgdFuse {
  float* p = nullptr; float* v = nullptr; uint16_t* shadow = nullptr;
  float lr = 0.f, mu = 0.f, wd = 0.f, scale = 1.f;
};
// Returns the name of the path taken ("tcgen05" or "simt").
const char* gemm(const GemmDesc& g, cudaStream_t s);
// true when g runs on the tcgen05 path (the only one with the update epilogue)
bool gemm_tc_ok(const GemmDesc& g);
// true when g.upd can run (bf16, 16-B aligned P/V rows, 8-B aligned shadow)
bool gemm_update_ok(const GemmDesc& g);
// Encode counters for tests/bench (which path ran).
uint64_t gemm_tcgen05_calls();
uint64_t gemm_simt_calls();

// ------------------------------------------------------------------ pointwise
void fill(void* x, int64_t n, be_dtype dt, double v, cudaStream_t s);
void cast(const void* x, be_dtype xd, void* y, be_dtype yd, int64_t n, cudaStream_t s);
void split_tf32(const float* x, float* hi, float* lo, int64_t n, cudaStream_t s);
void relu_fwd(const void* x, void* y, int64_t n, be_dtype dt, cudaStream_t s);
// dx (+)= dy * [y > 0]
void relu_bwd(const void* dy, const void* y, void* dx, int64_t n, be_dtype dt, float beta, cudaStream_t s);
// d1 (+)= dy·[y>0], d2 (+)= dy·[y>0] in one pass (residual add+ReLU backward); d1/d2 may be null
void relu_bwd2(const void* dy, const void* y, void* d1, float b1, void* d2, float b2, int64_t n, be_dtype dt,
               cudaStream_t s);
// y = a + b with b broadcast: general strided (rank<=6) over out shape
struct BcastDesc {
  int rank;
  int64_t shape[6];
  int64_t sa[6], sb[6];  // element strides of a,b in out index space (0 = broadcast)
};
void add_bcast(const void* a, const void* b, void* y, const BcastDesc& d, be_dtype dt, int act, cudaStream_t s);
void add_same(const void* a, const void* b, void* y, int64_t n, be_dtype dt, int act, cudaStream_t s);
void mul_same(const void* a, const void* b, void* y, int64_t n, be_dtype dt, cudaStream_t s);
// y (+)= a * b
void mul_acc(const void* a, const void* b, void* y, int64_t n, be_dtype dt, float beta, cudaStream_t s);
// y = alpha*x + beta*y   (accumulation helper; dtypes may differ: x dt_x, y dt_y)
void axpby(const void* x, be_dtype xd, void* y, be_dtype yd, int64_t n, float alpha, float beta, cudaStream_t s);
// y = x * (*scalar_dev)
void scale_dev(const void* x, be_dtype xd, void* y, be_dtype yd, int64_t n, const float* scalar, cudaStream_t s);
// out[c] (+)= Σ_r x[r, c]  (x [rows, cols] row-major, dt), fp32 out, deterministic
void colsum(const void* x, int64_t rows, int64_t cols, be_dtype dt, float* out, float beta, cudaStream_t s);
// fused ReLU-backward + column sum: dz = dy*[y>0] (dz may alias dy), db (+)= Σ_r dz
void relu_bwd_colsum(const void* dy, const void* y, void* dz, int64_t rows, int64_t cols, be_dtype dt,
                     float* db, float db_beta, int act, cudaStream_t s);
// sum of all elements into out[0] (fp32), scale applied (mean)
void reduce_sum(const void* x, int64_t n, be_dtype dt, float* out, float scale, float* scratch, cudaStream_t s);
void broadcast_scalar(const float* g, void* dx, be_dtype dt, int64_t n, float scale, float beta, cudaStream_t s);

// ------------------------------------------------------------------ losses
// loss_out[0] = mean_i (LSE(z_i) − z_i[y_i]); dz = (softmax − onehot)/B written in dz_dt;
// argmax (first max) to argmax_out (may be null). row_loss: scratch [B] fp32.
void softmax_xent(const void* z, be_dtype zd, int64_t ldz, const int32_t* y, int64_t B, int64_t C,
                  float* row_loss, float* loss_out, void* dz, be_dtype dzd, int32_t* argmax_out,
                  cudaStream_t s);
void bce_logits(const void* z, be_dtype zd, const int32_t* y, int64_t B, float* row_loss, float* loss_out,
                void* dz, be_dtype dzd, cudaStream_t s);

// ------------------------------------------------------------------ SGD
struct SgdEntry {
  float* p; const float* g; uint16_t* shadow; float* mom; int64_t n;
};
// blocks_per_sm: persistent grid of num_sms × blocks_per_sm blocks
void sgd_multi(const SgdEntry* e, int n_entries, float lr, float momentum, float wd, float scale,
               cudaStream_t s, int blocks_per_sm = 8);

// ------------------------------------------------------------------ conv / pool / bn
// Implicit-GEMM convolution on tcgen05 (bf16, C % 64 == 0): y[NPQ, K] =
// conv(x NHWC, w KRSC) (+bias, act, beta). Returns false when unsupported.
// stride-1 conv weight gradient (C = K ∈ {64, 128}) from one shared input patch per
// tile with shifted UMMA operands (gemm_sm100.cu conv_wgrad_patch_kernel);
// dw fp32 [K, R·S·C], dw = (beta ? dw : 0) + dW.  false: shape not supported
bool conv_wgrad_patch(const void* dy, const void* x, void* dw, be_dtype dwt, const ConvGeom& g, float beta,
                      cudaStream_t s);
// stem conv weight gradient (C = 8, K = 64): im2col slices built in smem from
// a per-row input patch (gemm_sm100.cu conv_wgrad_stem_kernel); false: not applicable
// dW (fp32, [K, R·S·C]) (+)= dYᵀ·im2col(x) with the im2col slice gathered in smem (C % 64, K % 128)
bool conv_wgrad_gather(const void* dy, const void* x, void* dw, be_dtype dwt, const ConvGeom& g, float beta,
                       cudaStream_t s);
bool conv_wgrad_stem(const void* dy, const void* x, void* dw, be_dtype dwt, const ConvGeom& g, float beta,
                     cudaStream_t s);
// bw (data gradient as a convolution of dY): w is the FORWARD weight W[K_fwd = g.C][R_f, S_f, C_fwd = g.K],
// read in place as the MN-major B operand; tap (t_r, t_s) of this convolution reads forward tap
// (bw[0] + bw[1]·t_r, bw[2] + bw[3]·t_s); bw[4] = S_f, bw[5] = R_f·S_f·C_fwd
bool conv_implicit(const void* x, const void* w, void* y, const ConvGeom& g, be_dtype yd, const float* bias, int act,
                   float beta, cudaStream_t s, float* stats = nullptr, int* stats_parts = nullptr,
                   const int* bw = nullptr);
// stride-2+ dgrad by phases (gemm_sm100.cu conv_dgrad_phases; false = not applicable)
bool conv_dgrad_phases(const void* dy, const void* w, void* dx, const ConvGeom& g, float beta, cudaStream_t s);
// zero the dx pixels of phases without taps (cr[ρh] == 0 or cs[ρw] == 0)
void conv_phase_zero(void* dx, const ConvGeom& g, const int* cr, const int* cs, cudaStream_t s);
// cols[M, R*S*C] (row-major, ldc = padded RSC) from x NHWC
void im2col(const void* x, void* cols, int64_t ldc, const ConvGeom& g, be_dtype dt, cudaStream_t s);
// dx NHWC (+)= col2im(dcols)   (gather formulation, deterministic)
void col2im(const void* dcols, int64_t ldc, void* dx, const ConvGeom& g, be_dtype dt, float beta, cudaStream_t s);
void im2col_offsets(const ConvGeom& g, int64_t* out_dev, cudaStream_t s);
void maxpool_fwd(const void* x, void* y, uint8_t* am, const ConvGeom& g, be_dtype dt, cudaStream_t s);
void maxpool_bwd(const void* dy, const uint8_t* am, void* dx, const ConvGeom& g, be_dtype dt, float beta, cudaStream_t s);
void avgpool_fwd(const void* x, void* y, int N, int HW, int C, be_dtype dt, cudaStream_t s);
void avgpool_bwd(const void* dy, void* dx, int N, int HW, int C, be_dtype dt, float beta, cudaStream_t s);
// BN train: stats per channel over rows (x as [rows, C]); mean/invstd fp32 [C]
void bn_stats(const void* x, int64_t rows, int C, be_dtype dt, float eps, float* mean, float* invstd,
              float* partial, float* run_mean, float* run_var, float momentum, cudaStream_t s);
// y = act(γ·(x − μ)·is + β [+ res])   (res: optional residual, same layout/dtype as x)
void bn_apply(const void* x, void* y, int64_t rows, int C, be_dtype dt, const float* mean, const float* invstd,
              const float* gamma, const float* beta, int act, cudaStream_t s, const void* res = nullptr,
              uint8_t* mbits = nullptr, int early = 0);
// y = act(γ·(x − μ)·is + β + γr·(xr − μr)·isr + βr) — the ResNet projection block output with the
// shortcut's BN applied in the same pass (bf16 stream path), optional 1-bit mask as bn_apply
void bn_apply_stream2(const uint16_t* x, uint16_t* y, int64_t rows, int C, const float* mean, const float* invstd,
                      const float* gamma, const float* beta, int act, const uint16_t* xr, const float* mean_r,
                      const float* invstd_r, const float* gamma_r, const float* beta_r, cudaStream_t s,
                      uint8_t* mbits);
// true when bn_apply can also write the 1-bit ReLU mask of its output (mbits:
// rows·C/8 bytes, bit j of byte r·C/8 + c/8 ⇔ y[r, c + j] > 0) for bn_bwd's rbits
bool bn_mask_bits_ok(const void* x, const void* y, const void* res, int64_t rows, int C, be_dtype dt);
size_t bn_partial_floats(int64_t rows, int C);
// mean / invstd (+ running stats) from unshifted per-part column sums: Σ in
// partial[0..parts)[C], Σx² in partial[parts..2·parts)[C] (conv epilogue)
void bn_stats_from_partials(const float* partial, int parts, int64_t rows, int C, float eps, float* mean,
                            float* invstd, float* run_mean, float* run_var, float momentum, cudaStream_t s);
// backward: dgamma, dbeta (fp32, with beta-accumulate flags) and dx
void bn_bwd(const void* dy, const void* x, const void* y, int act, void* dx, int64_t rows, int C, be_dtype dt,
            const float* mean, const float* invstd, const float* gamma, float* dgamma, float* dbeta,
            float gb_beta, float dx_beta, float* partial, cudaStream_t s, const float* bn_beta = nullptr,
            const void* rmask = nullptr, void* gout = nullptr, const uint8_t* rbits = nullptr);
// rmask (residual BN, y = relu(bn(x) + r)): the upstream is first masked,
// g = dy·1[rmask > 0], written to gout (the shortcut's gradient) — fused into
// the reduction pass on the bf16 path; act must be 0

// ------------------------------------------------------------------ embedding
void embedding_fwd(const float* table, int64_t D, const int32_t* ids, int64_t B, void* out, be_dtype od,
                   cudaStream_t s);
// dtable (+)= scatter(ids, drows): deterministic via sort-by-id then segmented sum
void embedding_bwd(const void* drows, be_dtype dd, const int32_t* ids, int64_t B, int64_t D, float* dtable,
                   int64_t V, float beta, void* scratch, size_t scratch_bytes, cudaStream_t s);
size_t embedding_bwd_scratch(int64_t B);
// the two phases of embedding_bwd: stable sort of (id, position) into scratch
// [0, 8·B) (needs 16·B bytes), then per-id segment sums from that sorted list
void embedding_sort(const int32_t* ids, int64_t B, int64_t V, void* scratch, cudaStream_t s);
void embedding_bwd_sorted(const void* drows, be_dtype dd, int64_t B, int64_t D, float* dtable, int64_t V, float beta,
                          const void* sorted, cudaStream_t s);
// sparse SGD of the touched rows from the sorted (id, position) pairs (see embedding_sort)
void embedding_sgd_sorted(const void* drows, be_dtype dd, int64_t B, int64_t D, float* table, float lr, float scale,
                          const void* sorted, cudaStream_t s);
void concat_cols(const void* const* xs, const int64_t* widths, int n, int64_t rows, void* y, be_dtype dt,
                 cudaStream_t s);
void slice_cols(const void* y, int64_t ldy, int64_t col0, int64_t width, int64_t rows, void* x, be_dtype dt,
                float beta, cudaStream_t s);


// ------------------------------------------------------------------ mobile.cu
// inverted dropout y (+)= x·keep·1/(1−p), keep_i = (Philox4x64-10(i/4, offset; seed)[i%4] >> 32) >= ⌊p·2^32⌋
void dropout_apply(const void* x, void* y, int64_t n, be_dtype dt, uint64_t seed, uint64_t offset, double p,
                   float beta, cudaStream_t s);
// depthwise conv, x/y NHWC (C % 8 == 0), w RSC fp32
void dw_conv_fwd(const void* x, const float* w, void* y, const ConvGeom& g, be_dtype dt, cudaStream_t s);
void dw_conv_dgrad(const void* dy, const float* w, void* dx, const ConvGeom& g, be_dtype dt, float beta,
                   cudaStream_t s);
size_t dw_wgrad_partial_floats(const ConvGeom& g, int num_sms);
void dw_conv_wgrad(const void* dy, const void* x, float* dw, float* part, const ConvGeom& g, be_dtype dt,
                   float beta, int num_sms, cudaStream_t s);

// ------------------------------------------------------------------ p2p.cu
// One gradient bucket of the peer-memory allreduce fused with SGD (see p2p.cu).
// Pointers are device addresses valid in this process (own allocations or
// CUDA-IPC mappings of the peers'); tables live in device memory.
struct P2PBucketArgs {
  int rank = 0, world = 1;
  int64_t numel = 0;                      // bucket length (params at 64-aligned offsets)
  int nseg = 0;                           // parameters in the bucket
  const int64_t* seg_off = nullptr;       // [nseg] offset of each parameter in the bucket (ascending)
  const int64_t* seg_n = nullptr;         // [nseg] numel of each parameter
  float* const* grad = nullptr;           // [R] bucket base on every rank
  float* const* p = nullptr;              // [nseg·R] fp32 master of parameter s on rank q
  uint16_t* const* shadow = nullptr;      // [nseg·R] bf16 shadow (entries may be null) or null
  float* const* mom = nullptr;            // [nseg] local momentum buffers (μ ≠ 0)
  unsigned long long* flags_arrive = nullptr;        // [R] local
  unsigned long long* flags_done = nullptr;          // [R] local
  unsigned long long* const* flags_peer = nullptr;      // [R] rank q's flags_arrive
  unsigned long long* const* flags_peer_done = nullptr; // [R] rank q's flags_done
  unsigned int* counter = nullptr;        // local, cumulative
  int* status = nullptr;                  // local: 1 = barrier timeout
  unsigned long long epoch = 0;
  int lr_on = 0;                          // 1: SGD (lr, mu, wd); 0: plain mean allreduce into the buckets
  float lr = 0.f, mu = 0.f, wd = 0.f;
};
void p2p_allreduce_sgd(const P2PBucketArgs& a, int blocks, cudaStream_t s);
}}  // namespace be::k
