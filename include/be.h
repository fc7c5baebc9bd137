/*
 * be.h — C ABI of the B200-native eager training-step library ("be" =
 * B200 eager).  This is the boundary of the hot path named by
 * BASELINE.json north_star: tensor create/free, op dispatch + record-to-tape,
 * backward(), step(), served by a stream-ordered caching allocator, with a
 * bucketed data-parallel gradient allreduce.
 *
 * Paper passages (arXiv 1912.01703, /root/reference/PAPER.md line numbers):
 *   - tensors + operators + autograd in a C++ core ..... PAPER.md:177 (§5.1)
 *   - define-by-run tape, reverse mode, versions ....... PAPER.md:158-165 (§4.3)
 *   - async queueing on a CUDA stream .................. PAPER.md:183-187 (§5.2)
 *   - caching allocator, 512-B rounding, pool/stream ... PAPER.md:193-204 (§5.3)
 *   - refcount-driven immediate free ................... PAPER.md:221-229 (§5.5)
 *   - all-reduce gradient synchronisation .............. PAPER.md:216 (§5.4)
 * SPEC.md (a CPU spec written from the paper) fixes the error names and the
 * small contracts cited as S:n.
 *
 * General rules
 *   - Every function returns be_status: 0 (BE_OK) or an error code below.
 *     Nothing throws or aborts across the ABI; be_last_error() returns a
 *     thread-local message for the most recent failure on this thread.
 *   - Ownership: every be_tensor written through an `out` pointer carries ONE
 *     reference owned by the caller, who must be_release() it.  The last
 *     release returns the memory block to the allocator pool of the stream
 *     it was allocated on, immediately.
 *   - Asynchrony: all device work is enqueued on the library's compute stream
 *     (PAPER.md:185); calls return before the kernels finish.  Only
 *     be_tensor_to_host, be_item and be_synchronize wait.  Environment
 *     BE_SYNC=1 synchronises after every launch (debug).
 *   - Single device per process; grad mode is thread-local.
 *   - There is NO CPU fallback: a missing/unsupported device path returns
 *     BE_E_UNSUPPORTED.
 */
#ifndef BE_H_
#define BE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct be_tensor_s* be_tensor;   /* opaque, intrusive refcount */
typedef int be_status;

/* dtype codes 0-3 follow SPEC's MTNS codes. */
typedef enum {
  BE_F32 = 0, BE_F64 = 1, BE_I64 = 2, BE_BOOL = 3, BE_BF16 = 4, BE_I32 = 5, BE_U8 = 6
} be_dtype;

enum {
  BE_OK = 0,
  BE_E_SHAPE = 1,            /* ShapeMismatch */
  BE_E_BROADCAST = 2,        /* BroadcastError */
  BE_E_DTYPE = 3,            /* DTypeMismatch / UnsupportedDType */
  BE_E_AXIS = 4,             /* AxisOutOfRange */
  BE_E_EMPTY_REDUCTION = 5,  /* EmptyReduction */
  BE_E_NONCONTIG = 6,        /* NonContiguous */
  BE_E_VERSION = 7,          /* saved tensor mutated before backward */
  BE_E_DOUBLE_BACKWARD = 8,  /* second backward without retain_graph */
  BE_E_NO_UPSTREAM = 9,      /* non-scalar root without upstream */
  BE_E_INPLACE_LEAF = 10,    /* in-place on a leaf requiring grad */
  BE_E_MISSING_GRAD = 11,    /* optimizer step on a param without grad */
  BE_E_OOM = 12,             /* after one empty_cache retry */
  BE_E_DOUBLE_FREE = 13,
  BE_E_BAD_HANDLE = 14,
  BE_E_CUDA = 15,            /* CUDA error; async faults surface at the next sync */
  BE_E_NCCL = 16,
  BE_E_UNSUPPORTED = 17,     /* no device path for this request (no CPU fallback) */
  BE_E_NOT_INIT = 18,
  BE_E_ARG = 19
};

/* ------------------------------------------------------------------ init */
/* Bind the library to CUDA device `device` and a compute stream.
 * cuda_stream: a cudaStream_t cast to uint64 (e.g. torch's current stream)
 * that the library adopts but never destroys; 0 = create an own stream.
 * Must be called once per process before any other call (BE_E_NOT_INIT). */
be_status be_init(int device, uint64_t cuda_stream);
/* Returns the compute stream in use (cudaStream_t as uint64). */
be_status be_get_stream(uint64_t* out);
const char* be_last_error(void);
/* Number of kernels this library launched since init (all streams). */
be_status be_launch_count(uint64_t* out);

/* ------------------------------------------------------------------ tensors
 * Shapes are row-major, rank <= 6.  Device layouts used by the ops:
 * activations NHWC (4-D) or [rows, cols] (2-D); conv weights KRSC;
 * Linear weights [in, out] (Listing 1). */
/* Allocate a contiguous tensor and copy `host` (row-major, nbytes =
 * numel*size(dtype)) into it; host may be NULL (uninitialised).  The copy
 * is stream-ordered; `host` must stay valid until the next synchronising
 * call (use pinned memory for async copies).  requires_grad marks a leaf
 * (S:48-54). */
be_status be_tensor_create(const void* host, const int64_t* shape, int rank, be_dtype dtype,
                           int requires_grad, be_tensor* out);
be_status be_tensor_empty(const int64_t* shape, int rank, be_dtype dtype, be_tensor* out);
/* Zero-copy wrap of device memory.  `release`
 * (may be NULL) is invoked with ctx exactly once when the last reference
 * dies.  strides may be NULL (contiguous). */
be_status be_tensor_from_device(void* dptr, const int64_t* shape, const int64_t* strides,
                                int rank, be_dtype dtype, void (*release)(void*), void* ctx,
                                be_tensor* out);
/* Synchronous device→host copy of a tensor (any strides) into dst, row-major. */
be_status be_tensor_to_host(be_tensor t, void* dst, size_t nbytes);
/* Async stream-ordered host↔device copies for a contiguous tensor. */
be_status be_tensor_copy_from_host_async(be_tensor t, const void* src, size_t nbytes);
be_status be_tensor_copy_to_host_async(be_tensor t, void* dst, size_t nbytes);
/* Metadata. */
be_status be_tensor_info(be_tensor t, int* rank, int64_t* shape /*6*/, int64_t* strides /*6*/,
                         be_dtype* dtype, uint64_t* device_ptr);
be_status be_tensor_version(be_tensor t, uint64_t* out);
be_status be_tensor_requires_grad(be_tensor t, int* out);
be_status be_retain(be_tensor t);
be_status be_release(be_tensor t);                                  /* BE_E_DOUBLE_FREE */
/* In-place fill (bumps the version by 1).  BE_E_INPLACE_LEAF when t
 * is a leaf that requires grad and grad mode is on. */
be_status be_fill_(be_tensor t, double value);
/* Copy src into dst in place (same shape; dtype cast allowed; bumps version). */
be_status be_copy_(be_tensor dst, be_tensor src);

/* ------------------------------------------------------------------ ops
 * be_op both dispatches (launches the kernels on the compute stream) and,
 * when grad mode is on and an input requires grad, records a tape node
 * holding version-pinned saved tensors. */
typedef enum {
  BE_OP_LINEAR = 1,        /* in: x[B,in], w[in,out], b[out] (n_in 2|3); attrs be_linear_attrs; out: y[B,out] */
  BE_OP_MATMUL = 2,        /* in: a[M,K], b[K,N]; out: [M,N] */
  BE_OP_ADD = 3,           /* in: a, b (right-aligned broadcast); attrs int* act (NULL|0 none, 1 relu) */
  BE_OP_MUL = 4,           /* in: a, b same shape */
  BE_OP_RELU = 5,          /* in: x */
  BE_OP_SOFTMAX_XENT = 6,  /* in: logits[B,C], labels i32[B]; out: loss f32 [] (mean), optional out[1]: argmax i32[B] */
  BE_OP_BCE_LOGITS = 7,    /* in: z[B,1] or [B], labels i32[B] (0|1); out: loss f32 [] (mean) */
  BE_OP_CONV2D = 8,        /* in: x NHWC[N,H,W,C], w KRSC[K,R,S,C], b[K] optional; attrs be_conv_attrs; out NHWC[N,P,Q,K] */
  BE_OP_MAXPOOL2D = 9,     /* in: x NHWC; attrs be_pool_attrs; out: y NHWC, optional out[1]: argmax u8 window index (r*k+u) */
  BE_OP_AVGPOOL_GLOBAL = 10, /* in: x NHWC[N,H,W,C]; out [N,C] */
  BE_OP_BATCHNORM2D = 11,  /* in: x NHWC, gamma[C], beta[C], running_mean[C]?, running_var[C]?, residual?; attrs be_bn_attrs */
  BE_OP_RESHAPE = 12,      /* in: x contiguous; attrs be_shape_attrs; out: view (shares storage) */
  BE_OP_EMBEDDING = 13,    /* in: table[V,D] (f32 param), ids i32[B]; out [B,D] */
  BE_OP_CONCAT = 14,       /* in: n 2-D tensors [B,Di]; concatenated along axis 1 */
  BE_OP_SUM = 15,          /* in: x; out: [] */
  BE_OP_MEAN = 16,         /* in: x; out: [] */
  BE_OP_CAST = 17,         /* in: x; attrs be_dtype*; out: x cast (RN-even for f32→bf16) */
  BE_OP_ADD_RELU = 18,     /* residual: y = relu(a + b), same shape */
  BE_OP_DROPOUT = 19,      /* in: x (contiguous f32|bf16); attrs be_dropout_attrs; out: y = x·keep/(1−p) (
                              PAPER.md:64).  keep_i = (Philox4x64-10(counter (i/4, offset, 0, 0), key (seed, 0))[i%4] >> 32)
                              >= floor(p·2^32), i the row-major element index — regenerated in backward, no mask stored */
  BE_OP_CONV2D_DEPTHWISE = 20, /* in: x NHWC[N,H,W,C] (C % 8 == 0), w f32 RSC [3,3,C]; attrs be_dwconv_attrs;
                              out NHWC[N,P,Q,C]: y[n,p,q,c] = Σ_{r,s} x[n, p·st−pad+r, q·st−pad+s, c]·w[r,s,c]
                              (MobileNet's depthwise conv, Table 1; oracle conv2d_depthwise) */
  BE_OP_BN_CONV1X1 = 21   /* in: x NHWC[N,H,W,C] bf16, gamma[C], beta[C], running_mean[C]?, running_var[C]?, w KRSC
                              [K,1,1,C]; attrs be_bn_attrs (act 0|1|2, residual 0); out NHWC[N,H,W,K] = conv1x1(act(bn(x)), w):
                              the batch norm (train mode, as BE_OP_BATCHNORM2D) applied inside the GEMM's operand load — its
                              output never reaches HBM ("convolution, batch normalization") */
} be_op_id;

typedef struct { int act; /* 0 none, 1 relu */ int out_f32; /* 1: fp32 output even in bf16 mode */ } be_linear_attrs;
typedef struct {
  int stride, pad, act;
  int out_f32;
  int bn_stats;  /* 1: the output feeds a batchnorm2d — the conv's epilogue also produces the per-channel
                    statistics of the stored values (no bias/act only), so the BN skips its reduction pass */
} be_conv_attrs;
typedef struct { int k, stride, pad; } be_pool_attrs;
typedef struct {
  float eps, momentum;
  int act;       /* fused activation after the affine (and after the residual add): 0 none, 1 ReLU, 2 ReLU6
                    (MobileNetV2; not with residual) */
  int residual;  /* 1: the LAST input is a residual r (x's shape/dtype): y = act(bn(x) + r) — the ResNet block
                    output in one pass; r receives the gradient act'(y)·dy.
                    2: the last FIVE inputs are a second batch norm's xr, gamma_r, beta_r, running_mean_r?,
                    running_var_r? (bf16, xr of x's shape; act 0 or 1): y = act(bn(x) + bn_r(xr)) — the projection
                    block output with the shortcut's BN applied in the same pass (its output is never stored);
                    both BNs train-mode with their own statistics; xr, gamma_r, beta_r receive gradients */
} be_bn_attrs;
typedef struct { int rank; int64_t shape[6]; } be_shape_attrs;
typedef struct {
  double p;          /* drop probability in [0, 1]; p = 1 drops everything */
  int training;      /* 0: identity (eval mode) */
  uint64_t seed;     /* Philox key word 0 */
  uint64_t offset;   /* Philox counter word 1: distinct per dropout site / step */
} be_dropout_attrs;
typedef struct { int stride, pad; } be_dwconv_attrs;

be_status be_op(int op_id, const be_tensor* in, int n_in, const void* attrs,
                be_tensor* out, int n_out);

/* Grad mode (thread-local). */
be_status be_set_grad_enabled(int on);
be_status be_is_grad_enabled(int* out);
/* Compute dtype: BE_F32 (GEMMs run 3xTF32 on tcgen05; fp32 activations) or
 * BE_BF16 (GEMM/conv read a bf16 shadow of fp32 params, emit bf16
 * activations; grads and master weights stay fp32). */
be_status be_set_compute_dtype(be_dtype d);
be_status be_detach(be_tensor t, be_tensor* out);

/* ------------------------------------------------------------------ autograd
 * Reverse-mode sweep: dependency counts over the
 * reachable tape, nodes issued in reverse-topological order, saved tensors
 * version-checked at unpack (BE_E_VERSION) and released right after their
 * node ran unless retain_graph; leaf grads accumulate with +=.
 * upstream NULL requires a 1-element root (BE_E_NO_UPSTREAM). */
be_status be_backward(be_tensor root, be_tensor upstream, int retain_graph);
/* +1 reference to leaf's grad in *out, or *out = NULL when absent. */
be_status be_grad(be_tensor leaf, be_tensor* out);
/* Releases the grads (not zero-fill). */
be_status be_zero_grad(const be_tensor* params, int n);

/* ------------------------------------------------------------------ optimizer
 * One fused multi-tensor SGD launch per <=256 params:
 *   g' = scale*g + wd*p;  v = mu*v + g' (v starts at 0);  p -= lr*(mu ? v : g')
 * and, in bf16 mode, the bf16 shadow copy is rewritten in the same pass.
 * scale = 1/world_size when DDP is attached.  BE_E_MISSING_GRAD if a param
 * has no grad.  Each param's version bumps by 1. */
be_status be_sgd_step(const be_tensor* params, int n, float lr, float momentum,
                      float weight_decay);
/* Overlapped SGD (the optimizer step inside backward; "overlap
 * ... execution"): registers params (f32 leaves, one ref each is taken) for the
 * same update as be_sgd_step, applied by every later be_backward as soon as a
 * param's gradient is final (all edges to it processed), on a side stream
 * that overlaps the remaining backward kernels; with DDP attached, on the comm
 * stream right behind the param's bucket allreduce.  be_backward returns with
 * the compute stream ordered after every update, so the next op sees the new
 * values.  Results are bitwise those of be_sgd_step.  Registered params must
 * not be passed to be_sgd_step (BE_E_ARG).  n = 0 unregisters all.
 * Params that get no gradient in a backward are not updated. */
be_status be_sgd_overlap(const be_tensor* params, int n, float lr, float momentum,
                         float weight_decay);
/* Sparse SGD of embedding tables (NCF): registers
 * f32 [V, D] tables (one reference each; n = 0 unregisters all) for the
 * update p[row] -= lr·g_row applied INSIDE the embedding backward to the rows
 * the step looked up — SPEC S:581 with μ = 0, wd = 0, for which the update of
 * an untouched row (g_row = 0) is the identity, so the result equals the dense
 * step exactly.  No gradient tensor is produced (be_grad returns NULL).  With
 * a communicator of R > 1 ranks (be_dist_init) the embedding backward
 * all-gathers each rank's ids and upstream rows and applies the global-batch
 * update with g = (1/R)·Σ over all ranks' rows, in the same order on every
 * rank (replicas bitwise equal); the table must not be DDP-attached.  A table
 * whose gradient arrives densely (several lookups per step) is updated from
 * it when final (R = 1 only; else BE_E_UNSUPPORTED).  Tables may not also be
 * passed to be_sgd_overlap / be_sgd_step (BE_E_ARG). */
be_status be_sgd_sparse(const be_tensor* tables, int n, float lr);
/* The SGD momentum buffer v of f32 parameter `param` (SPEC S:578-586 update
 * above; the paper names the optimizer without formulas): *out receives a NEW
 * f32 tensor of the param's shape holding a copy of v, taken on the compute
 * stream after every update enqueued so far (caller owns one reference), or
 * NULL when no momentum step has run for this param.  Inspection / parity
 * only; BE_E_BAD_HANDLE on an invalid handle. */
be_status be_sgd_momentum(be_tensor param, be_tensor* out);

/* ------------------------------------------------------------------ allocator */
struct be_alloc_stats {
  uint64_t raw_alloc_count, raw_free_count, cache_hit_count;
  uint64_t bytes_in_use, bytes_cached, peak_bytes_in_use;
};
be_status be_alloc_stats(struct be_alloc_stats* out);
be_status be_alloc_reset_peak(void);
be_status be_empty_cache(uint64_t* bytes_released);
/* Pure helper: rounded size (512-B quantum). */
uint64_t be_round_size(uint64_t nbytes);
/* Mark that t's block is used on `stream` (cudaStream_t as uint64); its
 * reuse is deferred until an event recorded there completes. */
be_status be_record_stream(be_tensor t, uint64_t stream);
/* Raw allocator access on the compute stream (for tests of §5.3 semantics). */
be_status be_raw_alloc(uint64_t nbytes, uint64_t stream, uint64_t* dptr);
be_status be_raw_free(uint64_t dptr);

/* ------------------------------------------------------------------ data parallel
 * One process per GPU.  nccl_unique_id: 128 bytes from rank 0 (ncclGetUniqueId
 * via be_dist_unique_id), distributed by the caller (torch.distributed). */
be_status be_dist_unique_id(void* out128);
be_status be_dist_init(int rank, int world, const void* nccl_unique_id);
/* Attach params for DDP: broadcast from rank 0;
 * grads become views into fp32 buckets of ~bucket_bytes in reverse param
 * order; each bucket is all-reduced (ncclAvg: the bucket holds the MEAN
 * gradient) on a comm stream as soon as the last gradient
 * of every parameter in it is final (all tape edges into a tied / shared
 * weight have run) during backward.  be_backward returns with the compute
 * stream ordered after every bucket, so grads read afterwards are reduced and
 * a second (accumulating) backward gives mean(g1) + mean(g2).  Fails
 * (BE_E_ARG) without side effects if a param is invalid or listed twice. */
be_status be_ddp_attach(const be_tensor* params, int n, size_t bucket_bytes);
/* Broadcast f32 buffers (e.g. BatchNorm running mean / var) from rank 0 on the
 * compute stream, as data-parallel training does before each forward; BN
 * statistics used by the step stay local to each replica (DESIGN R6). */
be_status be_ddp_sync_buffers(const be_tensor* bufs, int n);
/* rank / world of the communicator (BE_E_NOT_INIT before be_dist_init). */
be_status be_dist_world(int* rank, int* world);
be_status be_ddp_detach(void);
/* Pure host function (no GPU needed): the bucket plan be_ddp_attach uses.
 * numels[n] = parameter sizes in registration order.  Buckets are filled in
 * REVERSE registration order (the order backward produces gradients) until
 * they reach bucket_bytes (fp32); each parameter's offset inside its bucket
 * is 64-element (256-B) aligned.  Outputs: bucket_of[n], offset_of[n]
 * (elements), bucket_numel[*n_buckets] (cap entries). */
be_status be_ddp_plan(const int64_t* numels, int n, size_t bucket_bytes, int* bucket_of, int64_t* offset_of,
                      int64_t* bucket_numel, int cap, int* n_buckets);
/* Peer-memory data parallelism (§5.4): the
 * bucketed gradient allreduce FUSED with the SGD update, one kernel per bucket
 * (p2p.cu) working over CUDA-IPC mappings of every rank's buckets, parameters
 * and bf16 shadows: rank r reduces its 1/R slice of the bucket by loading it
 * from every rank (NVLink peer loads, fixed rank order), applies ×1/R and the
 * overlapped-SGD update (be_sgd_overlap's lr / momentum / wd; bitwise the
 * update of be_sgd_step at R = 1) to that slice, and stores the new fp32
 * master and bf16 shadow into every rank's copy; cross-GPU barriers are
 * system-scope flags in peer memory (10 s timeout → be_p2p_status = 1).
 * Buckets whose parameters are not all registered for overlapped SGD are
 * plain mean-allreduced into the buckets instead (then be_sgd_step).
 *   be_p2p_attach: bucket params as be_ddp_attach does (NO broadcast: every
 *     rank must load identical parameters), allocate the barrier flags, create
 *     the bf16 shadows (bf16 mode) and momentum buffers, and write this rank's
 *     export blob (a header + one cudaIpcMemHandle_t per allocation) into
 *     blob (cap bytes; *blob_bytes = size needed; blob may be NULL to query).
 *   be_p2p_connect: `all` = the world blobs, rank-major, gathered by the
 *     caller over any transport (torch.distributed, gloo); maps the peers'
 *     allocations and arms DDP.  Needs no NCCL communicator.  be_ddp_detach
 *     unmaps everything. */
be_status be_p2p_attach(const be_tensor* params, int n, size_t bucket_bytes, int rank, int world, void* blob,
                        size_t cap, size_t* blob_bytes);
be_status be_p2p_connect(const void* all, size_t blob_bytes);
/* 0 healthy; 1 = some bucket kernel timed out waiting for a peer.  Synchronises. */
be_status be_p2p_status(int* status);
/* Plain allreduce (sum, fp32/bf16) of a contiguous tensor on the compute stream. */
be_status be_allreduce_(be_tensor t);

/* ------------------------------------------------------------------ profiling
 * When enabled, every GEMM / conv / SGD launch (the dominant kernel classes) is bracketed
 * by CUDA events on the stream it is launched on; be_prof_read synchronises
 * and returns one record per launch (then clears).  flops / bytes are the
 * ALGORITHMIC counts of that launch: 2·M·N·K and the operand + output bytes. */
typedef struct {
  char name[32];
  double flops, bytes;
  float ms;
  int m, n, k;
  float t_start_ms;  /* start relative to the first record's start (timeline across streams) */
} be_prof_rec;
be_status be_prof_enable(int on);
be_status be_prof_read(be_prof_rec* out, int cap, int* n_out);

/* ------------------------------------------------------------------ streams / events
 * Side streams and events for overlapping host↔device traffic with the
 * compute stream (PAPER.md:185 FIFO queues; :147-149 the data loader's
 * pinned-memory hand-off).  Handles are cudaStream_t / cudaEvent_t as uint64.
 * A tensor written on a side stream must be ordered before its use on the
 * compute stream with be_stream_wait_event(0, ev) (0 = compute stream). */
be_status be_stream_create(uint64_t* stream);
be_status be_stream_destroy(uint64_t stream);
be_status be_event_create(uint64_t* event);
be_status be_event_destroy(uint64_t event);
be_status be_event_record(uint64_t event, uint64_t stream /*0 = compute*/);
be_status be_stream_wait_event(uint64_t stream /*0 = compute*/, uint64_t event);
/* Async host→device copy into contiguous t on `stream` (0 = compute); bumps t's version. */
be_status be_tensor_copy_from_host_on(be_tensor t, const void* src, size_t nbytes, uint64_t stream);

/* ------------------------------------------------------------------ misc */
be_status be_synchronize(void);
/* Read a 1-element tensor as double (synchronises). */
be_status be_item(be_tensor t, double* out);
/* Parity hook for the bit-exact "im2col offsets" object (
 * SPEC S:113-121 conv geometry): runs the product's own im2col kernel (the
 * column builder of the stride-2 dgrad / materialised wgrad paths) on a probe
 * input whose NHWC element i holds the int32 i + 1, and returns the gathered
 * values − 1: out[M*R*S*C] int64 = the NHWC offset each column entry was
 * copied from, -1 in the zero padding.  conv_geom = {N,C,H,W,R,S,stride,pad}.
 * Synchronises.  (The implicit-GEMM conv kernels' gathers are checked through
 * the conv op itself with one-hot weights, tests/test_gpu_cnn.py.) */
be_status be_debug_im2col_offsets(const int64_t* conv_geom, int64_t* out);
/* Direct GEMM entry (tests): D[M,N] = A[M,K]·B[K,N] (+bias[N]) (act),
 * all row-major contiguous device tensors; A/B dtype f32 (3xTF32) or bf16;
 * transpose flags select Aᵀ / Bᵀ storage.  beta in {0,1}. */
be_status be_gemm(be_tensor A, int trans_a, be_tensor B, int trans_b, be_tensor D,
                  be_tensor bias, int act, float beta);

#ifdef __cplusplus
}
#endif
#endif /* BE_H_ */
