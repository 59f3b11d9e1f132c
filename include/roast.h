/*
 * roast.h — C ABI of libroast.so, the B200 (sm_100a) hot path of ROAST hashing
 * (Desai, Zhou, Shrivastava, "Efficient model compression with Random Operation
 * Access Specific Tile (ROAST) hashing", arXiv 2207.10702).
 *
 * Citations "P:n" are PAPER.md line numbers (section / equation / algorithm in
 * brackets); "R<n>" are the readings listed in DESIGN.md §Readings.
 *
 * Conventions (all entry points)
 *   - extern "C"; every call returns roast_status_t; nothing throws; no torch types.
 *   - Pointers named d_* / tensor arguments are DEVICE pointers owned by the caller,
 *     row-major and densely packed unless stated otherwise.  Pointers named *_host
 *     are host pointers.  The library never frees caller memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Every device-side effect of the compute calls is stream-ordered and
 *     asynchronous.  Calls that build or read host-side tables synchronise: the
 *     registrations (tile-map upload), roast_touched_size and the first touched
 *     exchange / touched-only update after a registration (interval tables; never
 *     under graph capture), the first autotuned launch of a shape, roast_get_error
 *     and roast_debug_tile_map.
 *   - Argument / geometry validation is synchronous: on a non-OK return nothing
 *     was launched.  Device-detected faults (embedding index out of range) are
 *     sticky and reported by roast_get_error() (and by the next call).
 *   - A handle is not thread-safe; use one per thread / rank.  Calls of one handle may be
 *     issued to several streams (e.g. dX on one, dM on another): scratch is per call
 *     (deterministic dM partials and the deterministic embedding sort are allocated with
 *     cudaMallocAsync / cudaFreeAsync on the call's stream) and a chained launch takes the
 *     next of 64 ready-counter slots, so concurrent calls never share device scratch.  The
 *     dM exchange calls (roast_grad_allreduce / _exchange_step / p2p) share the packed
 *     touched-set buffer and must stay on one stream (they are collectives anyway).
 *   - The tcgen05 GEMMs use programmatic dependent launch among themselves: each is launched
 *     with cudaLaunchAttributeProgrammaticStreamSerialization and signals
 *     griddepcontrol.launch_dependents on entry, so only a following kernel that is itself
 *     launched with that attribute (and executes griddepcontrol.wait) may start early.
 *     Ordinary launches after a ROAST call keep full stream order (ROAST_PDL=0 disables it).
 *   - roast_last_error() returns a human-readable detail string for the last
 *     non-OK status returned on the calling thread.
 *
 * The mapping (P:268-289 [§4.1], P:315, P:326 [§4.2]; concrete family: R1-R3, R8)
 *   h(key) = A * (poly61(c_off, key) mod R),  R = floor((|M| - T) / A) + 1
 *   g(key) = (poly61(c_sgn, key) & 1) ? -1 : +1
 *   poly61 = c3 k^3 + c2 k^2 + c1 k + c0 over GF(2^61 - 1),
 *   c_r    = splitmix64(seed ^ splitmix64((module << 8) | (role << 4) | r)) mod (2^61 - 1)
 *   linear tile key  (x << 32) | y        (x = i / Z1 along in_features, y = j / Z2)
 *   embedding chunk  row * ceil(d / Z) + j
 *   lambda = fp32(C / sqrt(fan_in))
 * Module ids are 0-based registration order shared by linears and embeddings;
 * they key the hash family, so registration order is part of the model.
 */
#ifndef ROAST_H_
#define ROAST_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ROAST_OK = 0,
  ROAST_ERR_CONFIG = 1,    /* invalid configuration value (C <= 0, bad enum, ...)            */
  ROAST_ERR_GEOMETRY = 2,  /* tile/chunk does not fit |M|, H % Z1 or O % Z2 != 0, T % A != 0 */
  ROAST_ERR_SHAPE = 3,     /* tensor sizes inconsistent with the module                        */
  ROAST_ERR_BOUNDS = 4,    /* embedding index outside [0, num_rows) (sticky, device-detected)  */
  ROAST_ERR_CAPACITY = 5,  /* allocation failure / too many modules                            */
  ROAST_ERR_STATE = 6,     /* not bound, unknown module id, comm not initialised, ...          */
  ROAST_ERR_CUDA = 7,      /* a CUDA runtime / driver call failed                              */
  ROAST_ERR_NCCL = 8,      /* an NCCL call failed or libnccl could not be loaded               */
  ROAST_ERR_UNSUPPORTED = 9 /* valid request with no kernel for it (bf16 off the tcgen05 path  */
                            /* without roast_config_t.simt_bf16)                               */
} roast_status_t;

typedef struct roast_ctx* roast_t;
typedef void* roast_stream_t; /* a cudaStream_t */

/* Hash-tile geometry of every linear (P:280-281 [§4.1]): Z1 rows along
 * in_features (the K dimension of Y = X W), Z2 columns along out_features.
 * Fixed at create time and part of the model (R10). */
typedef struct {
  int32_t z1, z2;
} roast_tile_t;

typedef enum { ROAST_FP32 = 0, ROAST_BF16 = 1 } roast_dtype_t;

typedef enum { ROAST_ROW_MAJOR = 0, ROAST_SW128 = 1 } roast_tile_layout_t; /* R4 */
typedef enum { ROAST_MAP_HASH = 0, ROAST_MAP_IDENTITY = 1 } roast_mapping_t; /* R22 */

typedef struct {
  double C;              /* GMS init scale: M ~ U(-1/C, 1/C), lambda = C/sqrt(n); default 1 */
  int32_t align_elems;   /* A: offsets are multiples of A elements; default 8 (16 B in bf16, R3)      */
  int32_t tile_layout;   /* roast_tile_layout_t; default ROW_MAJOR                            */
  int32_t mapping;       /* roast_mapping_t; IDENTITY = no sharing, lambda 1, g +1 (test mode)        */
  int32_t use_sign;      /* 1 = multiply by g, default 1                                       */
  int32_t deterministic; /* 1 = dM accumulated in a fixed order, bitwise reproducible (default 0)     */
  int32_t simt_bf16;     /* bf16 linears the tcgen05 path cannot take (tile != 64 x 64, SW128 layout, */
                         /* A % 8 != 0, tokens >= 2^31): 0 (default) = ROAST_ERR_UNSUPPORTED; 1 = run  */
                         /* them on the SIMT FFMA kernels (HashedNet 1 x 1 tiles, C1's 32 x 32 tiles) */
} roast_config_t;

/* Fill *cfg with the defaults listed above. */
void roast_config_default(roast_config_t* cfg);

/* Create a handle for a compressed array M of `mem_size` fp32 elements (GMS:
 * one M for every module, P:318-321 [§4.2]) with master hash seed `seed`.
 * Errors: CONFIG (mem_size <= 0, bad cfg), GEOMETRY (z1 or z2 <= 0). */
roast_status_t roast_create(roast_t* out, int64_t mem_size, uint64_t seed, roast_tile_t tile);
roast_status_t roast_create_ex(roast_t* out, int64_t mem_size, uint64_t seed, roast_tile_t tile,
                               const roast_config_t* cfg);
roast_status_t roast_destroy(roast_t h);

/* Bind the caller-owned device arrays d_M (values) and d_dM (gradient), each
 * mem_size fp32 elements, 16-byte aligned.  Allocates the library-owned bf16
 * shadow [+bf16(M) | -bf16(M)] (sign folded into the load address) and fills
 * it on `stream` (= roast_sync_shadow).  Rebinding is allowed. */
roast_status_t roast_bind(roast_t h, float* d_M, float* d_dM, roast_stream_t stream);

/* Register a ROAST linear W (in_features x out_features), Y = X W (Alg. 1
 * P:294-313).  Computes and uploads its static tile map (a0).  lambda =
 * fp32(C / sqrt(in_features)).  *id receives the module id.
 * Errors: GEOMETRY (Z1 Z2 > |M|, in % Z1, out % Z2, Z1 Z2 % A, or identity
 * mapping overflowing |M|), CAPACITY, CUDA. */
roast_status_t roast_register_linear(roast_t h, int64_t in_features, int64_t out_features, int32_t* id);

/* Register a ROAST/ROBE block embedding of num_rows x dim recovered in chunks of
 * `chunk` elements (P:268-276 [§4.1 Lookup]).  fan_in <= 0 selects dim (R7).
 * Errors: GEOMETRY (chunk > |M|, chunk % A != 0, chunk % 4 != 0, dim % 4 != 0). */
roast_status_t roast_register_embedding(roast_t h, int64_t num_rows, int32_t dim, int32_t chunk,
                                        double fan_in, int32_t* id);

/* LMS (NEXT #4): the same registrations, but the module hashes into
 * its own memory M_i = M[seg_base, seg_base + seg_size) instead of all of M (GMS,
 * P:322; roast_register_* == the _seg form with 0, |M|).  offset = seg_base +
 * A * (poly mod R_i), R_i = floor((seg_size - span) / A) + 1.  The segments of a
 * LMS model are the caller's (roast.lms_segments: |M_i| = floor(f_i |M|) aligned
 * down to A, f_i = n_i / n, remainder to the last piece - reading R23); overlapping
 * segments are legal (they share memory).  Errors: GEOMETRY (segment outside M,
 * seg_base % A != 0, span > seg_size), CONFIG (identity mapping), as above otherwise. */
roast_status_t roast_register_linear_seg(roast_t h, int64_t in_features, int64_t out_features, int64_t seg_base,
                                         int64_t seg_size, int32_t* id);
roast_status_t roast_register_embedding_seg(roast_t h, int64_t num_rows, int32_t dim, int32_t chunk,
                                            double fan_in, int64_t seg_base, int64_t seg_size, int32_t* id);

/* LMS partition ("each layer will have independent compressed memory", P:330 f_i =
 * n_i / n, sum |M_i| = |M|; reading R14/R23): piece i of the n modules, sizes[i] virtual
 * parameters each, gets |M_i| = floor(sizes[i] |M| / sum sizes) rounded down to a multiple of
 * `align` (so every base stays A-aligned), the last piece the remainder; bases are contiguous
 * from 0.  Pure host function (no handle, no GPU).  seg_base / seg_size: caller-owned host
 * arrays of n entries, written on success.  A tiny module may get size 0 (registering it then
 * fails with GEOMETRY).  Errors: CONFIG (n < 1, a size < 1, mem_size < 1, align < 1, null). */
roast_status_t roast_lms_segments(const int64_t* sizes, int32_t n, int64_t mem_size, int32_t align,
                                  int64_t* seg_base, int64_t* seg_size);

/* Fuse already-registered linears that share in_features into one GEMM along out_features
 * (e.g. BERT's Q, K, V projections of the same input): the group's virtual weight is
 * [W_1 | W_2 | ... | W_n] (in x sum out_i), its tile map the members' maps side by side, so
 * every slot, sign and lambda is the members' own (each keeps its independent hash)
 * and Y_group = [Y_1 | ... | Y_n], dX_group = sum_i dY_i W_i^T, dM += every member's
 * scatter — one launch each instead of n, over a wider N (more CTA pairs busy on small
 * layers).  *group_id is usable wherever a linear id is (fwd / fwd_bias / bwd / bwd_dx /
 * bwd_dm / tuning / debug_materialize); group ids live outside the module id space
 * (>= 2^24), so creating a group never changes the hash keys of later registrations.
 * Errors: STATE (a member is not a registered linear), SHAPE (in_features differ). */
roast_status_t roast_register_linear_concat(roast_t h, const int32_t* ids, int32_t n, int32_t* group_id);

/* Kernel-configuration autotuner (NEXT #4).  The paper autotunes its
 * tile per layer shape, either inference-optimal (tune the forward kernel, the
 * backward kernels share its tile) or training-optimal (tune forward and backward
 * kernels together).  Here the hash tile is part of the model (R10), so the tuned
 * parameter is the tcgen05 kernel configuration: WM for the forward / dX kernels and
 * (WM, split-K) for the dM kernel.  The first call for a (kernel, in, out, tokens)
 * outside CUDA-graph capture times each candidate with CUDA events on its stream
 * (synchronising the host once) and caches the winner; the dM kernel's timed runs
 * are undone (dM is snapshot and restored).  OFF (default) = the makespan model.
 * Results never depend on the choice beyond fp32 summation order. */
typedef enum { ROAST_TUNE_OFF = 0, ROAST_TUNE_INFERENCE = 1, ROAST_TUNE_TRAINING = 2 } roast_autotune_t;
roast_status_t roast_set_autotune(roast_t h, roast_autotune_t strategy);
/* The cached choice for a kernel (0 forward, 1 dX, 2 dM) of linear `id` at `tokens`:
 * *wm and *splits; for kernels 0 / 1 `splits` holds the output columns per unit / 64
 * (4 = 256; 3 = 192, with wm = 2 on 192-divisible outputs: a 768-wide output fills 64 of
 * 74 CTA pairs instead of 48; 1 = legacy, read as 4).  ROAST_ERR_STATE if that shape was
 * never tuned, BAD_ID. */
roast_status_t roast_get_tuned(roast_t h, int32_t id, int32_t kernel, int64_t tokens, int32_t* wm, int32_t* splits);
/* Seed the cache with a known choice (e.g. one tuned earlier and saved: a tuning cache
 * shared across processes); used whatever the strategy.  Errors: CONFIG (kernel not
 * 0..2, wm not 1..2, splits not 1..64, or splits not in {1, 3, 4} for kernels 0 / 1),
 * BAD_ID. */
roast_status_t roast_set_tuned(roast_t h, int32_t id, int32_t kernel, int64_t tokens, int32_t wm, int32_t splits);

/* a1: Y[tokens x out] = lambda * X[tokens x in] * W~, W~ tiles read from M
 * through the hash with sign g (Alg. 1; lambda once per output tile,
 * P:308).  dt = ROAST_FP32: X, Y fp32, SIMT FMA path on M (fp32).
 * dt = ROAST_BF16: X, Y bf16, tcgen05 path on the bf16 shadow (requires
 * Z1 = Z2 = 64, in % 64 == 0, out % 64 == 0, tokens any >= 0), fp32 accumulate. */
roast_status_t roast_linear_fwd(roast_t h, int32_t id, const void* d_X, void* d_Y, int64_t tokens,
                                roast_dtype_t dt, roast_stream_t stream);

/* a1 with a bias (NEXT #3): Y = lambda X W~ + b, b added in fp32 inside the GEMM
 * epilogue before the single rounding to the output type.  d_bias: out_features fp32
 * on the device, 16-byte aligned, or NULL (== roast_linear_fwd).  A model whose bias
 * is ROAST-compressed gets b from roast_bias_fwd. */
roast_status_t roast_linear_fwd_bias(roast_t h, int32_t id, const void* d_X, void* d_Y, int64_t tokens,
                                     roast_dtype_t dt, const float* d_bias, roast_stream_t stream);

/* Two dependent linears in ONE persistent tcgen05 launch (C2's MLP block: in -> a -> b).
 *   fwd_chain:    Y_a = lambda_a X W~_a (+ bias_a),  Y_b = lambda_b Y_a W~_b (+ bias_b)
 *   bwd_dx_chain: dY_a = lambda_b dY_b W~_b^T,       dX = lambda_a dY_a W~_a^T
 * Same results as the two single calls (each output rounded once); Y_a / dY_a are still
 * written (the backward needs them).  The second GEMM's work units start on CTA pairs the
 * first leaves idle and wait per output tile of the first (ready counters), filling the
 * quantisation gaps each launch has alone.  Shapes that are not on the tcgen05 path, or for
 * which the scheduler predicts no gain, run as two launches.  The first call for a shape
 * must not be under stream capture to chain (it plans and uploads a static schedule).
 * Requires out_features(a) == in_features(b).  Errors as roast_linear_fwd / _bwd_dx. */
roast_status_t roast_linear_fwd_chain(roast_t h, int32_t id_a, int32_t id_b, const void* d_X, void* d_Y_a,
                                      void* d_Y_b, int64_t tokens, roast_dtype_t dt, const float* d_bias_a,
                                      const float* d_bias_b, roast_stream_t stream);
roast_status_t roast_linear_bwd_dx_chain(roast_t h, int32_t id_a, int32_t id_b, const void* d_dY_b, void* d_dY_a,
                                         void* d_dX, int64_t tokens, roast_dtype_t dt, roast_stream_t stream);

/* The whole backward of a chained pair a -> b (the backward of roast_linear_fwd_chain, with
 * the identity between the layers): given X_a, Y_a (= X_b) and dY_b,
 *   dY_a = lambda_b dY_b W~_b^T                 (a2 of b; written to d_dY_a, tokens x in_b)
 *   dM  += scatter_b(lambda_b g Y_a^T dY_b)     (a3 of b)
 *   dX_a = lambda_a dY_a W~_a^T                 (a2 of a; written to d_dX_a, tokens x in_a)
 *   dM  += scatter_a(lambda_a g X_a^T dY_a)     (a3 of a)
 * (P:338-346 with g by the chain rule, R12).  On the tcgen05 path (bf16, 64 x 64 tiles, every
 * feature dimension a multiple of 256, fast / atomic dM) the four GEMMs run as ONE persistent
 * launch: their units are list-scheduled over all CTA pairs and the dependent ones (dX_a, the
 * dM of a) stream behind the published tiles of dY_a; otherwise the four calls run one after
 * the other.  Requires out_a == in_b; d_dX_a must not be NULL.  The first call of a shape plans
 * the schedule (synchronous; not under graph capture).  Errors as roast_linear_bwd. */
roast_status_t roast_linear_bwd_chain(roast_t h, int32_t id_a, int32_t id_b, const void* d_X_a, const void* d_Y_a,
                                      const void* d_dY_b, void* d_dY_a, void* d_dX_a, int64_t tokens,
                                      roast_dtype_t dt, roast_stream_t stream);

/* Bias vectors via L ("ROAST uses L to implement ... bias vectors").  A bias of
 * n elements is row 0 of an embedding registered as (num_rows 1, dim n, chunk Z,
 * fan_in = the owning layer's in_features, reading R24).
 *   roast_bias_fwd:  d_b[0..n) = row 0 of bias_id (== roast_embedding_fwd of index 0).
 *   roast_bias_bwd:  dM[h1(c) + o] += lambda g(c) sum_t dY[t, jZ + o]  (P:340 with
 *                    dOut = the column sums of dY [tokens x n], bf16 or fp32, fp32
 *                    accumulation in a fixed order; deterministic mode as a5).
 * Errors: BAD_ID (not an embedding), CONFIG (null / unaligned: d_b 16 B, dY 8 B), SHAPE. */
roast_status_t roast_bias_fwd(roast_t h, int32_t bias_id, float* d_b, roast_stream_t stream);
roast_status_t roast_bias_bwd(roast_t h, int32_t bias_id, const void* d_dY, int64_t tokens, roast_dtype_t dt,
                              roast_stream_t stream);
/* The same with dY rows `ld` elements apart (ld >= the bias length, even): the bias of one
 * member of a roast_register_linear_concat group reads its column slice of the group's dY. */
roast_status_t roast_bias_bwd_ld(roast_t h, int32_t bias_id, const void* d_dY, int64_t tokens, int64_t ld,
                                 roast_dtype_t dt, roast_stream_t stream);
/* The first half of the bias backward alone: db[j] = sum_t dY[t, j] (fp32, fixed order; rows
 * `ld` elements apart, -1 = n; n and ld even; db 8-byte aligned, caller-owned, overwritten).
 * A model with many biases via L (BERT: 72) collects every bias's db this way and scatters
 * them all with one roast_embedding_bwd_multi per (dim, chunk) group (row 0 of each 1 x n
 * table) instead of one L backward per bias. */
roast_status_t roast_colsum(const void* d_dY, int64_t tokens, int32_t n, int64_t ld, roast_dtype_t dt, float* d_db,
                            roast_stream_t stream);
/* As roast_colsum, but db[j] += sum_t dY[t, j] (accumulate != 0) instead of overwriting: a
 * bias whose layer runs backward more than once before the scatter (gradient accumulation
 * over micro-batches, a module applied twice) keeps every contribution. */
roast_status_t roast_colsum_ex(const void* d_dY, int64_t tokens, int32_t n, int64_t ld, roast_dtype_t dt, float* d_db,
                               int32_t accumulate, roast_stream_t stream);

/* Activation fused into the linear's epilogue (the ROASTed BERT MLP, SURVEY.md §8(f) NEXT #3;
 * the activation itself is an N-operation).  bf16 on the tcgen05 path only (the
 * WM = 2 register-held epilogue); ROAST_ERR_UNSUPPORTED elsewhere (the caller applies the
 * activation itself).  act: ROAST_ACT_GELU_TANH, gelu(u) = u/2 (1 + tanh(sqrt(2/pi)(u + 0.044715
 * u^3))) (torch's gelu(approximate="tanh"), the original BERT's form), tanh evaluated with the
 * hardware approximation (rel. error ~2^-11, below bf16's 2^-8).
 * roast_linear_fwd_act: Y = lambda X W~ (+ bias) as roast_linear_fwd_bias, and A = act(Y) from
 *   the stored (bf16-rounded) Y, both [tokens x out_features] bf16; A 16-byte aligned.
 * roast_linear_bwd_dx_act: dX = bf16(lambda dY W~^T) * act'(U) elementwise, U [tokens x
 *   in_features] bf16 the pre-activation whose act(U) was this layer's input (so dX is the
 *   gradient with respect to U).  No dM: pair it with roast_linear_bwd_dm(X = act(U)).
 *   act = ROAST_ACT_RESIDUAL (this call only): U is R, the gradient the layer input also
 *   receives through a residual connection, and dX = bf16(bf16(lambda dY W~^T) + R) — the bits
 *   of the dX GEMM followed by a separate bf16 add, in one pass (U may alias dX). */
typedef enum { ROAST_ACT_NONE = 0, ROAST_ACT_GELU_TANH = 1, ROAST_ACT_RESIDUAL = 2 } roast_act_t;
roast_status_t roast_linear_fwd_act(roast_t h, int32_t id, const void* d_X, void* d_Y, void* d_A, int64_t tokens,
                                    roast_dtype_t dt, const float* d_bias, int32_t act, roast_stream_t stream);
roast_status_t roast_linear_bwd_dx_act(roast_t h, int32_t id, const void* d_dY, const void* d_U, void* d_dX,
                                       int64_t tokens, roast_dtype_t dt, int32_t act, roast_stream_t stream);
/* The MLP pair b(act(a(X))) with the activation inside the chained launches (as
 * roast_linear_fwd_chain / roast_linear_bwd_chain):
 * roast_linear_fwd_chain_act: U = a(X) (+ bias_a), A = act(U), Y_b = b(A) (+ bias_b); one launch
 *   on the tcgen05 path (b's units stream behind a's published tiles of A), else
 *   roast_linear_fwd_act + roast_linear_fwd_bias.
 * roast_linear_bwd_chain_act: dU = (dY_b W~_b^T) * act'(U), dM += b(A, dY_b), dX_a = dU W~_a^T,
 *   dM += a(X_a, dU); one launch on the tcgen05 path, else the four calls. */
roast_status_t roast_linear_fwd_chain_act(roast_t h, int32_t id_a, int32_t id_b, const void* d_X, void* d_U,
                                          void* d_A, void* d_Y_b, int64_t tokens, roast_dtype_t dt,
                                          const float* d_bias_a, const float* d_bias_b, int32_t act,
                                          roast_stream_t stream);
roast_status_t roast_linear_bwd_chain_act(roast_t h, int32_t id_a, int32_t id_b, const void* d_X_a, const void* d_A,
                                          const void* d_U, const void* d_dY_b, void* d_dU, void* d_dX_a,
                                          int64_t tokens, roast_dtype_t dt, int32_t act, roast_stream_t stream);

/* LayerNorm of the ROASTed BERT workload (an N-operation, P:263-265,
 * not part of the ROAST hashing itself): at C3's 65 536 tokens torch's LayerNorm takes 0.85 ms
 * per call, more than the layer's ROAST GEMMs.  Rows of n features, n % 8 == 0, n <= 2048
 * (else ROAST_ERR_SHAPE); 16-byte aligned device arrays; dt = activations, pdt = gamma / beta.
 * roast_layernorm_fwd: s = x + r (r may be NULL: s = x; with r, s is rounded to dt and written to
 *   s_out [rows x n], the input the backward needs), y = (s - mean) * rstd * gamma + beta with
 *   mean / rstd (fp32 [rows], outputs) over the row, rstd = 1 / sqrt(var + eps).
 * roast_layernorm_bwd: from dy and the LN input s (x, or s_out): ds = d(loss)/ds [rows x n] dt
 *   (with a residual it is the gradient of x and of r alike), dgamma / dbeta fp32 [n]
 *   (overwritten) = column sums of dy * xhat / dy in a fixed order (bitwise reproducible).
 *   Scratch per call (cudaMallocAsync on the stream).  Stream-ordered, capturable. */
roast_status_t roast_layernorm_fwd(const void* d_x, const void* d_r, const void* d_gamma, const void* d_beta, void* d_y,
                                   void* d_s_out, float* d_mean, float* d_rstd, int64_t rows, int32_t n, float eps,
                                   roast_dtype_t dt, roast_dtype_t pdt, roast_stream_t stream);
roast_status_t roast_layernorm_bwd(const void* d_dy, const void* d_s, const void* d_gamma, const float* d_mean,
                                   const float* d_rstd, void* d_ds, float* d_dgamma, float* d_dbeta, int64_t rows,
                                   int32_t n, roast_dtype_t dt, roast_dtype_t pdt, roast_stream_t stream);

/* a2 + a3: dX = lambda * dY W~^T (skipped if d_dX == NULL), and
 * dM[h(x,y) + pi(o1,o2)] += lambda * g(x,y) * (X^T dY)[i, j] for every virtual
 * weight (P:338-346 [§4.3 eq. gradient rule] with g by the chain rule, R12),
 * without materialising W.  dM accumulates (+=).  Deterministic
 * mode sums every slot in a fixed order (bitwise reproducible). */
roast_status_t roast_linear_bwd(roast_t h, int32_t id, const void* d_X, const void* d_dY, void* d_dX,
                                int64_t tokens, roast_dtype_t dt, roast_stream_t stream);
/* roast_linear_bwd_fused: the same result as roast_linear_bwd with dX (dX overwritten, dM +=),
 * computed on the tcgen05 path by ONE persistent launch that co-schedules the dX GEMM's and the
 * dM GEMM's units over the CTA pairs when its plan beats the two launches (small token counts:
 * a 768-wide dX has 48 units of 512 x 256 for 74 pairs), else by the two launches.  dX is
 * required (ROAST_ERR_CONFIG if NULL).  Fast mode only; in deterministic mode it is exactly
 * roast_linear_bwd.  Plans are made on an eager call (not under stream capture). */
roast_status_t roast_linear_bwd_fused(roast_t h, int32_t id, const void* d_X, const void* d_dY, void* d_dX,
                                      int64_t tokens, roast_dtype_t dt, roast_stream_t stream);

/* The two halves of roast_linear_bwd, for callers that overlap them on two
 * streams (dX is on the critical path of the previous layer, dM is not):
 * a2 alone: dX = lambda * dY W~^T;  a3 alone: dM += scatter(lambda g X^T dY). */
roast_status_t roast_linear_bwd_dx(roast_t h, int32_t id, const void* d_dY, void* d_dX, int64_t tokens,
                                   roast_dtype_t dt, roast_stream_t stream);
roast_status_t roast_linear_bwd_dm(roast_t h, int32_t id, const void* d_X, const void* d_dY, int64_t tokens,
                                   roast_dtype_t dt, roast_stream_t stream);

/* a4: out[b, jZ + o] = g(c) * fp32(lambda * M[h1(c) + o]),  c = idx[b] * ceil(d/Z) + j
 * (P:270).  idx: n int64 device indices; out: n x dim fp32.  An index outside
 * [0, num_rows) yields a zero row and raises the sticky BOUNDS flag. */
roast_status_t roast_embedding_fwd(roast_t h, int32_t id, const int64_t* d_idx, int64_t n, float* d_out,
                                   roast_stream_t stream);

/* a5: dM[h1(c) + o] += lambda * g(c) * dOut[b, jZ + o]; duplicate indices add (R15). */
roast_status_t roast_embedding_bwd(roast_t h, int32_t id, const int64_t* d_idx, int64_t n,
                                   const float* d_dOut, roast_stream_t stream);

/* a4 / a5 over several tables in one launch (DLRM's 26 sparse features, C4):
 * table t = ids[t] (host array of ntables embedding ids, all with the same dim and
 * chunk; a table may repeat) looks up idx[t n + b]; batch rows are table-major, so
 * d_idx is ntables x n int64, d_out / d_dOut are (ntables n) x dim fp32 and row
 * t n + b equals roast_embedding_fwd(ids[t], idx[t n + b]) bit for bit.  Backward
 * adds every table's gradient into dM (the same sum as ntables single calls, up to
 * fp32 rounding order).  Deterministic mode sorts the items of up to 32 tables together
 * (groups of 32 in table order beyond that): bitwise reproducible run to run, but the
 * per-slot order differs from ntables single calls, so the two agree only to rounding.
 * Errors: CONFIG (null / unaligned pointers, ids of differing dim or chunk), BAD_ID,
 * SHAPE. */
roast_status_t roast_embedding_fwd_multi(roast_t h, const int32_t* ids, int32_t ntables, const int64_t* d_idx,
                                         int64_t n, float* d_out, roast_stream_t stream);
roast_status_t roast_embedding_bwd_multi(roast_t h, const int32_t* ids, int32_t ntables, const int64_t* d_idx,
                                         int64_t n, const float* d_dOut, roast_stream_t stream);

/* a6: data-parallel exchange.  Rank 0 calls roast_comm_unique_id; the caller
 * broadcasts the 128 bytes (e.g. torch.distributed); every rank calls
 * roast_comm_init.  roast_grad_allreduce sums dM over ranks in place
 * (ncclAllReduce, fp32 sum) on `stream`.  world == 1 with id == NULL creates no communicator
 * and the exchange is a no-op; world == 1 with an id builds a 1-rank NCCL communicator.
 * libnccl.so.2 is loaded at run time (ROAST_ERR_NCCL if absent). */
roast_status_t roast_comm_unique_id(uint8_t id_out[128]);
/* In deterministic mode roast_comm_init sets NCCL_ALGO=Ring (unless already set) before
 * creating the communicator, so the cross-rank sum is taken in a fixed order run to run. */
roast_status_t roast_comm_init(roast_t h, int32_t rank, int32_t world, const uint8_t id[128]);
roast_status_t roast_grad_allreduce(roast_t h, roast_stream_t stream);

/* a6 in the large-|M| regime ("communication is directly
 * proportional to model size"): the touched-set exchange.  Offsets are static, so the
 * slots any rank can write are the union of [off_t, off_t + Z1 Z2) over every linear's
 * tiles plus, per embedding, its exact chunks (tables of <= 2^16 chunks, e.g. biases
 * via L) or its whole memory (GMS: all of M; LMS: its segment).  All other slots of dM
 * are zero on every rank.  In TOUCHED mode roast_grad_allreduce packs the touched
 * intervals (a library-owned fp32 buffer), all-reduces the packed buffer and unpacks it:
 * the same sum, with NVLink traffic <= min(|M|, n) elements.  AUTO (default) picks
 * TOUCHED when the touched set is at most |M| / 2, else DENSE.  The interval tables are
 * built on the host on first use after a registration (synchronous); under CUDA-graph
 * capture they must already exist (call roast_touched_size first), else ROAST_ERR_STATE.
 * Slots outside the touched set are neither read nor written by the exchange. */
typedef enum { ROAST_EXCHANGE_AUTO = 0, ROAST_EXCHANGE_DENSE = 1, ROAST_EXCHANGE_TOUCHED = 2 } roast_exchange_mode_t;
roast_status_t roast_set_exchange(roast_t h, int32_t mode);
/* Builds the interval tables if needed; *n_touched = elements in the touched set,
 * *n_intervals = disjoint intervals (either pointer may be NULL). */
roast_status_t roast_touched_size(roast_t h, int64_t* n_touched, int64_t* n_intervals);
/* Host utility (no GPU, no handle): merge [starts_in[i], starts_in[i] + span) into sorted
 * disjoint, non-adjacent intervals -> starts_out / lens_out (host arrays of cap entries);
 * *count = number of intervals.  ROAST_ERR_CAPACITY (count still set) if count > cap. */
roast_status_t roast_touched_intervals(const int64_t* starts_in, int64_t n, int64_t span, int64_t* starts_out,
                                       int64_t* lens_out, int64_t cap, int64_t* count);

/* dM <- 0. */
roast_status_t roast_zero_grad(roast_t h, roast_stream_t stream);
/* shadow <- [+bf16_RNE(M) | -bf16_RNE(M)]; call after every update of M (H7). */
roast_status_t roast_sync_shadow(roast_t h, roast_stream_t stream);
/* (a7, minimal) M <- M - lr * dM, then shadow refresh.  Fused elementwise kernel. */
roast_status_t roast_sgd_step(roast_t h, float lr, roast_stream_t stream);

/* NEXT #1: the update after the exchange, fused into ONE elementwise pass
 * over |M| (`tab:total-opt` P:749-813: optimizer cost scales with |M|, not with
 * the virtual model): read M, dM and the optimizer state, write M, the bf16 shadow
 * [+bf16(M) | -bf16(M)], the state, and (zero_grad != 0) dM <- 0.  State (fp32, |M|
 * elements each) is owned by the handle and allocated on first use.  Formulas are
 * PyTorch's (the paper's optimizers): with g = dM + weight_decay * M,
 *   SGD      M -= lr g
 *   ADAGRAD  G += g^2;                      M -= lr g / (sqrt(G) + eps)
 *   ADAM     m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
 *            M -= lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)     (t = step >= 1). */
typedef enum { ROAST_OPT_SGD = 0, ROAST_OPT_ADAGRAD = 1, ROAST_OPT_ADAM = 2 } roast_opt_kind_t;
typedef struct {
  int32_t kind;        /* roast_opt_kind_t */
  float lr, beta1, beta2, eps, weight_decay;
  int32_t zero_grad;   /* 1: dM <- 0 in the same pass */
  int32_t touched_only;/* 1: visit only the touched set of roast_touched_size ("the
                          same restriction applies to zeroing and updates"); slots outside it are
                          never read by any module, so every model output is unchanged, at
                          O(touched) instead of O(|M|) cost.  Under capture the tables must exist. */
} roast_opt_config_t;
roast_status_t roast_optimizer_step(roast_t h, const roast_opt_config_t* cfg, int64_t step, roast_stream_t stream);

/* NEXT #1, the exchange fused with its consumer: a6 + the update in one call.  Dense
 * exchange (see roast_set_exchange): in-place ncclAllReduce of dM, then the optimizer pass
 * over |M|.  Touched exchange (AUTO / TOUCHED mode, or cfg->touched_only): pack the touched
 * intervals, all-reduce the packed buffer, and the optimizer pass over the touched slots
 * reads the summed gradient directly from the packed buffer (the unpack pass and its dM
 * round trip disappear) and zeroes dM there.  Same M, state and shadow as
 * roast_grad_allreduce + roast_optimizer_step (touched_only = the mode's choice) bit for bit.
 * Without a communicator (world 1) the exchange is the identity.  dM afterwards: zero on
 * the touched slots if zero_grad, else the summed gradient.  Errors as roast_optimizer_step. */
roast_status_t roast_grad_exchange_step(roast_t h, const roast_opt_config_t* cfg, int64_t step,
                                        roast_stream_t stream);

/* ---- one-shot P2P exchange fused with the update ---
 * The a6 exchange and the a7 update in one pass without NCCL:
 * every rank maps every other rank's exchange window (CUDA IPC over NVLink / NVSwitch), and
 * the update kernel reads the W packed gradients of the touched slots straight from the
 * peers' memory, sums them in rank order 0..W-1 (so all ranks get bit-identical sums and M
 * stays replicated), and applies the optimizer, the bf16 shadow refresh and the dM zeroing.
 * Only the touched slots (roast_touched_size) are exchanged and updated, as in
 * roast_grad_exchange_step with touched_only.  All calls below after every module is
 * registered; re-registering invalidates the window (ROAST_ERR_STATE until re-opened).
 *
 * roast_p2p_window: allocate (once) this handle's window, a device buffer the library owns:
 *   [0, 128) int32 flags[world] | [128, 256) int32 flags2[world] (two-shot) |
 *   [256, 512) int32 epoch, uint32 arrival counter | [512, ...) three fp32 buffers of
 *   the touched-slot count (rounded up to 4) each; flags and epoch start at 0.  *window /
 *   *bytes (either may be NULL) receive its device address and size.
 * roast_p2p_ipc_handle: the window's cudaIpcMemHandle (64 bytes, host buffer) for the other
 *   ranks of the node (exchange them out of band, e.g. torch.distributed all_gather).
 * roast_p2p_open: map every rank's window from handles[world * 64] (rank r's handle at
 *   r * 64; this rank's own entry is ignored).  1 <= world <= 8, else ROAST_ERR_CONFIG;
 *   ROAST_ERR_CUDA if a handle cannot be opened.
 * roast_p2p_attach: the same with device pointers windows[world] already mapped in this
 *   process (ranks sharing a process; windows[rank] must be this handle's window).
 * roast_p2p_post (stream-ordered, capturable): pack this rank's dM touched slots into
 *   buffer (epoch + 1) & 1, then (its last CTA) publish epoch + 1 in every rank's
 *   flags[rank] (release, system scope) and advance the epoch.  1 launch.
 * roast_p2p_finish (stream-ordered, capturable): wait until every rank has posted this epoch
 *   (acquire, system scope), then the fused sum + update (cfg as roast_optimizer_step; dM on
 *   the touched slots afterwards: zero if zero_grad, else the summed gradient).  1 launch.
 *   A rank that never posts: after 20 s the kernel sets the sticky error (roast_get_error ->
 *   ROAST_ERR_STATE) and traps, so the context reports an error instead of hanging.
 * roast_grad_exchange_p2p: post + finish.  Every rank must call it once per step, in the same
 *   order as the other ranks; ranks sharing one stream must post all before finishing any. */
roast_status_t roast_p2p_window(roast_t h, void** window, int64_t* bytes);
roast_status_t roast_p2p_ipc_handle(roast_t h, uint8_t handle[64]);
roast_status_t roast_p2p_open(roast_t h, int32_t rank, int32_t world, const uint8_t* handles);
roast_status_t roast_p2p_attach(roast_t h, int32_t rank, int32_t world, void* const* windows);
roast_status_t roast_p2p_post(roast_t h, roast_stream_t stream);
roast_status_t roast_p2p_finish(roast_t h, const roast_opt_config_t* cfg, int64_t step, roast_stream_t stream);
roast_status_t roast_grad_exchange_p2p(roast_t h, const roast_opt_config_t* cfg, int64_t step,
                                       roast_stream_t stream);

/* Two-shot variant (same window, same post): the one-shot finish reads (W - 1) n values
 * from the peers per rank, which for large touched sets is more NVLink traffic than a ring
 * (2 (W - 1) / W n).  Here rank r owns the packed-index slice [r per, (r + 1) per),
 * per = ceil(n / W) rounded up to 4:
 * roast_p2p_reduce: wait for every post, sum the slice's gradients over the ranks (rank
 *   order), update M / optimizer state / shadow / dM (zeroed) on the slice, copy the new
 *   values into this rank's M buffer, then publish flags2 on every rank.  2 launches.
 * roast_p2p_gather: wait for every rank's flags2, copy the other slices' new values from
 *   the owners' M buffers into M at the touched slots, refresh the shadow, zero dM.  1 launch.
 * roast_grad_exchange_p2p2: post + reduce + gather.  Result bit-identical to the one-shot
 * path for M and the shadow.  The optimizer state of a slice lives on its owner only, so keep
 * one variant and one world size for a whole run.  zero_grad must be 1 (else
 * ROAST_ERR_CONFIG).  Ranks sharing one stream: post all, reduce all, then gather all. */
roast_status_t roast_p2p_reduce(roast_t h, const roast_opt_config_t* cfg, int64_t step, roast_stream_t stream);
roast_status_t roast_p2p_gather(roast_t h, roast_stream_t stream);
roast_status_t roast_grad_exchange_p2p2(roast_t h, const roast_opt_config_t* cfg, int64_t step,
                                        roast_stream_t stream);

/* NVLS variant (the a6 exchange P:194 fused with the a7
 * update P:440).  On an NVSwitch system the exchange windows of all ranks can be
 * bound to one multicast object: the finish / reduce kernels then read the SUM over the ranks
 * with multimem.ld_reduce (reduced in the switch, one NVLink read per value instead of W - 1),
 * the two-shot reduce broadcasts its slice's new values with multimem.st (the gather reads only
 * local memory), and the flags are written to every rank by one multimem.st.  Once bound, the
 * p2p entry points above run the NVLS kernels unchanged in meaning: roast_grad_exchange_p2p
 * (one-shot: every rank reduces all n values in the switch and updates all of M; replication
 * then relies on the switch returning the same fp32 sum to every rank) and
 * roast_grad_exchange_p2p2 (two-shot: only a slice's owner computes its update and broadcasts
 * it, so M stays replicated bit for bit by construction).  Set-up, after every module is
 * registered, all ranks in this order:
 * roast_nvls_supported: *supported = CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED of `device` (0 when
 *   the driver lacks the multicast entry points).  Never fails for a valid pointer.
 * roast_nvls_create (rank 0): cuMulticastCreate for `world` devices (1..8), sized for this
 *   handle's window (layout as roast_p2p_window); *fd = a POSIX file descriptor of the object,
 *   owned by the caller (send it to the other ranks, e.g. SCM_RIGHTS; close it afterwards).
 * roast_nvls_import (ranks != 0): import the object from the descriptor received.
 * roast_nvls_add_device: add this handle's device.  Every rank must return from it before any
 *   rank calls roast_nvls_bind.
 * roast_nvls_bind: allocate this rank's window (cuMemCreate), bind it to the object, map its
 *   unicast and multicast aliases and zero it; the window then replaces the P2P one (open /
 *   attach return ROAST_ERR_STATE).  Barrier all ranks before the first exchange.
 * roast_nvls_bound: *bound = 1 once roast_nvls_bind succeeded.
 * roast_nvls_reset: release this handle's multicast object / window in any set-up state (a rank
 *   whose peers failed a step backs out this way); the next P2P call allocates a fresh window.
 * Errors: ROAST_ERR_UNSUPPORTED without the driver entry points; ROAST_ERR_CUDA with the
 * CUresult when the driver refuses a step (e.g. no NVSwitch multicast); a failed bind undoes
 * everything, so the handle stays usable on the P2P and NCCL paths (the binding's fallback). */
roast_status_t roast_nvls_supported(int32_t device, int32_t* supported);
roast_status_t roast_nvls_create(roast_t h, int32_t world, int32_t* fd);
roast_status_t roast_nvls_import(roast_t h, int32_t world, int32_t fd);
roast_status_t roast_nvls_add_device(roast_t h);
roast_status_t roast_nvls_bind(roast_t h, int32_t rank);
roast_status_t roast_nvls_bound(roast_t h, int32_t* bound);
roast_status_t roast_nvls_reset(roast_t h);

/* Sticky device-side error (synchronises the handle's bound stream is NOT done:
 * call after a stream synchronize to observe faults of completed work). */
roast_status_t roast_get_error(roast_t h);
const char* roast_status_str(roast_status_t st);
const char* roast_last_error(void);

/* ---- test hooks (parity tier T1) ---------------------------------------- */
/* Copy module `id`'s tile map to host: off_host[x * ny + y], sgn_host[x * ny + y]
 * (nx = in/Z1, ny = out/Z2).  Synchronous. */
roast_status_t roast_debug_tile_map(roast_t h, int32_t id, int64_t* off_host, int8_t* sgn_host);
/* Evaluate the embedding kernels' __device__ chunk hash for n rows: d_off / d_sgn
 * are n x ceil(dim/chunk) device arrays. */
roast_status_t roast_debug_chunk_map(roast_t h, int32_t id, const int64_t* d_rows, int64_t n,
                                     int64_t* d_off, int8_t* d_sgn, roast_stream_t stream);
/* Recovered W (in x out) on device.  dt = FP32: g * fp32(lambda * M) (fp32 def.);
 * dt = BF16: g * bf16(M) read from the shadow (the tensor-core operand, lambda deferred). */
roast_status_t roast_debug_materialize(roast_t h, int32_t id, roast_dtype_t dt, void* d_W,
                                       roast_stream_t stream);

/* Test hook: copy the optimizer state of roast_optimizer_step to the host.  which = 0: the
 * first state array (Adagrad G, Adam m), 1: the second (Adam v); out_host: mem_size fp32.
 * Synchronous.  Errors: STATE (not bound, or that state was never allocated). */
roast_status_t roast_debug_opt_state(roast_t h, int32_t which, float* out_host);
/* Evaluate the library's hash (the same __host__ __device__ code the kernels run,
 * including the reciprocal `mod R`) on the HOST for n keys of module `module`:
 * off_out[i] = A * (poly(key) mod R), R = floor((mem_size - span)/align) + 1, and
 * sgn_out[i] = g(key).  Needs no GPU (CPU parity tests).  keys < 2^60. */
roast_status_t roast_debug_hash_host(uint64_t seed, int32_t module, const uint64_t* keys_host, int64_t n,
                                     int64_t mem_size, int64_t span, int32_t align, int32_t use_sign,
                                     int64_t* off_out_host, int8_t* sgn_out_host);
/* Touched-set exchange without NCCL: pack dM's touched intervals, then unpack them
 * scaled: dM[touched] *= scale, every other slot untouched (tests the interval maps on
 * one GPU). */
roast_status_t roast_debug_exchange(roast_t h, float scale, roast_stream_t stream);
/* Number of kernels this handle has launched since creation (bench evidence). */
int64_t roast_launch_count(roast_t h);

#ifdef __cplusplus
}
#endif

#endif /* ROAST_H_ */
