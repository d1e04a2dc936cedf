/*
 * lsw.h -- C ABI of the B200-native LoRA-Switch hot path (arXiv 2405.17741).
 *
 * The paper's statement of the problem (Alg. 1, P:296-309 of PAPER.md): at
 * token t, given the input token and all model parameters, (1) compute the
 * pre-gate G^1(x^1) once (Eq. 2), (2-4) switch every adapted linear of
 * every layer in ONE kernel (Eq. 5/9/10, SGMM Eq. 11, "a single CUDA
 * kernel operation", in place P:328), (5) run the plain backbone forward on the
 * merged weights (Eq. 3).  This library implements steps 1-5 for the
 * adapted linears (q,k,v,o,gate,up,down) as four calls:
 *
 *     lsw_router_topk         Eq. 2                       (kernel K2)
 *     lsw_merge_all_layers    Eq. 6 (first token) / Eq. 10 (fused switch) (K1)
 *     lsw_unmerge_all_layers  Eq. 7 (end of sequence)     (K1)
 *     lsw_decode_linear       Eq. 3, one batch-1 GEMV     (K4) [+ NCCL allreduce under TP]
 *
 * plus grouped / whole-token conveniences built only from those kernels.
 *
 * Conventions (all calls)
 *  - Memory: every tensor pointer is CALLER-OWNED DEVICE memory (allocated by
 *    the caller, e.g. torch), borrowed for the lifetime of the ctx, unless the
 *    parameter name ends in _h (HOST memory, ideally pinned).  The ctx owns only
 *    its own state: the merged-decision slots, the device error latch, packed
 *    tensor-core operand copies of the LoRA factors (see lsw_create), TMA
 *    descriptors, staging buffers and the NCCL communicator.
 *  - Layouts (row-major, C order, contiguous):
 *      W[kind]  [L, d_out, d_in]   backbone weight f (nn.Linear layout), MUTATED IN PLACE
 *      A[kind]  [L, N, r, d_in]    LoRA_DOWN bank (P:139 W_down)
 *      B[kind]  [L, N, d_out, r]   LoRA_UP   bank (P:139 W_up)
 *      router_w [N, d_model]       W_g, the single pre-gate at the first
 *                                  expanded linear
 *    d_out/d_in are this rank's LOCAL (tensor-parallel shard) sizes.
 *  - dtype: LSW_BF16 (W, A, B, router_w and every x are bf16) or LSW_F32 (all
 *    fp32).  Accumulation is fp32 (GEMV, switch) / fp64 (router logits); one
 *    round-to-nearest-even store of W per pass.
 *  - Update (Eq. 4-10, readings R1-R3 of DESIGN.md):
 *      W <- RNE( W + sum_j c_j * B[e_j] @ A[e_j] )
 *    with c_j = (alpha/r) * g_j for the current decision and -(alpha/r) * g_j for
 *    the previously merged one (Eq. 9 with its double negation corrected: the
 *    sign is on the coefficient).  Experts present in both decisions are
 *    combined into one term c = (alpha/r)(g_t - g_{t-1}); terms with c == 0 are
 *    dropped, so prev == cur is an exact no-op (R12).
 *  - Asynchrony: hot calls validate their arguments on the host, then only
 *    ENQUEUE work on `stream` (a cudaStream_t; NULL = legacy default stream) and
 *    return.  Decisions (idx, gate) never come back to the host, so a token is
 *    CUDA-graph capturable.  Exceptions: lsw_device_status and
 *    lsw_decode_token_host synchronize `stream`.
 *  - Errors: argument / shape / state errors are returned synchronously BEFORE
 *    anything is enqueued (LSW_E_ARG / LSW_E_SHAPE / LSW_E_STATE), with a
 *    message in lsw_last_error() (thread-local) naming the offending values.
 *    Errors detected on the device (non-finite router logits, expert index out
 *    of range or duplicated, non-finite gate) are LATCHED in the ctx; the
 *    affected kernel becomes a no-op (W untouched); lsw_device_status() reports
 *    and clears the latch.  No exception crosses the ABI, nothing is printed,
 *    nothing calls exit().
 *  - State machine (SPEC SwitchState S:234-237):  none --merge(d)--> merged(d);
 *    merged(d) --merge(d')--> merged(d') [one fused Eq. 10 pass];
 *    merged(d) --unmerge--> none.  unmerge in state none is LSW_E_STATE.  The
 *    host mirrors only "merged or not"; the decision itself lives on the device.
 *  - Launch count: exactly ONE switch-kernel launch per merge / unmerge call,
 *    independent of L, N, k, r.
 *  - Threading: one consumer thread per ctx; no internal locking.
 */
#ifndef LSW_H_
#define LSW_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define LSW_API __attribute__((visibility("default")))
#else
#define LSW_API
#endif

#define LSW_ABI_VERSION 1
#define LSW_MAX_TOPK 8        /* k <= 8                                     */
#define LSW_MAX_EXPERTS 64    /* N <= 64                                    */
#define LSW_NKIND 7

typedef struct lsw_ctx lsw_ctx;

typedef enum {
  LSW_OK = 0,
  LSW_E_ARG = 1,          /* null pointer, bad enum, misaligned pointer       */
  LSW_E_SHAPE = 2,        /* inconsistent or unsupported sizes                */
  LSW_E_STATE = 3,        /* call not allowed in the current merge state      */
  LSW_E_CUDA = 4,         /* CUDA runtime / driver failure                    */
  LSW_E_NCCL = 5,         /* NCCL failure or TP call without a communicator   */
  LSW_E_DEVICE = 6,       /* a device-side error was latched (device_status)  */
  LSW_E_OOM = 7,          /* ctx-owned allocation failed                      */
  LSW_E_UNSUPPORTED = 8   /* requested implementation not available           */
} lsw_status;

/* Device-side error codes latched by the kernels (lsw_device_status). */
enum {
  LSW_DEV_OK = 0,
  LSW_DEV_NONFINITE_LOGITS = 1,  /* router: a logit is NaN/Inf     */
  LSW_DEV_BAD_INDEX = 2,         /* switch: idx out of [0,N) or duplicated  */
  LSW_DEV_BAD_GATE = 3           /* switch: non-finite gate value           */
};

typedef enum { LSW_F32 = 0, LSW_BF16 = 1 } lsw_dtype;

typedef enum {
  LSW_Q = 0, LSW_K = 1, LSW_V = 2, LSW_O = 3, LSW_GATE = 4, LSW_UP = 5, LSW_DOWN = 6
} lsw_kind;

/* GEMV groups: sites that share one input vector in a decode step (R18). */
typedef enum { LSW_G_QKV = 0, LSW_G_O = 1, LSW_G_GATE_UP = 2, LSW_G_DOWN = 3, LSW_NGROUP = 4 } lsw_group;

/* Switch-kernel implementation (K1 variants). */
typedef enum {
  LSW_IMPL_AUTO = 0,   /* TC for bf16, SIMT for fp32                         */
  LSW_IMPL_SIMT = 1,   /* CUDA-core fp32 FFMA, per-expert fp32 accumulators   */
  LSW_IMPL_TC = 2      /* tcgen05 + TMEM + TMA, per-expert TMEM accumulators  */
} lsw_impl;

typedef struct {
  void*       W;             /* [L, d_out, d_in]  device, mutated in place           */
  const void* A;             /* [L, N, r, d_in]   device, read at create (packing)   */
                             /*                   and by the SIMT switch             */
  const void* B;             /* [L, N, d_out, r]  device                              */
  int64_t     d_out, d_in;   /* LOCAL sizes of this rank's shard                     */
  int32_t     row_parallel;  /* 1: d_in is sharded (o, down) -> the decode GEMV     */
                             /*    output is sum-allreduced when tp_size > 1         */
  int32_t     reserved;
} lsw_kind_desc;

typedef struct {
  int32_t n_layers;          /* L >= 1                                               */
  int32_t n_experts;         /* N in [1, LSW_MAX_EXPERTS]                             */
  int32_t rank;              /* r >= 1                                               */
  int32_t top_k;             /* k in [1, min(N, LSW_MAX_TOPK)]              */
  float   alpha;             /* LoRA alpha; scale = alpha / r  (R3; paper: 16)        */
  int32_t dtype;             /* lsw_dtype                                            */
  int64_t d_model;           /* router input length                                  */
  int32_t tp_rank, tp_size;  /* tensor-parallel position (1 GPU: 0, 1)               */
  int32_t impl;              /* lsw_impl                                             */
  int32_t reserved;
} lsw_config;

typedef struct {
  int64_t  tiles_total;      /* switch tiles per pass (all layers, all kinds)        */
  int32_t  switch_impl;      /* lsw_impl actually used                               */
  int32_t  grid;             /* persistent switch grid (CTAs)                        */
  int32_t  tile_m, tile_n;   /* switch tile shape                                    */
  int32_t  merged;           /* host mirror of the state machine                     */
  int32_t  num_sms;
  uint64_t kernel_launches;  /* kernels this ctx has launched so far                 */
  int64_t  packed_bytes;     /* ctx-owned packed operand bytes on the device         */
  int64_t  xs_elems, ys_elems; /* token I/O sizes (lsw_decode_token)                  */
  int32_t  switch_kernel;    /* tensor-core switch mode: 3 = folded coefficients, one */
                             /* accumulator per tile; 4 = per-term accumulators;     */
                             /* 5 = per-term, B staged per unit; 6 = the fold on     */
                             /* CTA pairs (cta_group::2); 7 = the fold with its      */
                             /* (hi, lo) B strip in TMEM; 0 = SIMT                   */
  int32_t  reserved;
} lsw_info;

/* Returns LSW_ABI_VERSION. */
LSW_API int32_t lsw_abi_version(void);

/* Thread-local message describing the last non-OK status of this thread. */
LSW_API const char* lsw_last_error(void);

/*
 * Validate shapes, build the tile table, allocate the ctx state and, for the
 * tensor-core switch, pack the LoRA factors into K-major tcgen05 operand
 * copies (A^T per expert, rank padded to a multiple of 16; ctx-owned, about
 * N*r*(d_in + d_out)*L*2 B per kind) and encode the TMA descriptors.  The
 * packing kernels run on the legacy default stream and are complete when
 * lsw_create returns.  Device = the current CUDA device.
 * Errors: LSW_E_ARG (null/misaligned pointers, bad enums), LSW_E_SHAPE (d_in
 * not a multiple of 8, k > N, N > 64, ...), LSW_E_UNSUPPORTED (TC requested
 * for fp32 or on a GPU without sm_100), LSW_E_OOM, LSW_E_CUDA.
 */
LSW_API lsw_status lsw_create(const lsw_config* cfg, const lsw_kind_desc kinds[LSW_NKIND],
                      const void* router_w, lsw_ctx** out);

/* Free ctx-owned memory and the communicator.  Synchronizes the device. */
LSW_API lsw_status lsw_destroy(lsw_ctx* ctx);

/* Fill `info`. Never fails for a valid ctx. */
LSW_API lsw_status lsw_get_info(const lsw_ctx* ctx, lsw_info* info);

/*
 * Tensor parallelism (tp_size > 1): rank 0 calls lsw_nccl_get_unique_id,
 * broadcasts the 128 bytes out of band (e.g. torch.distributed), then every
 * rank calls lsw_attach_nccl (collective; blocks until all ranks joined).
 */
LSW_API lsw_status lsw_nccl_get_unique_id(void* id_out_128B_h);
LSW_API lsw_status lsw_attach_nccl(lsw_ctx* ctx, const void* id_128B_h);
/*
 * NCCL is not linked: the first NCCL call binds libnccl.so.2 with dlopen --
 * the copy already loaded in the process if there is one (torch's, after
 * `import torch`), else the variant option nccl_path (lsw_debug.h), else the
 * loader's search path.  Reports NCCL_VERSION_CODE of the bound library
 * (e.g. 22809 for 2.28.9) and, if path_h is non-null, its file name (HOST
 * buffer of path_len bytes, NUL-terminated, truncated).  LSW_E_NCCL if no
 * NCCL can be loaded.  Needs no GPU.
 * A tp_size = 1 ctx accepts lsw_attach_nccl too (a 1-rank communicator): its
 * row-parallel decode GEMVs then run the all-reduce call (an identity) --
 * the TP call site on one GPU.
 */
LSW_API lsw_status lsw_nccl_version(int32_t* version_h, char* path_h, int64_t path_len);

/*
 * Eq. 2: z = W_g x1 accumulated in fp64 (R6), S = top-k by
 * (z desc, index asc) (R5), g = softmax over z_S only (R4).
 *   x1   [d_model] device, cfg dtype
 *   idx  [top_k] int32 device, out: sorted by descending g
 *   gate [top_k] fp32  device, out: sums to 1
 * Non-finite logits latch LSW_DEV_NONFINITE_LOGITS and write idx = -1.
 */
LSW_API lsw_status lsw_router_topk(lsw_ctx* ctx, const void* x1, int32_t* idx, float* gate, void* stream);

/*
 * State none:      Eq. 6  W <- RNE(W + sum_j (alpha/r) g_j B_j A_j)          (merge)
 * State merged(d): Eq. 10 W <- RNE(W + Delta(idx,gate) - Delta(d))           (fused switch)
 * ONE kernel over every tile of every adapted matrix of every layer.  The new
 * decision is recorded on the device by the same kernel.  idx/gate: device
 * [top_k] (typically straight from lsw_router_topk).
 */
LSW_API lsw_status lsw_merge_all_layers(lsw_ctx* ctx, const int32_t* idx, const float* gate, void* stream);

/* Eq. 7: W <- RNE(W - Delta(d)) for the merged decision d; state -> none.
 * LSW_E_STATE if nothing is merged. */
LSW_API lsw_status lsw_unmerge_all_layers(lsw_ctx* ctx, void* stream);

/*
 * Restore-from-pristine switch (the paper rejects it for memory,
 * P:266, which B200's 180 GB makes affordable):  W <- RNE(P + Delta(idx, gate))
 * for every adapted matrix of every layer, ONE launch, from any state; state ->
 * merged(idx, gate).  Same 4 B/element as the fused switch, k (not 2k) terms,
 * and no drift: W after a token depends only on that token's decision.
 *   lsw_attach_pristine: P[kind] [L, d_out, d_in] caller-owned DEVICE copies
 *   of the original W (same layout and dtype, 16-byte aligned), borrowed for
 *   the ctx lifetime; call once.  LSW_E_ARG on null / misaligned pointers.
 *   lsw_restore_merge_all_layers: LSW_E_STATE if no pristine copy is attached.
 */
LSW_API lsw_status lsw_attach_pristine(lsw_ctx* ctx, const void* const P[LSW_NKIND]);
LSW_API lsw_status lsw_restore_merge_all_layers(lsw_ctx* ctx, const int32_t* idx, const float* gate,
                                                void* stream);

/*
 * Eq. 3: y = W*[layer, kind] x, batch 1, fp32 accumulate.
 *   x [d_in] device cfg dtype;  y [d_out] fp32 device, overwritten.
 * Row-parallel kinds with tp_size > 1 (or a communicator attached): y is
 * sum-allreduced (fp32, in place, on `stream`) over the TP group.
 */
LSW_API lsw_status lsw_decode_linear(lsw_ctx* ctx, int32_t layer, int32_t kind, const void* x, float* y,
                             void* stream);

/* One GEMV launch for every kind of `group` (they share x): y is the
 * concatenation of the kinds' outputs in kind order (e.g. QKV -> [q | k | v]). */
LSW_API lsw_status lsw_decode_group(lsw_ctx* ctx, int32_t layer, int32_t group, const void* x, float* y,
                            void* stream);

/*
 * Alg. 1 l.5 (Eq. 3) for a whole token on the current weights: for
 * every layer, in order, the four group GEMVs (QKV, O, GATE_UP, DOWN).
 * xs packs the GEMV inputs layer-major, group-minor (each of its local d_in,
 * cfg dtype); ys packs the fp32 outputs the same way (each group's concatenated
 * local d_out).  Sizes: lsw_get_info xs_elems / ys_elems.  tp_size == 1: ONE
 * persistent launch in which group g reads its x only after every CTA has
 * finished group g-1 (decoder order); tp_size > 1: one launch per group plus
 * the NCCL all-reduce of the row-parallel groups.  Results are bitwise equal
 * to lsw_decode_group called group by group.
 */
LSW_API lsw_status lsw_decode_all_layers(lsw_ctx* ctx, const void* xs, float* ys, void* stream);

/*
 * Unmerged decode ("the honest comparison"; Eq. 2 at P:228 run
 * without merging): y = W x + sum_j (alpha/r) g_j B[e_j] (A[e_j] x) for every
 * site of `group`, on the UN-merged weights.  W is read once (2 B/element)
 * instead of being switched (4 B) and then read (2 B).  One launch per group:
 * extra warps of each CTA compute the group's k*r LoRA-down products per site
 * (spread over the grid, published through a device counter) and the LoRA-up
 * terms of the CTA's rows while its W rows stream; y = (W x) + term, one
 * rounding of the sum per row; deterministic (fixed reduction orders).
 *   idx/gate: device [top_k] (from lsw_router_topk).  x, y as lsw_decode_group.
 *   LSW_E_STATE if the ctx is merged (W must be the pristine weight).
 *   Tensor parallel: as lsw_decode_linear -- a row-parallel group (o, down:
 *   W[:, shard], A[:, shard]) writes its partial sum, all-reduced in place
 *   (Eq. 2 is linear in the d_in shards, so no all-reduce of A x is needed);
 *   LSW_E_NCCL before enqueuing if tp_size > 1 and no communicator.
 */
LSW_API lsw_status lsw_decode_group_unmerged(lsw_ctx* ctx, int32_t layer, int32_t group, const void* x, float* y,
                                             const int32_t* idx, const float* gate, void* stream);
/*
 * Prefill ("For the prefilling phase, we have not
 * implemented specific optimizations"): the unmerged forward of `group` for T
 * prompt tokens, each with its OWN pre-gated decision, so nothing can be
 * merged -- Eq. 2 as written:
 *   Y[t] = W x_t + sum_j (alpha/r) gate[t][j] B[idx[t][j]] (A[idx[t][j]] x_t).
 *   X: device [T, d_in] (storage dtype, row-major, 16-byte aligned); idx:
 *   device int32 [T, top_k]; gate: device fp32 [T, top_k]; Y: device fp32
 *   [T, rows], rows = the group's output rows in site order (as
 *   lsw_decode_group), overwritten.  bf16 with the tensor-core switch: three
 *   launches of our tcgen05 kernels -- the LoRA-down products of every expert
 *   (one GEMM over the bank A [N*r, d_in], K split over the grid), the
 *   gate-scaled products of each token's selected experts as an exact-to-2^-16
 *   (hi, lo) bf16 pair, and ONE tcgen05 contraction per 128-row x 128-token
 *   tile over K = d_in (W x^T) + 2 N rp (the LoRA-up term against the ctx's
 *   packed B) -- fp32 accumulation; for the single-CTA groups (o, down) with
 *   top_k <= 4 the first two are folded into the third launch (A-bank tiles
 *   whose epilogue builds the operand; variant option pf_fuse_u); otherwise
 *   two CUDA-core kernels (only the k selected experts).  Deterministic.
 *   Scratch and the tensor-core plan are ctx-owned, built / grown on demand
 *   (the first call, or a larger T: not graph-capturable then); a captured
 *   call takes the three-launch path (tests/test_gpu_graph.py).
 *   LSW_E_STATE if the ctx is merged; LSW_E_ARG for T outside [1, 2^20].
 *   Invalid idx values contribute nothing.  Tensor parallel: row-parallel
 *   groups' partial Y all-reduced in place (as lsw_decode_group_unmerged);
 *   LSW_E_NCCL before enqueuing if tp_size > 1 and no communicator.
 */
LSW_API lsw_status lsw_prefill_group(lsw_ctx* ctx, int32_t layer, int32_t group, const void* X, int64_t T,
                                     const int32_t* idx, const float* gate, float* Y, void* stream);
/* Every group of every layer, in order (layouts as lsw_decode_all_layers). */
LSW_API lsw_status lsw_decode_all_layers_unmerged(lsw_ctx* ctx, const void* xs, float* ys, const int32_t* idx,
                                                  const float* gate, void* stream);

/*
 * One whole Alg. 1 token: router(x1) -> merge_all_layers -> lsw_decode_all_layers.
 * idx/gate receive the decision (device).
 */
LSW_API lsw_status lsw_decode_token(lsw_ctx* ctx, const void* x1, const void* xs, float* ys,
                            int32_t* idx, float* gate, void* stream);

/*
 * Fused switch + decode: the same token as lsw_decode_token --
 * router, then every adapted matrix of every layer switched in ONE launch --
 * but the switch kernel also computes the group GEMVs from the freshly
 * rounded weight tiles, so W is read once and written once per token (4
 * B/element instead of 6).  Tiles are walked in decoder order, one segment per
 * (layer, group); a segment's outputs are accumulated only after every tile of
 * the previous segment is done (y final), as a decoder needs.  The fused
 * launch is the fold mode of the tensor-core switch: W ends bitwise as after
 * lsw_merge_all_layers; ys equals lsw_decode_all_layers on those weights up
 * to fp32 summation order (accumulated in 64-bit fixed point: bitwise
 * reproducible).  A decision equal to the merged one (nothing to add) still
 * computes ys.  Layouts as lsw_decode_token.  LSW_E_UNSUPPORTED unless the
 * ctx switches with the fold mode and tp_size == 1.
 */
LSW_API lsw_status lsw_decode_token_fused(lsw_ctx* ctx, const void* x1, const void* xs, float* ys, int32_t* idx,
                                          float* gate, void* stream);

/* Same as lsw_decode_token from HOST buffers: copies x1_h, xs_h to ctx-owned
 * device staging, runs the token, copies ys/idx/gate back and synchronizes
 * `stream` (and a ctx-owned side stream).  The copies overlap the token: xs
 * travels on the side stream while the router and the switch run, and each
 * layer's outputs return as soon as that layer's GEMVs are done.  Host buffers
 * should be pinned for asynchronous copies.  From the second call on, the
 * token is replayed as ONE CUDA graph (captured on a ctx-owned stream, one per
 * state of the decision slot: merge / switch; captured again when any of the
 * five host pointers changes), so the host adds one launch per token; results
 * are bitwise those of the eager path (variant option host_graph=0). */
LSW_API lsw_status lsw_decode_token_host(lsw_ctx* ctx, const void* x1_h, const void* xs_h, float* ys_h,
                                 int32_t* idx_h, float* gate_h, void* stream);

/* Synchronize `stream`, then return LSW_OK or LSW_E_DEVICE and write + clear
 * the latched device error code (LSW_DEV_*) into *code (may be NULL). */
LSW_API lsw_status lsw_device_status(lsw_ctx* ctx, void* stream, int32_t* code);

#ifdef __cplusplus
}  /* extern "C" */
#endif
#endif  /* LSW_H_ */
