/*
 * ttround.h — C-ABI of the B200-native randomized TT-rounding library
 * (libttround.so, built from paper_2110_04393_b200/csrc).
 *
 * Method: arXiv 2110.04393 ("Randomized algorithms for rounding in the
 * Tensor-Train format").  Citations "P:n" are lines of the paper text
 * (PAPER.md); DESIGN.md lists every reading of the paper the library makes
 * (R1..R17) and is the companion of this header.
 *
 * ------------------------------------------------------------------------
 * Conventions shared by every entry point
 * ------------------------------------------------------------------------
 * TT-tensor: d >= 2 cores X_n, n = 1..d, X_n in R^{R_{n-1} x I_n x R_n},
 * R_0 = R_d = 1.  All values are IEEE fp64.
 *
 * Core layout ("a-fastest", column-major in (a, i, b)): element (a, i, b) of
 * core n is stored at  a + R_{n-1} * (i + I_n * b).  Hence
 *   V(X_n) is the column-major R_{n-1}I_n x R_n matrix at the same
 *          address with leading dimension R_{n-1}I_n (row index a + R_{n-1} i;
 *          the paper stacks slices, i.e. the same rows in another order), and
 *   H(X_n) is the column-major R_{n-1} x I_n R_n matrix with leading
 *          dimension R_{n-1} (column index i + I_n b; the paper's is b-fastest).
 * Both unfoldings are reshape-only; the row/column permutations w.r.t. the
 * paper are applied consistently to every operand, so every product of
 * unfoldings the algorithms form is the paper's (R1).
 * In PyTorch terms: a tensor of logical shape (R_{n-1}, I_n, R_n) with strides
 * (1, R_{n-1}, R_{n-1} I_n), i.e. torch.empty(R_n, I_n, R_{n-1}).permute(2,1,0).
 *
 * Memory: input cores are BORROWED (read-only) and may live in device memory
 * of the context's device or in host memory (pageable or pinned); host inputs
 * are copied to the device inside the call, overlapped with the computation.
 * Results (tt_tensor_t) and sketches (tt_sketch_t) are OWNED by the library and
 * released with the matching *_destroy.  Every call is ordered on the
 * context's CUDA stream and returns after the work completed (results are
 * readable on return).  Calls on one context must not overlap (one thread at a
 * time); different contexts are independent.
 *
 * Errors: every entry point returns an int, TT_OK (0) on success or a negative
 * TT_ERR_* code; no exception crosses the ABI; out-parameters are untouched on
 * error; tt_last_error() returns a thread-local message for the last failure.
 * A rank capped below the request is not an error (TT_FLAG_RANK_CAPPED).
 */
#ifndef TTROUND_H
#define TTROUND_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ------------------------------------------------------- */
#define TT_OK             0
#define TT_ERR_ARG       -1   /* null pointer, d < 2, S < 1 (world 1), bad mode/option */
#define TT_ERR_SHAPE     -2   /* dims differ across summands; bond ranks mismatch   */
#define TT_ERR_RANK      -3   /* a rank < 1, or R_0 != 1 or R_d != 1                */
#define TT_ERR_NONFINITE -4   /* NaN/Inf in the summands (or overflow of their sketch contractions), detected on the trace of a QR Gram */
#define TT_ERR_OOM       -5   /* device allocation failed                           */
#define TT_ERR_CUDA      -6   /* CUDA runtime error (message in tt_last_error)      */
#define TT_ERR_NCCL      -7   /* NCCL missing or failed                             */
#define TT_ERR_NUMERIC   -8   /* QR/SVD breakdown even after the Householder fallback */

/* ---- rounding modes (tt_round_opts.mode) -------------------------------- */
#define TT_SKETCH_ONLY 0  /* Alg. 7 output with the (capped) sketch ranks l_n, left-orthogonal */
#define TT_RANK        1  /* sketch with l = rank + oversample, then truncate to rank (R6)           */
#define TT_TOL         2  /* sketch with l = oversample (initial), truncate to eps0 (R3-R5) */

/* ---- result flags (tt_tensor_info) -------------------------------------- */
#define TT_FLAG_RANK_CAPPED   1u  /* some l_n was capped below the request (R7)             */
#define TT_FLAG_LEFT_ORTH     2u  /* cores 1..d-1 left-orthogonal (TT_SKETCH_ONLY)  */
#define TT_FLAG_RIGHT_ORTH    4u  /* cores 2..d right-orthogonal (after truncation, R3)    */
#define TT_FLAG_ZERO          8u  /* the sum was exactly zero: all ranks 1, zero cores (R16) */
#define TT_FLAG_QR_FALLBACK  16u  /* a Householder fallback QR ran at least once           */
#define TT_FLAG_SLAB         32u  /* cores hold this rank's mode slabs (tt_round_sum_slab)  */

typedef struct tt_ctx*    tt_ctx_t;
typedef struct tt_sketch* tt_sketch_t;
typedef struct tt_tensor* tt_tensor_t;

/* A borrowed TT-tensor.  dims[d], ranks[d+1] (ranks[0] = ranks[d] = 1) and
 * cores[d] are host arrays; cores[n] points to R_{n-1} I_n R_n doubles in the
 * layout above (device memory of the context's device, or host memory). */
typedef struct {
  int32_t d;
  const int64_t* dims;
  const int64_t* ranks;
  const double* const* cores;
} tt_view;

typedef struct {
  int32_t  mode;        /* TT_SKETCH_ONLY | TT_RANK | TT_TOL                                  */
  int32_t  adaptive;    /* TT_TOL only: grow l (x2) while a bond is saturated (R8)            */
  int64_t  rank;        /* TT_RANK: target rank r (uniform); TT_TOL: optional extra cap (0=none) */
  int64_t  oversample;  /* TT_RANK: p, sketch rank l = r + p; TT_SKETCH_ONLY/TT_TOL: l itself  */
  double   tol;         /* TT_TOL: relative tolerance eps0 > 0 (Alg. 2)                */
  uint64_t seed;        /* Philox key of the Gaussian sketch (Def. 3.1 / R9)                  */
  int64_t  max_rank;    /* adaptive upper bound on l (0 = structural caps only)               */
  const int64_t* ranks; /* optional per-bond targets r_1..r_{d-1} (host array of d-1 entries,
                         * each >= 1; NULL = the uniform `rank`): the paper's "target TT-ranks
                         * {l_n}".  tt_round_sum / tt_round_sum_slab in
                         * TT_RANK mode: sketch ranks l_n = r_n + oversample (capped, R7), bond n
                         * truncated to r_n; `rank` is ignored; no user sketch.
                         * tt_round_deterministic: the cap of bond n (with or without tol).
                         * Ignored in TT_SKETCH_ONLY / TT_TOL modes of tt_round_sum.          */
} tt_round_opts;

/* ---- context ------------------------------------------------------------- */
/* NCCL unique id (128 bytes) for tt_ctx_create; call on one rank, broadcast the
 * bytes (e.g. torch.distributed), pass them to tt_ctx_create on every rank. */
int tt_get_nccl_unique_id(uint8_t id[128]);

/* Diagnostic for the exchange step of the sharded sweep (the sum
 * over summands of Alg. 7 line 9): builds a ONE-rank NCCL communicator
 * the way tt_ctx_create does for world > 1 (libnccl resolved with dlopen,
 * ncclCommInitRank) and runs the path's two collectives on the context's
 * stream: an fp64-sum allreduce of n device doubles (library-owned scratch) and
 * the int64 allreduce of the status words.  With one rank the result must equal
 * the input; *max_abs_diff (host) receives the largest deviation (0.0 when
 * exact).  Lets a one-GPU box exercise the NCCL plumbing.  Synchronises the
 * stream.  TT_ERR_ARG (NULL, n < 0 or n > 2^28), TT_ERR_NCCL, TT_ERR_CUDA. */
int tt_nccl_selftest(tt_ctx_t ctx, int64_t n, double* max_abs_diff);

/* Create a context on CUDA device `device` using stream `cuda_stream`
 * (a cudaStream_t, or NULL for a library-created non-blocking stream; to run
 * on the legacy default stream pass cudaStreamLegacy, i.e. (void*)0x1).
 * nccl_id == NULL: single-GPU (world must be 1).  world > 1: the summands of a
 * rounding are sharded across `world` processes (one per GPU); each passes its
 * local summands and all receive the same result.  world == 1 WITH
 * an id: a one-rank NCCL communicator is built and the sharded code path (agreed
 * validation, ncclAllReduce of Y_n per sweep step) runs through it -- the
 * same results as the single-GPU context; for boxes with one GPU. */
int tt_ctx_create(int device, void* cuda_stream, const uint8_t* nccl_id,
                  int rank, int world, tt_ctx_t* out);
int tt_ctx_destroy(tt_ctx_t ctx);

/* Loopback communicator: `world` ranks as contexts of ONE process on one
 * device, each driven by its own host thread (calls release no lock, so the
 * ranks run concurrently).  It runs the sharded code path of tt_round_sum /
 * tt_round_sum_two_sided (per-rank summand shards, one exchange of
 * Y_n per sweep step; the last core) where only one GPU exists:
 * a rank's allreduce copies its partial into its own device slot, synchronises
 * its stream, meets the other ranks at a host barrier, sums all slots in rank
 * order 0..world-1 (so every rank holds identical bits) and meets them at a
 * second barrier.  No kernel waits on another rank.  A barrier that waits more
 * than 300 s returns TT_ERR_NCCL.  Correctness/test path, not a performance
 * path (the NCCL communicator of tt_ctx_create is).  1 <= world <= 16.  The
 * group must outlive every context created on it. */
typedef struct tt_loopback* tt_loopback_t;
int tt_loopback_create(int world, tt_loopback_t* out);
int tt_loopback_destroy(tt_loopback_t group);
/* Context of rank `rank` of a loopback group (device/stream as tt_ctx_create). */
int tt_ctx_create_loopback(int device, void* cuda_stream, tt_loopback_t group, int rank,
                           tt_ctx_t* out);

/* ---- sketch (Def. 3.1) --------------------------------------- */
/* Random Gaussian TT with ranks (1, l_1..l_{d-1}, 1): cores n = 2..d filled
 * in place with N(0, 1/(l_{n-1} I_n l_n)) entries from Philox4x32-10 keyed by
 * `seed`, counter (k_lo, k_hi, n, tag) for element pair k (R9).  Core 1 is
 * never used by Alg. 3/5/7 (R10) and is not materialised.  ranks has d+1
 * entries with ranks[0] = ranks[d] = 1 and must already be capped (R7). */
int tt_sketch_create(tt_ctx_t ctx, int32_t d, const int64_t* dims,
                     const int64_t* ranks, uint64_t seed, uint32_t tag,
                     tt_sketch_t* out);
/* Device pointer of core n (1-based, n >= 2) of a sketch (read-only). */
int tt_sketch_core(tt_sketch_t sk, int32_t n, const double** core);
int tt_sketch_destroy(tt_sketch_t sk);

/* ---- the hot path: Alg. 7 + truncation ----------- */
/* Round Y = sum_j Y^(j) of S_local summands (this process's shard; with
 * world > 1 a rank may hold none, S_local = 0 and terms = NULL, and then adds
 * zeros to every exchange; every rank must pass the same opts and sketch-ness;
 * the shapes and options are agreed across ranks before the first collective,
 * so a bad argument on one rank makes every rank return an error, never hang).
 *  1. caps l_n = min(l, l_{n-1} I_n, prod_{k>n} I_k, sum_j R^(j)_n)    (R7)
 *  2. sketch R (Def. 3.1) — from opts->seed, or `sketch` if non-NULL (it must
 *     have exactly the capped ranks, else TT_ERR_SHAPE)
 *  3. W^(j)_n = PartialContractionsRL(Y^(j), R) for every summand     (Alg. 3)
 *  4. left-to-right sweep: Y_n = V(X_n)[W^(1)_n; ...], Q_n = qr(Y_n),
 *     M_n = Q_n^T V(X_n), fold M^(j)_n into core n+1 of every summand   (Alg. 7)
 *  5. TT_RANK / TT_TOL: right-to-left QR+SVD truncation of the left-orthogonal
 *     result (R3-R5), with adaptive growth of l in TT_TOL (R8).
 * The result has ranks (1, k_1..k_{d-1}, 1) and is returned in *out. */
int tt_round_sum(tt_ctx_t ctx, int32_t S_local, const tt_view* terms,
                 const tt_round_opts* opts, tt_sketch_t sketch, tt_tensor_t* out);

/* Mode-slab sharding of the same rounding (SURVEY §8e alternative, §8f NEXT-2):
 * every rank holds ALL S summands, but of every core n only the mode-index slab
 * i in [slab_lo[n], slab_lo[n] + terms[j].dims[n]) of the global mode size
 * gdims[n] (terms[j].dims are the local slab sizes; the ranks' slabs must tile
 * every mode).  Alg. 7 then runs with every row-distributed step local:
 *  - the sketch: each rank generates its slab of G_n (the same Philox bits as
 *    the full core, so the result does not depend on the number of ranks);
 *  - Alg. 3: W_{n-1} = H(Z_n)H(G_n)^T is a sum over i_n -> one allreduce of the
 *    sum_j R_{n-1} x l_{n-1} stack per step (C5: 2.4 MB instead of Y_n's 42.5 MB);
 *  - line 10's QR of the row-distributed Y_n and the truncation's R-only QRs:
 *    CholeskyQR passes with the l x l Gram all-reduced (R replicated, Q local);
 *  - line 11: M = Q_n^T V(X_n) summed over the slabs (l x sum_j R allreduce);
 *  - carries, output cores, the truncation products and the SVDs of R: local /
 *    replicated, identical on every rank.
 * The result holds this rank's slab of every core (global ranks, local dims,
 * TT_FLAG_SLAB); concatenating the ranks' slabs along the mode axis gives the
 * rounded tensor.  Same opts as tt_round_sum (no user sketch).  world == 1:
 * the slab must be the whole mode.  Not supported (TT_ERR_ARG): a truncation
 * bond of rank > 160 or a wide unfolding (they need the non-distributed SVD);
 * a breakdown of every CholeskyQR route gives TT_ERR_NUMERIC (no distributed
 * Householder fallback). */
int tt_round_sum_slab(tt_ctx_t ctx, int32_t S, const tt_view* terms, const int64_t* gdims,
                      const int64_t* slab_lo, const tt_round_opts* opts, tt_tensor_t* out);

/* Deterministic TT-rounding of the assembled sum: Alg. 1 + Alg. 2
 * with eps0 = opts->tol (and opts->rank as an optional rank cap).
 * Assembles the sum, orthogonalises right to left (Alg. 1, economy
 * QR; a wide H(X_n)^T shrinks its bond) and truncates left to right with QR +
 * one-sided Jacobi SVD (Alg. 2, R5, R13).  Single GPU.  Ranks above 160 use the
 * generic (slow) Cholesky and the Jacobi that accumulates V.  Output ranks
 * (1, k_1..k_{d-1}, 1), left-orthogonal. */
int tt_round_deterministic(tt_ctx_t ctx, int32_t S, const tt_view* terms,
                           const tt_round_opts* opts, tt_tensor_t* out);

/* Two-Sided-Randomization (generalized Nystrom), Alg. 6, of the sum
 * Y = sum_j Y^(j) of S_local summands (R18-R21).
 *  - ell: target ranks l (>= 1); rho: right sketch rank (>= ell), 0 = ceil(1.5 l)
 *    (P:944); both capped per bond by R7, so l_n <= rho_n.
 *  - seed: Philox key of the left sketch L (tag 0x10001, cores 1..d-1) and the
 *    right sketch R (tag 0x10002, cores 2..d), Def. 3.1.
 *  - W^L_n = PartialContractionsLR(Y^(j), L) (R18), W^R_n = Alg. 3 with R, per
 *    summand; P_n = W^L_n W^R_n (sum over summands, all-reduced over ranks);
 *    SVD P_n = U S V^T; L_n = W^R_n V S^{-1/2}, R_n = S^{-1/2} U^T W^L_n with the
 *    pseudo-inverse cutoff s_i > max(l_n, rho_n) eps s_1 (R20);
 *    X_n = sum_j Y^(j)_n x1 R^(j)_{n-1} x3 L^(j)_n (R19).
 * Output ranks (1, l_1..l_{d-1}, 1), not orthogonal; an exactly zero
 * sum gives a zero TT of ranks 1 (TT_FLAG_ZERO).  Errors as tt_round_sum;
 * TT_ERR_NUMERIC for a non-finite singular value. */
int tt_round_sum_two_sided(tt_ctx_t ctx, int32_t S_local, const tt_view* terms,
                           int64_t ell, int64_t rho, uint64_t seed, tt_tensor_t* out);

/* ---- TT-GMRES on a Kronecker-sum operator --- */
#define TT_KRON_IDENTITY 0
#define TT_KRON_DIAG     1
#define TT_KRON_DENSE    2
/* The operator  sum_{i=1..nterms} A_{i,1} x ... x A_{i,d}.
 * kinds[i*d + n] selects factor A_{i,n+1}: TT_KRON_IDENTITY (mats entry ignored),
 * TT_KRON_DIAG (mats entry: I_n doubles, the diagonal), TT_KRON_DENSE (mats
 * entry: I_n x I_n column-major).  mats are device pointers of the context's
 * device (borrowed).  A factor acts on core n by the mode-2 product
 * core(a, i, b) <- sum_j A(i, j) core(a, j, b) (rank-preserving). */
typedef struct {
  int32_t d;
  int32_t nterms;
  const int64_t* dims;
  const int32_t* kinds;
  const double* const* mats;
} tt_kron_op;

/* (sum_i A_{i,1} x ... x A_{i,d}) x as its nterms UNROUNDED summands
 * (P:1033-1035): out[i] has the ranks of x; identity factors copy the core.
 * out must have room for op->nterms results (each freed by tt_tensor_destroy). */
int tt_kron_apply(tt_ctx_t ctx, const tt_kron_op* op, const tt_view* x, tt_tensor_t* out);

typedef struct {
  double   tol;         /* relative residual target (the paper uses 1e-8)          */
  double   round_tol;   /* eps0 of every rounding; 0 -> tol / 10 (G1)              */
  int32_t  max_iter;    /* Arnoldi steps (no restart)                                        */
  int32_t  randomized;  /* 1: every sum rounded by tt_round_sum (Alg. 7 + truncation, TT_TOL,
                           adaptive sketch rank); 0: by tt_round_deterministic (Alg. 1+2)    */
  int32_t  precond;     /* 1: right preconditioner ((sum_i A_{i,1})^{-1} x I x ... x I),
                           P:1036; sum_i A_{i,1} must be symmetric positive definite         */
  int32_t  oversample;  /* randomized: initial sketch rank = largest summand bond rank + this */
  int64_t  max_rank;    /* cap on every rounding's rank / sketch rank (0 = none)             */
  uint64_t seed;        /* rounding call c (0, 1, 2, ... in order) uses seed + c (G4)        */
} tt_gmres_opts;

typedef struct {
  int32_t iters;        /* Arnoldi steps taken                                              */
  int32_t converged;    /* 1 if the residual estimate reached tol                           */
  int32_t roundings;    /* rounding calls made                                              */
  int32_t max_basis_rank; /* largest internal rank of a Krylov basis vector V_k             */
  double  residual;     /* final relative residual estimate |beta e1 - H y| / beta          */
} tt_gmres_info;

/* Right-preconditioned TT-GMRES for op x = f: per step
 * Y = P V_k, W = round(sum_i (A_{i,1} x ... ) Y) (a sum of nterms
 * TT-tensors), h_jk = <V_j, W>, Z = round(W - sum_j h_jk V_j) (k+1
 * summands), V_{k+1} = Z / ||Z||; the (k+1) x k least-squares
 * problem on the host (Givens rotations); x = P round(sum_j y_j V_j).  The
 * result x is library-owned.  residuals (optional, host, max_iter + 1 doubles)
 * receives the residual estimates (1 first).  Errors: TT_ERR_ARG/SHAPE on a bad
 * operator, TT_ERR_NUMERIC if the preconditioner's Cholesky fails. */
int tt_gmres(tt_ctx_t ctx, const tt_kron_op* op, const tt_view* f, const tt_gmres_opts* opts,
             tt_tensor_t* x, tt_gmres_info* info, double* residuals);

/* ---- CUDA-graph plans for launch-bound small roundings ----------------- */
/* Capture B roundings of the same summands (TT_RANK or TT_SKETCH_ONLY opts,
 * sketch seed seeds[b] for rounding b) into ONE CUDA graph: an eager rounding
 * first sizes the workspaces and fixes the output shapes, then the B calls are
 * stream-captured (no host synchronisation inside); each writes its result into
 * plan-owned buffers and frees its temporaries inside the graph.  The inputs
 * must stay valid and unchanged while the plan is used.  The context must run on
 * a created (non-default) stream, one GPU.  tt_plan_launch replays the graph
 * on the context stream and returns after it completed; tt_plan_result copies
 * rounding b of the last replay into a new result (bitwise equal to
 * tt_round_sum with the same seed).  Errors: TT_ERR_ARG (mode, stream, world,
 * zero sum), TT_ERR_CUDA (capture). */
typedef struct tt_plan* tt_plan_t;
/* branches >= 1: the B roundings run as that many parallel branches of the
 * graph (rounding b on branch b mod branches), each with its own library-owned
 * stream and workspaces. */
int tt_plan_create(tt_ctx_t ctx, int32_t S, const tt_view* terms, const tt_round_opts* opts,
                   int32_t B, const uint64_t* seeds, int32_t branches, tt_plan_t* out);
int tt_plan_launch(tt_plan_t plan);
int tt_plan_result(tt_plan_t plan, int32_t b, tt_tensor_t* out);
int tt_plan_destroy(tt_plan_t plan);

/* <x, y> by the full right-to-left contraction (App. A); *out is a
 * host double.  x and y must have equal dims. */
int tt_inner(tt_ctx_t ctx, const tt_view* x, const tt_view* y, double* out);

/* ---- results ------------------------------------------------------------- */
/* Borrowed views of a result: *dims (d), *ranks (d+1), *cores (d device
 * pointers, layout above), valid until tt_tensor_destroy. */
int tt_tensor_info(tt_tensor_t t, int32_t* d, const int64_t** dims,
                   const int64_t** ranks, double* const** cores, uint32_t* flags);
/* Copy core n (1-based) to caller memory (host or device), R_{n-1} I_n R_n doubles. */
int tt_tensor_copy_core(tt_tensor_t t, int32_t n, double* dst);
/* Copy every core: dst[n] (host or device) receives core n+1; all copies are
 * queued on the result's stream before one synchronisation. */
int tt_tensor_copy_all(tt_tensor_t t, double* const* dst);
/* Number of rounding passes the adaptive loop made (1 if not adaptive). */
int tt_tensor_passes(tt_tensor_t t, int32_t* passes);
/* Frees a result: stream-ordered on the creating context's stream (no host
 * synchronisation) while that context lives, else after a device-wide sync.
 * Work reading the cores on OTHER streams must be complete before the call. */
int tt_tensor_destroy(tt_tensor_t t);

/* ---- diagnostics --------------------------------------------------------- */
const char* tt_last_error(void);
/* Number of CUDA kernels this library launched since load (all contexts). */
uint64_t tt_launch_count(void);
/* Per-phase device times (ms) of the last tt_round_sum on ctx, measured with
 * CUDA events on the context stream when timing is enabled:
 * [0] sketch, [1] phase 1 (Alg. 3), [2] sweep GEMMs, [3] QR, [4] collectives,
 * [5] truncation, [6] total.  Returns the number of entries written (<= n).
 * tt_round_sum_two_sided: [0] sketches, [1] Alg. 3 with R, [2] left contraction
 * and assembly GEMMs, [3] bond QR + SVD, [4] collectives, [5] bond factors. */
int tt_ctx_set_timing(tt_ctx_t ctx, int enable);
/* Copy the context's device status words (after the last call) to out[0..n):
 * [1] Householder fallback used, [2] zero sketch seen, [3] bit 1: Jacobi SVD hit
 * its sweep limit; the others are per-QR route flags.
 * Returns the number of words written. */
int tt_ctx_flags(tt_ctx_t ctx, int* out, int n);
int tt_ctx_last_timing(tt_ctx_t ctx, double* ms, int n);
/* Several independent roundings in flight on one GPU (one context per host
 * thread; SURVEY §8e "independent roundings").  reserve_sms: the persistent and
 * cooperative grids of this context (phase-1 Z GEMM, fused projection-and-carry,
 * CholeskyQR passes) are sized to (SM count - reserve_sms) SMs, so they can be
 * co-resident with another context's latency-bound kernels (0 = all SMs, the
 * default).  chain_priority != 0: the QR of Alg. 7 line 10 and the
 * truncation run on a highest-priority stream of the context,
 * ordered with the context stream by events, so their one-CTA Cholesky and
 * 8-CTA Jacobi are dispatched ahead of queued GEMM tiles of another context
 * (not for tt_round_sum_slab, whose QRs all-reduce Grams: one NCCL stream per
 * communicator).  chain_priority alone leaves the results unchanged bit for
 * bit (same kernels, same order); reserve_sms > 0 changes the split-K slicing of
 * the fused projection and the CholeskyQR passes' partial-Gram count, i.e. the
 * summation order (results equal to rounding).  TT_ERR_ARG if reserve_sms
 * is negative or leaves no SM; TT_ERR_CUDA if the stream cannot be created. */
int tt_ctx_set_concurrency(tt_ctx_t ctx, int reserve_sms, int chain_priority);

/* ---- kernel-level entry points (for the parity tests and bench) ---------- */
/* C = alpha*op(A)*op(B) + beta*C, column-major fp64, device pointers; the
 * FP64 tensor-core (DMMA) GEMM every contraction of the hot path runs on. */
int tt_dgemm(tt_ctx_t ctx, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
             double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
             double beta, double* C, int64_t ldc);
/* Thin QR of the column-major m x n (m >= n) device matrix A: Q (m x n, ld m)
 * and, if R != NULL, R (n x n upper triangular, ld n).  Q == NULL asks for R
 * only (the truncation's use).  Routes: CholeskyQR2, shifted CholeskyQR3, then
 * (R only) Householder TSQR or (with Q) single-CTA Householder; *fallback = 1
 * if one of the two Householder fallbacks ran. */
int tt_qr(tt_ctx_t ctx, int64_t m, int64_t n, const double* A, int64_t lda,
          double* Q, double* R, int* fallback);
/* Singular values (descending) and right singular vectors of the column-major
 * m x n (m >= n) device matrix A: AV (m x n, = U Sigma) and V (n x n). */
int tt_svd_jacobi(tt_ctx_t ctx, int64_t m, int64_t n, const double* A, int64_t lda,
                  double* AV, double* V, double* sigma);

/* The truncation's SVD (DESIGN.md §6 "Truncation design"): one-sided Jacobi of
 * the column-major m x n (n <= m <= 160) device matrix A WITHOUT forming V:
 * AV = U Sigma (m x n, ld m, columns sorted by descending sigma) and sigma (n).
 * Used on R^T of the truncation's R-only QR (P:667-670 via Alg. 2 line 7). */
int tt_svd_nov(tt_ctx_t ctx, int64_t m, int64_t n, const double* A, int64_t lda,
               double* AV, double* sigma);

/* The CholeskyQR passes' factorisation (DESIGN.md §6 "Cholesky kernel"): G
 * (n x n symmetric, lower triangle read, ld n, device) + shift I = L L^T with
 * L lower triangular; writes Rinv = L^{-T} (n x n upper, ld n) and, if L != NULL,
 * L (n x n lower, ld n).  shifted = 1 applies the shifted-CholeskyQR shift
 * 11 (m n + n (n + 1)) u tr(G) (Fukaya et al.; m = the tall matrix's row count),
 * shifted = 0 factors G itself (pivots below 64 n u max diag G are clamped, the
 * R-only QR's rule).  TT_ERR_NUMERIC if a pivot is not positive and finite. */
int tt_cholesky(tt_ctx_t ctx, int64_t n, const double* G, int64_t m, int shifted,
                double* Rinv, double* L);

/* One CholeskyQR pass in one persistent launch (DESIGN.md §6 "CholeskyQR
 * pass kernel"; the passes of the thin QR of Alg. 7 line 10, and of the
 * truncation's QR, Alg. 2 line 4 / P:667-670): Q = op(A) Rinv and G = Q^T Q.
 * op(A) = A (m x n, ld lda) or, trans = 1, A^T with A n x m (ld lda).  Rinv
 * (n x n upper triangular, ld n; entries below the diagonal are not read) or
 * NULL (Q = op(A)).  Q (m x n, ld ldq) and G (n x n, both triangles, ld n) are
 * optional outputs (at least one).  All device pointers; 1 <= n <= 144 else
 * TT_ERR_ARG.  Results are deterministic (fixed chunk-to-CTA map, CTA-ordered
 * Gram sum). */
int tt_cholqr_pass(tt_ctx_t ctx, int64_t m, int64_t n, const double* A, int64_t lda, int trans,
                   const double* Rinv, double* Q, int64_t ldq, double* G);

#ifdef __cplusplus
}
#endif
#endif /* TTROUND_H */
