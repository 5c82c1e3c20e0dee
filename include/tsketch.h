/*
 * tsketch.h -- C ABI of libtsketch, the B200 (sm_100a) hot path of the tensor-based
 * sketching method for low-rank approximation of matrix streams (arXiv 2209.14637).
 *
 * Problem (Eq. (1)): for every matrix A_d (m x n) of a stream,
 *     min_B ||A_d - B||_F  s.t.  rank(B) <= r.
 * Method (Algorithm 2):
 *   1. tensorise the training matrices A_1..A_D' (m x n) into a third-order tensor;
 *   2. S <- Tucker1 of that tensor along mode 1, i.e. S* = (U^(1))_k^T, the first k
 *      left singular vectors of A_(1) = [A_1|...|A_D'] -- computed here as the
 *      top-k eigenvectors of the mode-1 Gram G = A_(1) A_(1)^T = sum_d A_d A_d^T;
 *   3. A_hat <- SCW(A, S, r) for every test matrix A (Algorithm 1).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * - Matrices are fp32 (inputs/outputs named float*) or fp64 (double*), ROW-MAJOR and
 *   contiguous.  A stack of matrices [B][m][n] is slice-major (matrix b starts at b*m*n).
 * - Pointers may be DEVICE pointers (current device of the ctx) or HOST pointers (pageable or
 *   pinned).  The library detects which with cudaPointerGetAttributes: host inputs are copied
 *   to device workspace and host outputs are copied back before the call returns (the call is
 *   then synchronous).  With device pointers every call is asynchronous on the ctx stream.
 * - Alignment: device pointers to fp32 matrices must be 16-byte aligned and n % 4 == 0
 *   (TMA row pitch), else TSK_ESHAPE.
 * - Ownership: the caller owns all buffers; the library never frees or retains them past
 *   the call's stream completion.  The ctx owns its workspace.
 * - Errors: argument errors return synchronously and enqueue nothing.  Device faults surface
 *   as TSK_ECUDA on this or a later call (or tsk_sync).
 * - Threading: one ctx per host thread/stream; different ctxs are independent.
 * - Determinism: fixed reduction orders (fp64 partial sums are reduced at L2 by a single thread
 *   per address, in program order): identical inputs give bit-identical outputs.
 */
#ifndef TSKETCH_H_
#define TSKETCH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tsk_ctx_s* tsk_ctx;

typedef enum {
  TSK_OK = 0,
  TSK_WARN_RANK_CLAMPED = 1,  /* r > k: r clamped to k (reading c7); results valid */
  TSK_WARN_NOT_CONVERGED = 2, /* eigensolver hit max_iters; S valid but not converged */
  TSK_EINVAL = -1,            /* bad scalar: k < 1, k > m, r < 1, D < 1, B < 0, m/n < 1 */
  TSK_ESHAPE = -2,            /* n % 4 != 0, misaligned pointer */
  TSK_ENOMEM = -3,            /* device workspace allocation failed */
  TSK_ECUDA = -4,             /* CUDA runtime / launch / device fault */
  TSK_ENCCL = -5,             /* NCCL library not loadable, or an NCCL call failed */
  TSK_EDEVICE = -6,           /* device is not compute capability 10.0 (sm_100a) */
  TSK_ENONFINITE = -7,        /* NaN/Inf in the training input, only with opts->check_finite */
  TSK_ENULL = -8,             /* a required pointer is NULL */
  TSK_ENUMERIC = -9           /* numerical breakdown the fallbacks could not repair (e.g. the eigensolver's
                                 Householder/Jacobi fallback failed repeatedly); not a CUDA fault */
} tsk_status;

/* Create a context on `device`, enqueueing on `cuda_stream` (a cudaStream_t; NULL = legacy
   default stream).  Fails with TSK_EDEVICE unless the device is sm_100. */
tsk_status tsk_create(tsk_ctx* out, int device, void* cuda_stream);
tsk_status tsk_destroy(tsk_ctx ctx);
/* Re-target subsequent work to another stream of the same device. */
tsk_status tsk_set_stream(tsk_ctx ctx, void* cuda_stream);
/* Block until all work enqueued by this ctx has completed; reports deferred device faults. */
tsk_status tsk_sync(tsk_ctx ctx);
const char* tsk_status_string(tsk_status s);
/* Number of kernels this ctx has launched since creation (bench evidence). */
int64_t tsk_launch_count(tsk_ctx ctx);

/* ---------------------------------------------------------------------- multi-GPU */
/* one process per GPU; the training stream is sharded by matrix index (rank p owns
   the contiguous range [floor(pD/P), floor((p+1)D/P))), each rank accumulates its local Gram and ONE
   all-reduce (sum, fp64) of the m x m Gram over NVLink/NVSwitch gives G on every rank; every rank then
   runs the same deterministic eigensolver (identical S, no broadcast).  NCCL is loaded at run time
   (libnccl.so.2, reusing the copy already in the process if any): TSK_ENCCL if it is not available.
   tsk_get_unique_id: uid[128] (host memory) to be broadcast by the caller (e.g. over torch.distributed).
   tsk_comm_init: collective over the nranks processes (same uid, distinct rank in [0, nranks)); the
   ctx's device must be the rank's GPU.  Afterwards sketch_train treats A as the rank's LOCAL shard (which
   may be empty, D = 0) and all-reduces G on the ctx stream before the top-k solve; a rank whose arguments
   or local Gram fail still joins a status all-reduce first, so every rank returns the same error instead
   of leaving its peers blocked in the collective.  The communicator is destroyed with the ctx;
   calling tsk_comm_init again replaces it. */
tsk_status tsk_get_unique_id(unsigned char uid[128]);
tsk_status tsk_comm_init(tsk_ctx ctx, int nranks, int rank, const unsigned char uid[128]);
/* The test stream is sharded like the training stream: rank p holds the per-matrix errors of test
   matrices [floor(p B/P), floor((p+1) B/P)) (B = B_total).  tsk_allgather_errors gathers them, in
   stream order, into err_all [B_total] on every rank (NCCL all-gather of the shards padded to
   ceil(B/P), compacted on the device), so the paper's test-error metric (a mean over
   the whole test set) can be evaluated anywhere.  err_local [hi - lo] and err_all are DEVICE fp64
   pointers; without a communicator it copies err_local to err_all.  Collective: every rank calls it
   with the same B_total.  Asynchronous on the ctx stream. */
tsk_status tsk_allgather_errors(tsk_ctx ctx, const double* err_local, int64_t B_total, double* err_all);
/* The Gram all-reduce of sketch_train on its own (for callers that run sketch_gram and sketch_topk as
   separate calls, e.g. to time them): G64 [m][m] DEVICE fp64 summed in place over the communicator's
   ranks (ncclAllReduce, sum, ctx stream); a no-op without a communicator. */
tsk_status tsk_allreduce_gram(tsk_ctx ctx, double* G64, int m);

/* ---------------------------------------------------------------------- training */

typedef struct {
  int oversample;    /* block size p = min(m, k + oversample); p <= 128 when m > dense_max_m; default (<= 0): 16 */
  int max_iters;     /* subspace iterations cap; default 300 */
  double tol;        /* convergence: every wanted Ritz pair has ||G x - theta x|| <= tol * theta_k (theta_k =
                        the k-th Ritz value, not theta_1), or -- where theta_k / theta_{k+1} < 1.05 -- the
                        Kato-Temple estimate of the remaining Ky Fan deficit is <= tol / 5 of the wanted
                        energy not yet locked; default 1e-6 */
  int dense_max_m;   /* m <= this (<= 256): one dense eigensolve of G; default 256 */
  int gemm_chain;    /* tuning: K-chunks per TMEM accumulation chain (0 = default) */
  int gemm_splits;   /* tuning: K splits of the Gram (0 = auto) */
  const float* init_S; /* optional DEVICE [k][m] warm start of the subspace iteration (e.g. the sketch of
                          the stream so far); NULL = deterministic pseudo-random start.
                          Only the starting block changes: S is still the top-k of G to tol. */
  int check_finite;    /* != 0 (sketch_gram / sketch_train): scan the training input first (one HBM pass)
                          and return TSK_ENONFINITE if any entry is NaN or Inf (matrices are
                          finite); device inputs: nothing is computed; host inputs are checked per staged
                          chunk, so G64 is unspecified after the error */
  int cheb_degree;     /* cap on the Chebyshev filter degree per outer iteration (0 = adaptive, <= 40: the
                          largest degree whose dynamic range T_d(x_max) stays <= 1e7) */
  int tol_active;      /* kept for ABI compatibility, ignored: residuals are always measured against theta_k
                          (the semantics this flag used to select) */
} tsk_train_opts;

typedef struct {
  int iters;          /* subspace iterations run (0 for the dense path) */
  double kyfan;       /* sum_{i<k} theta_i, the Ky Fan energy tr(S G S^T) */
  double max_resid;   /* max_{i<k} ||G s_i - theta_i s_i|| / theta_k over the pairs not yet locked */
  int gram_splits;    /* K splits used by the Gram kernel */
  int gram_tiles;     /* 128x128 output tiles computed (lower triangle) */
  double gap_est;     /* theta_k / theta_{k+1} from the last Rayleigh-Ritz step (the eigengap of reading c6;
                         +inf when the block holds no (k+1)-th value or it is 0) */
} tsk_train_info;

/* Mode-1 Gram of a stack of D training matrices:
     G (+)= sum_{d<D} A_d A_d^T          A: [D][m][n] fp32;  G64: [m][m] fp64 (required)
   G32 (optional, may be NULL): fp32 copy of the result.  accumulate != 0 adds into G64
   (streaming: call once per chunk of the stream).  Only the lower-triangle 128x128 tiles are
   computed (3xTF32 tensor cores) and mirrored, so G64 is exactly symmetric. */
tsk_status sketch_gram(tsk_ctx ctx, const float* A, int64_t D, int m, int n, double* G64, float* G32,
                       int accumulate, const tsk_train_opts* opts, tsk_train_info* info);

/* Top-k eigenvectors of the symmetric PSD Gram: S [k][m] fp32 with orthonormal
   rows ordered by decreasing eigenvalue, each row sign-normalised (largest-|entry| positive,
   reading c5); lambda [k] fp64 (may be NULL) the Ritz values.  G64 [m][m] fp64. */
tsk_status sketch_topk(tsk_ctx ctx, const double* G64, int m, int k, float* S, double* lambda,
                       const tsk_train_opts* opts, tsk_train_info* info);

/* Algorithm 2 lines 1-2: sketch_gram followed by sketch_topk.  G64_out (optional) receives the Gram.
   Multi-GPU: after tsk_comm_init, A is the rank's local shard and G is all-reduced (NCCL, sum) between
   the two steps; alternatively call sketch_gram on each shard, all-reduce G64 with the caller's own
   collective, then sketch_topk on every rank (deterministic, identical S everywhere). */
tsk_status sketch_train(tsk_ctx ctx, const float* A, int64_t D, int m, int n, int k, float* S, double* lambda,
                        double* G64_out, const tsk_train_opts* opts, tsk_train_info* info);

/* ---------------------------------------------------------------------- test stream */

/* SCW (Algorithm 1) on a batch of B test matrices A [B][m][n] with the sketch
   S [k][m]:  V = orthonormal basis of rowspace(S A_b) (QR/eigen orthonormalisation),
   [A_b V]_r by the SVD of A_b V, A_hat_b = [A_b V]_r V^T = L_b R_b^T with
     L [B][m][r] = U_r diag(sigma_r),   R [B][n][r] = V W_r (orthonormal columns),
     sigma [B][r] fp32 the singular values of A_b V (decreasing).
   Any of L, R, sigma may be NULL.  r > k is clamped to k (TSK_WARN_RANK_CLAMPED); r <= min(m,n). */
tsk_status sketch_apply_scw(tsk_ctx ctx, const float* A, int64_t B, int m, int n, const float* S, int k, int r,
                            float* L, float* R, float* sigma);

/* Per-matrix SCW error err[b] = ||A_b - SCW(A_b, S, r)||_F (fp64).  err: [B] fp64 (device or host).
   B = 0 is a no-op and then accepts NULL pointers (as does sketch_apply_scw).
   Formula (tsk_set_scw_error_mode; reading c17): A_hat = [A V]_r V^T is A P with P the
   orthogonal projector onto span(V W_r), so by default
     err^2 = ||A||_F^2 - sum_{i<r} sigma_i^2
   with ||A||_F^2 summed in fp64 while the SA product streams A; where this cancels (err^2 below
   tau ||A||^2, default tau = 3e-3, e.g. exactly low-rank matrices) the matrix gets the dense residual
   ||A - L R^T||_F on tcgen05 with an fp64 reduction instead.  Mode 1: the dense residual for all. */
tsk_status scw_error(tsk_ctx ctx, const float* A, int64_t B, int m, int n, const float* S, int k, int r,
                     double* err);

/* Error formula of scw_error on this ctx: mode 0 = Pythagorean identity with the dense residual below
   tau ||A||^2 (tau <= 0: the default 3e-3), mode 1 = dense residual for every matrix.  TSK_EINVAL for
   another mode or tau >= 1 / NaN.  Host-side setting, no GPU work. */
tsk_status tsk_set_scw_error_mode(tsk_ctx ctx, int mode, double tau);

/* ---------------------------------------------------------------------- two-sided variant */
/* the paper's second algorithm (Section 3.2).  Pointers
   may be host or device memory: host arrays are staged whole into device workspace (copied in, outputs
   copied back) and the call returns synchronised, as the one-sided host path; device arrays are used in
   place (fp32 arrays 16-byte aligned, else TSK_ESHAPE). */

/* Mode-2 Gram (the HOSVD initial factor of Algorithm 5 along mode 2):
     G2 (+)= sum_{d<D} A_d^T A_d          A: [D][m][n] fp32 (m % 4 == 0);  G64: [n][n] fp64
   3xTF32 tensor cores with both operands read transposed (the contraction runs over the rows of
   every A_d), lower-triangle tiles, mirrored (exactly symmetric). */
tsk_status sketch_gram_mode2(tsk_ctx ctx, const float* A, int64_t D, int m, int n, double* G64, int accumulate);

typedef struct {
  int max_sweeps;    /* HOOI sweeps cap; default (<= 0): 10 */
  double rel_tol;    /* stop when |res_{s-1} - res_s| <= rel_tol * res_{s-1}; default 1e-6 */
} tsk_hooi_opts;

typedef struct {
  int sweeps;                   /* sweeps run */
  int converged;                /* rel_tol reached */
  double a_fro2;                /* ||A||_F^2 of the training tensor (trace of the mode-1 Gram) */
  double residual_history[65];  /* [0]: HOSVD init, [s]: after sweep s (||A - G x1 S^T x2 W^T||_F) */
} tsk_hooi_info;

/* Tucker2 of the training tensor by HOOI over modes 1-2 (Eq. (9); Algorithm 5,
   PAPER.md:446-473; readings t1-t4 in DESIGN.md): HOSVD init S <- top-k eigenvectors of
   sum A_d A_d^T, W <- top-l of sum A_d^T A_d; each sweep
     mode 1: Y_d = A_d W^T (m x l), S <- top-k eigenvectors of sum_d Y_d Y_d^T
     mode 2: Z_d = A_d^T S^T (n x k), W <- top-l eigenvectors of sum_d Z_d Z_d^T
   (the truncated SVDs of the projected unfoldings, through their Grams).  S [k][m], W [l][n]
   fp32 with orthonormal rows (sign rule c5).  1 <= k <= m, 1 <= l <= n, m % 4 == n % 4 == 0. */
tsk_status sketch_train_two_sided(tsk_ctx ctx, const float* A, int64_t D, int m, int n, int k, int l, float* S,
                                  float* W, const tsk_hooi_opts* opts, tsk_hooi_info* info);

/* Two-sided SCW (Algorithm 3) on B test matrices A [B][m][n] with S [k][m] and
   W [l][n]: Q = orthonormal basis of rowspace(S A_b), P = orthonormal basis of col(A_b W^T),
   A_hat_b = P [P^T A_b Q]_r Q^T = L_b R_b^T,  L [B][m][r], R [B][n][r] (orthonormal columns),
   sigma [B][r] the singular values of P^T A_b Q.  Any of L, R, sigma may be NULL.
   r > min(k, l) is clamped (TSK_WARN_RANK_CLAMPED). */
tsk_status sketch_apply_two_sided_scw(tsk_ctx ctx, const float* A, int64_t B, int m, int n, const float* S, int k,
                                      const float* W, int l, int r, float* L, float* R, float* sigma);

/* err[b] = ||A_b - two-sided SCW(A_b, S, W, r)||_F (fp64 dense residual), err [B] fp64. */
tsk_status two_sided_scw_error(tsk_ctx ctx, const float* A, int64_t B, int m, int n, const float* S, int k,
                               const float* W, int l, int r, double* err);

/* ---------------------------------------------------------------------- matrix-free sketch */
/* the Tucker1 sketch approximated by randomized block
   Krylov on A_(1) without forming the m x m Gram -- the pass-efficient direction the paper names as
   future work.  Not the paper's algorithm: readings mf1-mf4 in DESIGN.md.  Host or device
   pointers (host arrays staged whole, synchronous; as the two-sided entry points).
     Q_0 = orth(Omega);  for j = 1..q: Y_j = sum_d A_d (A_d^T Q_{j-1}),
       Krylov (default): Y_j -= sum_{i<j} Q_i Q_i^T Y_j (twice), Q_j = orth(Y_j), K = [Q_0|...|Q_q]
       subspace:         Q_j = orth(Y_j), K = Q_q
     Rayleigh-Ritz: Z_d = A_d^T K, H = sum_d Z_d^T Z_d = K^T G K, (theta, W) = eig(H) decreasing,
     S = (K W_k)^T (sign rule c5), lambda = theta_1..theta_k.
   Cost: 2q + 1 passes over A (3xTF32 tensor-core products), no m x m matrix.  The result is an
   approximation of the exact sketch: Ritz values satisfy theta_i <= lambda_i(G) (interlacing) and
   converge to them as q grows, at a rate set by the gap at k.
   orth() is fp64 CholQR2; on breakdown (a block numerically dependent on the previous ones) the
   dependent directions are replaced by pseudo-random ones orthogonal to K (reading mf3). */
typedef struct {
  int oversample;       /* block width p = k + oversample, rounded up to a multiple of 4, <= m;
                           default (<= 0): 16 */
  int power_iters;      /* q >= 0; default (< 0): the largest q <= 2 with width <= min(m, 256) */
  int subspace;         /* 1: plain subspace iteration (K = Q_q); 0 (default): block Krylov */
  const double* omega;  /* optional [m][p] fp64 start block (p as above; host or device); NULL = deterministic
                           pseudo-random uniform(-1, 1) block */
} tsk_mf_opts;

typedef struct {
  int block;            /* p */
  int power_iters;      /* q used */
  int width;            /* columns of K: (q + 1) p (Krylov) or p (subspace) */
  int passes;           /* passes over the training stack: 2 q + 1 */
  int repairs;          /* blocks completed with pseudo-random directions (breakdown) */
  double kyfan;         /* sum_{i<k} theta_i = tr(S G S^T) */
} tsk_mf_info;

/* A [D][m][n] fp32 (n % 4 == 0); S [k][m] fp32 (orthonormal rows, decreasing theta); lambda [k] fp64
   (may be NULL).  Requires 1 <= k <= p and width <= min(m, 256) (TSK_EINVAL otherwise). */
tsk_status sketch_train_matrix_free(tsk_ctx ctx, const float* A, int64_t D, int m, int n, int k, float* S,
                                    double* lambda, const tsk_mf_opts* opts, tsk_mf_info* info);

/* ---------------------------------------------------------------------- diagnostics */

/* Diagnostic entry to the Gram kernel (tests / microbenchmarks only; not part of the method):
   same contract as sketch_gram (device pointers only, accumulate = 0) with
     mode bit 0: skip the in-shared-memory hi/lo split (the MMA consumes the raw fp32 tiles),
     mode bit 1: issue only the H*H^T product (1xTF32),
     mode bit 2: disable the drift throttle between units sharing a K window,
     mode bit 3: use the SS kernel variant (A operand from shared memory instead of TMEM),
     mode bit 4: use the 1-CTA TS kernel instead of the CTA-pair kernel,
     mode bit 5: CTA-pair kernel with mbarrier waits that spin without a suspend-time hint,
   chain / splits as in tsk_train_opts (0 = default). */
tsk_status tsk_gram_probe(tsk_ctx ctx, const float* A, int64_t D, int m, int n, double* G64, int mode, int chain,
                          int splits);

/* Diagnostic: the batched symmetric eigensolver used inside sketch_topk / SCW (device pointers).
   H [batch][p][p] fp64 symmetric (row-major); W [batch][p][p] eigenvectors as columns; lam
   [batch][p] eigenvalues, decreasing; sweeps [batch] (may be NULL) Jacobi sweeps used.  p <= 256. */
tsk_status tsk_eig_probe(tsk_ctx ctx, const double* H, int p, int batch, double* W, double* lam, int* sweeps);

/* Diagnostic: the dense symmetric eigensolver of the Rayleigh-Ritz step (Householder tridiagonalisation,
   multisection bisection, twisted-factorisation eigenvectors; device pointers).  H [p][p] fp64 symmetric
   (row-major, read as (H + H^T)/2); W [p][nw] the top nw eigenvectors as columns; lam [nw] decreasing;
   flag (device int, may be NULL; set to 1 -- never cleared -- when max |W^T W - I| > orth_tol, i.e. an
   eigenvalue cluster the vectors could not resolve).  1 <= nw <= p <= 256. */
tsk_status tsk_syev_probe(tsk_ctx ctx, const double* H, int p, int nw, double* W, double* lam, int* flag,
                          double orth_tol);

#ifdef __cplusplus
}
#endif
#endif /* TSKETCH_H_ */
