// Internal declarations of libtsketch (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <cstdio>
#include <cstdlib>

#include "../../include/tsketch.h"

struct tsk_ctx_s;

namespace tsk {

// launch check: TSK_ECUDA on a launch error, with the CUDA message on stderr when TSK_DEBUG is set
inline tsk_status launch_status(const char* where) {
  const cudaError_t e = cudaPeekAtLastError();
  if (e == cudaSuccess) return TSK_OK;
  if (getenv("TSK_DEBUG")) fprintf(stderr, "[tsk] %s: %s\n", where, cudaGetErrorString(e));
  return TSK_ECUDA;
}

// one bit per device: kernel attributes (dynamic shared memory limits) are per device, so the
// "set once" flags of the launch helpers are kept per device
inline uint64_t device_bit() {
  int d = 0;
  cudaGetDevice(&d);
  return 1ull << (d & 63);
}

enum WorkspaceId {
  WS_GEMM_PARTIAL = 0,
  WS_EIG_A,      // fp64 m x p blocks
  WS_EIG_B,
  WS_EIG_C,
  WS_EIG_Q32,    // fp32 p x m (Q^T for the tensor-core product)
  WS_EIG_SMALL,  // fp64 p x p matrices, flags
  WS_EIG_G32,    // fp32 copy of G
  WS_HOST_IN,    // device staging of host inputs
  WS_HOST_OUT,
  WS_SCW_0,
  WS_SCW_1,
  WS_SCW_2,
  WS_SCW_3,
  WS_SCW_4,
  WS_SCW_5,
  WS_SCW_S,        // SCW: S with a 16-byte row pitch when m % 4 != 0
  WS_GRAM,       // fp64 Gram for sketch_train
  WS_JACOBI,
  WS_GEMM_PROGRESS,
  WS_GRAM_SCHED,   // pair-Gram schedule (units, tile map)
  WS_T2_G1,        // two-sided: projected mode-1 Gram (m x m fp64)
  WS_T2_G2,        // two-sided: projected mode-2 Gram (n x n fp64)
  WS_T2_Y,         // two-sided: A_d W^T stack
  WS_T2_Z,         // two-sided: A_d^T S^T stack
  WS_T2_SMALL,
  WS_SCW2_0,       // two-sided SCW scratch
  WS_SCW2_1,
  WS_SCW2_2,
  WS_MF_K,         // matrix-free sketch: Krylov blocks [nb][m][p] fp64
  WS_MF_Y,         // matrix-free sketch: product / temporaries (fp64)
  WS_MF_Z,         // matrix-free sketch: A_d^T K stack (fp32)
  WS_MF_Q32,       // matrix-free sketch: K^T (fp32, tensor-core operand)
  WS_MF_SMALL,     // matrix-free sketch: small fp64 matrices, flags
  WS_MF_SCR,       // matrix-free sketch: fp64 GEMM split scratch
  WS_CHECK,        // input validation flag (check_finite)
  WS_EIG_GQ,       // eigensolver: split-K partial tiles + tickets of the fp64 product
  WS_SYEV,         // small symmetric eigensolver: reflectors, tridiagonal, scratch
  WS_GATHER,       // tsk_allgather_errors: padded [P][per] gather buffer
  WS_SCW_EIG,    // per-part eigensolver scratch of the batched SCW (its parts run concurrently)
  WS_STAGE_0,    // host-pointer staging of the whole-array entry points (two-sided, matrix-free): 8 slots
  WS_STAGE_LAST = WS_STAGE_0 + 7,
  WS_COUNT
};

// per-context host-side caches (e.g. the pair-Gram schedule): owned by the ctx, freed with it
struct HostCache {
  virtual ~HostCache() = default;
};

struct Ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  void* ws[WS_COUNT] = {};
  size_t ws_size[WS_COUNT] = {};
  void* host_pinned = nullptr;  // small pinned scratch for flags / scalars
  size_t host_pinned_size = 0;

  // grow-only device workspace; returns nullptr on allocation failure
  void* workspace(int id, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (ws_size[id] >= bytes) return ws[id];
    if (ws[id]) {
      // the old buffer may be in use on this ctx's stream or its side stream (batched SCW)
      cudaDeviceSynchronize();
      cudaFree(ws[id]);
      ws[id] = nullptr;
      ws_size[id] = 0;
    }
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    ws[id] = p;
    ws_size[id] = bytes;
    return p;
  }
  void* pinned(size_t bytes) {
    if (host_pinned_size >= bytes) return host_pinned;
    if (host_pinned) cudaFreeHost(host_pinned);
    host_pinned = nullptr;
    host_pinned_size = 0;
    if (cudaMallocHost(&host_pinned, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    host_pinned_size = bytes;
    return host_pinned;
  }
  void count_launch(int n = 1) { launches += n; }
  // scw_error's error formula (tsk_set_scw_error_mode): 0 = Pythagorean identity with the dense
  // residual below tau ||A||^2 (tau <= 0: the library default), 1 = dense residual for every matrix
  int scw_err_mode = 0;
  double scw_tau = 0.0;
  // NCCL communicator of tsk_comm_init (ncclComm_t, opaque here; nullptr = single GPU)
  void* comm = nullptr;
  int nranks = 1, rank = 0;
  // side stream + fork/join events (batched SCW runs two halves of a chunk concurrently), created on
  // first use and destroyed with the ctx
  static constexpr int kSide = 3;
  cudaStream_t side[kSide] = {};
  cudaEvent_t ev[2 * kSide + 1] = {};  // [0] fork, [1 + j] after part j's first product, [1 + kSide + j] join
  bool side_ready() {
    if (side[0]) return true;
    for (auto& st : side)
      if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
    for (auto& e : ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
    return true;
  }
  // pair-Gram schedule last uploaded to ws[WS_GRAM_SCHED] (pointer + host schedule version)
  const void* gram_sched_dev = nullptr;
  long long gram_sched_ver = -1;
  std::unique_ptr<HostCache> gram_sched;  // host schedule of the last pair-Gram shape (gram_pair.cu)
};

struct GemmInfo {
  int splits = 0, units = 0, grid = 0, tiles = 0;
};

// C[M x N] (+)= sum_{z<D} X_z Y_z^T   (fp32 K-major operands via 3-D TMA maps)
struct GemmProblem {
  const float* X = nullptr;
  const float* Y = nullptr;
  int M = 0, N = 0, n = 0;
  long long D = 1;
  long long x_row_stride = 0, x_slice_stride = 0;
  long long y_row_stride = 0, y_slice_stride = 0;
  int sym = 0;
  double* out64 = nullptr;
  long long ldo64 = 0;
  float* out32 = nullptr;
  long long ldo32 = 0;
  int accumulate = 0;
  int splits = 0;               // 0 = auto
  int min_chunks_per_unit = 0;  // 0 = default
  int chain = 0;                // 0 = default
  int fold = 0;
  int products = 3;
  int raw = 0;
  int lag = -1;  // drift throttle (chunks); -1 = default, 0 = off
  int ss = 0;    // 1: force the SS kernel variant (A operand from shared memory)
  int spin_waits = 0;  // pair Gram: mbarrier waits without a suspend-time hint (diagnostics)
  int one_cta = 0;  // 1: symmetric Gram on the 1-CTA TS kernel instead of CTA pairs (diagnostics)
  int batch = 0;          // 1: D independent problems (no contraction over slices)
  int xt = 0;             // 1: X_z stored transposed, [K = n][M] with M contiguous (x_row_stride = K stride)
  int ybc = 0;            // 1: Y broadcast (slice 0 for every z; TS kernel only)
  int yt = 0;             // 1: Y_z stored transposed, [K = n][N] with N contiguous (y_row_stride = K stride)
  int drow = 0;           // direct output row-major: dout[b * dstride + row * ldd + col]
  // residual epilogue (batch mode): res_part[unit][8] = sum over the tile of (resA - X Y^T)^2
  const float* resA = nullptr;
  long long res_stride = 0;
  int res_ld = 0;
  double* res_part = nullptr;
  // batch mode: only problems b with only[b] != 0 are computed (the others' outputs are not written)
  const int* only = nullptr;
  const int* only_any = nullptr;  // optional: device count of nonzero only[b] (0: the launch does nothing)
  // TS kernel, batch mode: sq_part[unit][8] = fp64 sums of the squared X elements each unit reads
  // (unit u of problem b: u = b * tiles + tile; every X element of a problem in exactly one unit when N
  // fits one column block)
  double* sq_part = nullptr;
  int bn = 128;           // MMA N tile: 128 or 64
  float* dout = nullptr;  // direct fp32 output, transposed: dout[b * dstride + col * ldd + row]
  long long dstride = 0;
  int ldd = 0;
  GemmInfo* info = nullptr;
};

tsk_status gemm_tf32x3(Ctx* ctx, const GemmProblem& p);
// symmetric Gram on CTA pairs (tcgen05 cta_group::2), gram_pair.cu
tsk_status gram_pair(Ctx* ctx, const GemmProblem& p);

// two-sided variant (tucker2.cu)
tsk_status gram_mode2(Ctx* ctx, const float* A, long long D, int m, int n, double* G64, int accumulate);
tsk_status hooi_tucker2(Ctx* ctx, const float* A, long long D, int m, int n, int k, int l, float* S, float* W,
                        const tsk_hooi_opts* o, tsk_hooi_info* info);
// two-sided SCW (Algorithm 3), scw.cu; device pointers
tsk_status scw2_run(Ctx* ctx, const float* A, long long B, int m, int n, const float* S, int k, const float* W, int l,
                    int r, float* L, float* R, float* sigma, double* err);

// matrix-free Tucker1 sketch by randomized block Krylov (matrix_free.cu), device pointers
tsk_status matrix_free_sketch(Ctx* ctx, const float* A, long long D, int m, int n, int k, float* S, double* lambda,
                              const tsk_mf_opts* o, tsk_mf_info* info);

// eigensolver (eig.cu)
tsk_status topk_eigen(Ctx* ctx, const double* G64, int m, int k, float* S, double* lambda, const tsk_train_opts* o,
                      tsk_train_info* info);
// f64_products: fp64 G Q products (small m); X64 (optional): the eigenvectors [m][k] fp64, columns
tsk_status topk_eigen_ex(Ctx* ctx, const double* G64, int m, int k, float* S, double* lambda,
                         const tsk_train_opts* o, tsk_train_info* info, int f64_products, double* X64);

// SCW (scw.cu); all pointers device
tsk_status scw_run(Ctx* ctx, const float* A, long long B, int m, int n, const float* S, int k, int r, float* L,
                   float* R, float* sigma, double* err);

// top nw eigenpairs of a dense symmetric p x p matrix (p <= 256), syev.cu: W [p][ldw] columns,
// lam [nw] decreasing; flag (device, may be null) set to 1 if the vectors are not orthonormal to orth_tol
tsk_status syev_top(Ctx* ctx, const double* H, int p, int nw, double* W, int ldw, double* lam, int* flag,
                    double orth_tol);
// the same for a batch: H [batch][p][p], W [batch][p][ldw], lam [batch][nw]; flag set if any problem fails
// ws (optional): caller-owned scratch of syev_ws_doubles(p) doubles per problem (else the ctx's WS_SYEV,
// which two concurrent calls on different streams must not share)
// vmode 1: eigenvalues only (tridiagonalisation + bisection; no vectors, no orthogonality flag); vmode 2: the
// vectors (and values) of the problems with only[b] != 0, reusing the tridiagonalisation of a vmode-1 call
// on the same ws (batched small-p path; elsewhere vmode 1 computes everything and vmode 2 does nothing)
tsk_status syev_top_batched(Ctx* ctx, const double* H, int p, int nw, int batch, double* W, int ldw, double* lam,
                            int* flag, double orth_tol, long long lstride = 0, double* ws = nullptr, int vmode = 0,
                            const int* only = nullptr);
long long syev_ws_doubles(int p);

// batched symmetric PSD eigensolver (one-sided Jacobi), jacobi.cu
// H: [batch][p][p] fp64 symmetric (row-major, read only).  W: [batch][p][p] fp64 eigenvectors as
// COLUMNS (W[b][i][c] = component i of eigenvector c), lam: [batch][p] fp64 decreasing.
// gate (device int, may be null): the kernel returns at once unless *gate != 0 (a device-side fallback
// behind syev_top_batched's orthogonality flag, no host round trip)
// scratch (optional): caller-owned, jacobi_ws_doubles(p) doubles per problem (used only for p where the
// matrix pair does not fit shared memory; else the ctx's WS_JACOBI)
tsk_status jacobi_eig_batched(Ctx* ctx, const double* H, int p, int batch, double* W, double* lam,
                              int* sweeps = nullptr, double tol = 1e-13, const int* gate = nullptr,
                              double* scratch = nullptr);
long long jacobi_ws_doubles(int p);

}  // namespace tsk

struct tsk_ctx_s {
  tsk::Ctx c;
};
