// Batched symmetric eigensolver: cyclic two-sided Jacobi, one CTA per matrix.  Used for the
// Rayleigh-Ritz step of the top-k eigensolver (S = top-k eigenvectors of G) and
// for the small k x k problems of SCW (the SVDs of Algorithm 1 lines 1-2, PAPER.md:61-62,
// taken through their Gram matrices).
//
// Each round applies p/2 disjoint plane rotations (round-robin "circle" ordering), chosen to
// annihilate A_ij (Golub & Van Loan's symmetric Schur decomposition): the rotation parameters
// need only A_ii, A_jj, A_ij (no reductions), then all row rotations, then all column rotations
// (and V <- V J) are applied in parallel.  A sweep is p-1 rounds; sweeps repeat until no pair
// has |A_ij| > tol * sqrt(|A_ii A_jj|).  A and V live in shared memory (padded rows) when they
// fit, else in a global (L2-resident) scratch.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "ptx.cuh"
#include "tsk_internal.h"

namespace tsk {

constexpr int kJacThreads = 1024;
constexpr int kJacSmemMax = 222 * 1024;  // dynamic part: p <= 118 keeps A and V in shared memory

// pair k of round r in the circle ordering over pe (even) indices, no divisions
__device__ __forceinline__ void rr_pair(int r, int k, int pe, int& i, int& j) {
  const int n1 = pe - 1;
  if (k == 0) {
    i = r;
    j = n1;
  } else {
    i = r + k;
    if (i >= n1) i -= n1;
    j = r - k;
    if (j < 0) j += n1;
  }
  if (i > j) { const int t = i; i = j; j = t; }
}

// One half-warp (16 lanes) per rotation pair.  Phase 1 (per pair, no barrier needed because
// pairs are disjoint): every lane of the half-warp computes (c, s) from A_ii, A_jj, A_ij
// (broadcast reads: no shuffles, no divergence) and the half-warp rotates rows i and j.  Phase 2:
// the half-warp rotates columns i and j of A and of V.  NQ = ceil(p / 16) strided elements per
// lane, unrolled; KQ = pairs per half-warp (1, or 2 when p > 128).
template <bool kSmem, int NQ, int KQ>
__global__ void __launch_bounds__(kJacThreads)
    jacobi_eig_kernel(const double* __restrict__ H, int p, double* __restrict__ W, double* __restrict__ lam,
                      double* __restrict__ gscratch, int max_sweeps, double tol, int* __restrict__ sweeps_out,
                      const int* __restrict__ gate) {
  if (gate && *gate == 0) return;  // uniform: device-side fallback not needed
  extern __shared__ double jsm[];
  __shared__ int rot_count;
  __shared__ double lam_s[256];
  const int b = blockIdx.x;
  const int pe = p + (p & 1);
  const int ld = p + 1;  // padded row stride
  double* A = kSmem ? jsm : gscratch + (size_t)b * 2 * p * ld;
  double* V = A + (size_t)p * ld;
  const double* Hb = H + (size_t)b * p * p;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int hw = tid >> 4, hl = tid & 15, nhw = nt >> 4;  // half-warp id / lane
  const int npairs = pe / 2;
  __shared__ double amax_s;

  for (int e = tid; e < p * p; e += nt) {
    const int i = e / p, j = e - (e / p) * p;
    A[i * ld + j] = 0.5 * (Hb[(size_t)i * p + j] + Hb[(size_t)j * p + i]);
    V[i * ld + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();  // the diagonal scan below reads entries other threads wrote
  if (tid == 0) {
    double am = 0.0;
    for (int i = 0; i < p; ++i) am = fmax(am, fabs(A[i * ld + i]));
    amax_s = am;
  }
  __syncthreads();
  // absolute floor: off-diagonals below 1e-15 * max|A_ii| are rounding noise of the updates
  const double floor2 = (1e-15 * amax_s) * (1e-15 * amax_s);
  const double tol2 = tol * tol;

  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) rot_count = 0;
    __syncthreads();
    for (int r = 0; r < pe - 1; ++r) {
      double cc[KQ], ss[KQ];  // parameters of the pairs this half-warp owns this round
      int ii[KQ], jj[KQ];
#pragma unroll
      for (int q = 0; q < KQ; ++q) {
        const int k = hw + q * nhw;
        cc[q] = 1.0;
        ss[q] = 0.0;
        ii[q] = 0;
        jj[q] = 0;
        if (k < npairs) {
          int i, j;
          rr_pair(r, k, pe, i, j);
          ii[q] = i;
          jj[q] = j;
          if (j < p) {
            const double aii = A[i * ld + i], ajj = A[j * ld + j], aij = A[i * ld + j];
            // |A_ij| > max(tol sqrt|A_ii A_jj|, floor), squared: no fp64 square root on the chain
            if (aij * aij > fmax(tol2 * fabs(aii * ajj), floor2)) {
              // tan of the annihilating angle, in fp32 (the MUFU path; ~1e-7 relative).  Any t
              // gives an exactly orthogonal fp64 rotation (c^2 + s^2 = 1 to fp64 rounding); the
              // residual ~1e-7 A_ij it leaves is removed by the quadratically convergent sweeps.
              const float tau = __fdividef((float)(ajj - aii), (float)(2.0 * aij));
              const float tf = (tau >= 0.f ? 1.f : -1.f) / (fabsf(tau) + sqrtf(1.f + tau * tau));
              const double t = (double)tf;
              const double x = 1.0 + t * t;
              double y = (double)rsqrtf((float)x);  // c = x^-1/2: two fp64 Newton steps
              y = y * (1.5 - 0.5 * x * y * y);
              y = y * (1.5 - 0.5 * x * y * y);
              cc[q] = y;
              ss[q] = t * y;
              if (hl == 0) rot_count = 1;  // benign race: every writer stores 1
            }
          }
        }
      }
      // all reads of this round's diagonal entries precede the row updates (rows i, j of other
      // pairs are disjoint from this pair's, but A_ii / A_jj of THIS pair are rewritten below)
      __syncwarp();
#pragma unroll
      for (int q = 0; q < KQ; ++q) {
        const double c = cc[q], s = ss[q];
        if (s != 0.0) {
          double* Ai = A + ii[q] * ld;
          double* Aj = A + jj[q] * ld;
#pragma unroll
          for (int u = 0; u < NQ; ++u) {
            const int x = hl + 16 * u;
            if (x < p) {
              const double ai = Ai[x], aj = Aj[x];
              Ai[x] = c * ai - s * aj;
              Aj[x] = s * ai + c * aj;
            }
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < KQ; ++q) {
        const double c = cc[q], s = ss[q];
        if (s == 0.0) continue;
        const int i = ii[q], j = jj[q];
#pragma unroll
        for (int u = 0; u < NQ; ++u) {
          const int x = hl + 16 * u;
          if (x < p) {
            double* Ax = A + x * ld;
            double* Vx = V + x * ld;
            const double ai = Ax[i], aj = Ax[j];
            Ax[i] = c * ai - s * aj;
            Ax[j] = s * ai + c * aj;
            const double vi = Vx[i], vj = Vx[j];
            Vx[i] = c * vi - s * vj;
            Vx[j] = s * vi + c * vj;
          }
        }
      }
      __syncthreads();
    }
    if (rot_count == 0) break;
    __syncthreads();
  }
  if (sweeps_out && tid == 0) sweeps_out[b] = sweep;

  for (int c = tid; c < p; c += nt) lam_s[c] = A[c * ld + c];
  __syncthreads();
  // sort decreasing (stable: ties keep the lower index first); eigenvectors as columns of W
  double* Wb = W + (size_t)b * p * p;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  for (int c = warp; c < p; c += nw) {
    const double lc = lam_s[c];
    int rank = 0;
    for (int c2 = 0; c2 < p; ++c2) {
      const double l2 = lam_s[c2];
      rank += (l2 > lc) || (l2 == lc && c2 < c);
    }
    if (lane == 0) lam[(size_t)b * p + rank] = lc;
    for (int x = lane; x < p; x += 32) Wb[(size_t)x * p + rank] = V[x * ld + c];
  }
}

template <bool kSmem, int NQ, int KQ>
static void launch_jacobi(int batch, int threads, size_t smem, cudaStream_t st, const double* H, int p, double* W,
                          double* lam, double* scratch, double tol, int* sweeps, const int* gate) {
  static uint64_t attr = 0;
  if (kSmem && !(attr & device_bit())) {
    cudaFuncSetAttribute(jacobi_eig_kernel<kSmem, NQ, KQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, kJacSmemMax);
    attr |= device_bit();
  }
  jacobi_eig_kernel<kSmem, NQ, KQ><<<batch, threads, smem, st>>>(H, p, W, lam, scratch, 30, tol, sweeps, gate);
}

long long jacobi_ws_doubles(int p) { return (long long)2 * p * (p + 1); }

tsk_status jacobi_eig_batched(Ctx* ctx, const double* H, int p, int batch, double* W, double* lam, int* sweeps,
                              double tol, const int* gate, double* scratch_ext) {
  if (p < 1 || p > 256 || batch < 0) return TSK_EINVAL;
  if (batch == 0) return TSK_OK;
  const size_t need = (size_t)jacobi_ws_doubles(p) * sizeof(double);
  int use_smem = need <= (size_t)kJacSmemMax;
  double* scratch = nullptr;
  if (!use_smem) {
    scratch = scratch_ext ? scratch_ext : reinterpret_cast<double*>(ctx->workspace(WS_JACOBI, need * batch));
    if (!scratch) return TSK_ENOMEM;
  }
  const size_t smem = use_smem ? need : 0;
  // Rotate while |A_ij| > tol sqrt(|A_ii A_jj|) (and above an absolute rounding floor); the
  // eigenvectors come out accurate to ~tol / relative gap.
  // one half-warp per pair: p/2 pairs -> 8 p threads (at most 2 pairs per half-warp at p = 256)
  const int threads = std::min(kJacThreads, std::max(64, ((p + 1) / 2 * 16 + 31) / 32 * 32));
  cudaStream_t st = ctx->stream;
  if (use_smem) {
    if (p <= 32) launch_jacobi<true, 2, 1>(batch, threads, smem, st, H, p, W, lam, nullptr, tol, sweeps, gate);
    else if (p <= 64) launch_jacobi<true, 4, 1>(batch, threads, smem, st, H, p, W, lam, nullptr, tol, sweeps, gate);
    else launch_jacobi<true, 8, 1>(batch, threads, smem, st, H, p, W, lam, nullptr, tol, sweeps, gate);
  } else {
    if (p <= 128) launch_jacobi<false, 8, 1>(batch, threads, 0, st, H, p, W, lam, scratch, tol, sweeps, gate);
    else launch_jacobi<false, 16, 2>(batch, threads, 0, st, H, p, W, lam, scratch, tol, sweeps, gate);
  }
  if (cudaPeekAtLastError() != cudaSuccess) return TSK_ECUDA;
  ctx->count_launch();
  return TSK_OK;
}

}  // namespace tsk
