// Batched symmetric eigensolver by one-sided (Hestenes) Jacobi, one CTA per matrix,
// warp-level rotations.  Used for the Rayleigh-Ritz step of the top-k eigensolver
// (S = top-k eigenvectors of G) and for the small k x k problems of SCW
// (the SVDs of Algorithm 1 lines 1-2, done through Gram matrices).
//
// Columns of A (initially H) and V (initially I) are rotated together until all column
// pairs of A are orthogonal: A = H V with V orthogonal, so V holds the eigenvectors and
// lambda_c = a_c . v_c.  Pairs are scheduled in the round-robin ("circle") order, p/2
// disjoint pairs per round, one warp per pair.  Storage is column-major fp64 in shared
// memory when 2*p*p*8 bytes fit, otherwise in a global (L2-resident) scratch.
#include <algorithm>
#include <cmath>

#include "ptx.cuh"
#include "tsk_internal.h"

namespace tsk {

constexpr int kJacThreads = 512;
constexpr int kJacSmemMax = 200 * 1024;

__device__ __forceinline__ void rr_pair(int r, int k, int pe, int& i, int& j) {
  const int n1 = pe - 1;
  if (k == 0) {
    i = r;
    j = n1;
  } else {
    i = (r + k) % n1;
    j = (r - k + n1) % n1;
  }
  if (i > j) { int t = i; i = j; j = t; }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kJacThreads)
    jacobi_eig_kernel(const double* __restrict__ H, int p, double* __restrict__ W, double* __restrict__ lam,
                      double* __restrict__ gscratch, int use_smem, int max_sweeps, double tol) {
  extern __shared__ double jsm[];
  __shared__ int rot_count;
  __shared__ double lam_s[256];
  const int b = blockIdx.x;
  const int pe = p + (p & 1);
  double* Acol = use_smem ? jsm : gscratch + (size_t)b * 2 * pe * p;
  double* Vcol = Acol + (size_t)pe * p;
  const double* Hb = H + (size_t)b * p * p;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;

  for (int idx = tid; idx < pe * p; idx += blockDim.x) {
    const int c = idx / p, i = idx % p;
    Acol[idx] = (c < p) ? 0.5 * (Hb[(size_t)c * p + i] + Hb[(size_t)i * p + c]) : 0.0;
    Vcol[idx] = (c == i) ? 1.0 : 0.0;
  }
  __syncthreads();

  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) rot_count = 0;
    __syncthreads();
    for (int r = 0; r < pe - 1; ++r) {
      for (int k = warp; k < pe / 2; k += nw) {
        int ci, cj;
        rr_pair(r, k, pe, ci, cj);
        if (cj >= p) continue;  // dummy column of odd p
        double* ai = Acol + (size_t)ci * p;
        double* aj = Acol + (size_t)cj * p;
        double al = 0, be = 0, ga = 0;
        for (int x = lane; x < p; x += 32) {
          const double u = ai[x], v = aj[x];
          al += u * u;
          be += v * v;
          ga += u * v;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (fabs(ga) > tol * sqrt(al * be) && al > 0.0 && be > 0.0) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t);
          const double s = c * t;
          double* vi = Vcol + (size_t)ci * p;
          double* vj = Vcol + (size_t)cj * p;
          for (int x = lane; x < p; x += 32) {
            const double u = ai[x], v = aj[x];
            ai[x] = c * u - s * v;
            aj[x] = s * u + c * v;
            const double vu = vi[x], vv = vj[x];
            vi[x] = c * vu - s * vv;
            vj[x] = s * vu + c * vv;
          }
          if (lane == 0) atomicAdd(&rot_count, 1);
        }
        __syncwarp();
      }
      __syncthreads();
    }
    if (rot_count == 0) break;
    __syncthreads();
  }

  // eigenvalues lambda_c = a_c . v_c  (A = H V)
  for (int c = warp; c < p; c += nw) {
    const double* ac = Acol + (size_t)c * p;
    const double* vc = Vcol + (size_t)c * p;
    double s = 0;
    for (int x = lane; x < p; x += 32) s += ac[x] * vc[x];
    s = warp_sum(s);
    if (lane == 0) lam_s[c] = s;
  }
  __syncthreads();
  // sort decreasing (stable: ties keep the lower column first)
  double* Wb = W + (size_t)b * p * p;
  for (int c = warp; c < p; c += nw) {
    const double lc = lam_s[c];
    int rank = 0;
    for (int c2 = 0; c2 < p; ++c2) {
      const double l2 = lam_s[c2];
      rank += (l2 > lc) || (l2 == lc && c2 < c);
    }
    const double* vc = Vcol + (size_t)c * p;
    for (int x = lane; x < p; x += 32) Wb[(size_t)x * p + rank] = vc[x];
    if (lane == 0) lam[(size_t)b * p + rank] = lc;
  }
}

tsk_status jacobi_eig_batched(Ctx* ctx, const double* H, int p, int batch, double* W, double* lam) {
  if (p < 1 || p > 256 || batch < 0) return TSK_EINVAL;
  if (batch == 0) return TSK_OK;
  const int pe = p + (p & 1);
  const size_t need = (size_t)2 * pe * p * sizeof(double);
  int use_smem = need <= (size_t)kJacSmemMax;
  double* scratch = nullptr;
  if (!use_smem) {
    scratch = reinterpret_cast<double*>(ctx->workspace(WS_JACOBI, need * batch));
    if (!scratch) return TSK_ENOMEM;
  }
  const size_t smem = use_smem ? need : 0;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(jacobi_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kJacSmemMax) !=
        cudaSuccess)
      return TSK_ECUDA;
    attr = true;
  }
  const int threads = p <= 64 ? 256 : kJacThreads;
  const double tol = 8.9e-16 * sqrt((double)p);  // ~4 eps sqrt(p), cf. one-sided Jacobi SVD practice
  jacobi_eig_kernel<<<batch, threads, smem, ctx->stream>>>(H, p, W, lam, scratch, use_smem, 40, tol);
  if (cudaPeekAtLastError() != cudaSuccess) return TSK_ECUDA;
  ctx->count_launch();
  return TSK_OK;
}

}  // namespace tsk
