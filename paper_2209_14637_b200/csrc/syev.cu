// Small dense symmetric eigensolver (fp64, p <= 256): the Rayleigh-Ritz step of the top-k
// eigensolver (S = top-k eigenvectors of G, Algorithm 2 line 2) and the dense
// path for small m.
//
//   1. trd_kernel   (one CTA)  Householder tridiagonalisation H = Q T Q^T (LAPACK dsytd2 order:
//                              reflector j annihilates column j below the subdiagonal)
//   2. tev_kernel   (one CTA per wanted eigenpair)  the i-th largest eigenvalue of T by
//                              multisection of the Sturm count (scaled three-term determinant
//                              recurrence: FMA-only chain), its eigenvector by a twisted
//                              factorisation of T - lambda I (forward LDL^T and backward UDU^T
//                              concurrently, twist at min |gamma_r|), then back-transformed by
//                              the Householder reflectors
//   3. orth_kernel  (one CTA)  max |W^T W - I|: eigenvalues closer than the vectors can resolve
//                              (clusters at ~1e-10 ||T|| and below, e.g. a null space) give
//                              non-orthogonal vectors; the caller then falls back to Jacobi.
// Every eigenpair is independent (no reductions across CTAs): deterministic.
//
// Why not the one-CTA Jacobi of jacobi.cu: its p - 1 rounds per sweep are latency chains
// (~1.8 us per round at p = 76, 5-13 sweeps); here the sequential part is p Householder steps of
// ~4 barriers each, and the spectrum work is parallel over eigenpairs.
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "ptx.cuh"
#include "tsk_internal.h"

namespace tsk {

constexpr int kTrdThreads = 512;
#ifdef TSK_TRD_PROF
__device__ long long trd_prof[4];  // diagnostic build only: cycles of the three phases of trd_kernel's steps
#endif
constexpr int kTrdSmemMaxP = 160;  // A (p x (p+1) fp64) in shared memory up to p = 160

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Householder tridiagonalisation of the symmetric p x p matrix H (read as (H + H^T)/2).
// Outputs: d[p] diagonal, e[p-1] subdiagonal, tau[p-2] and reflector rows refl[j][j+1..p-1]
// (v_j[0] = 1 stored explicitly) so that H = Q T Q^T with Q = H_0 H_1 ... H_{p-3},
// H_j = I - tau_j v_j v_j^T acting on indices j+1..p-1.
// Delayed update: the rank-2 update A -= v w^T + w v^T of step j-1 is applied to column j by
// warp 0 while it builds v_j (no barrier), and to the trailing block in the same pass that forms
// the product A v_j -- one pass over A and three barriers per step.  Thread (ty, tx) of the 16 x 32
// layout owns rows ty + 16 r and columns tx + 32 c of the trailing block; row sums are reduced
// across the warp.  KR x KC bounds the rows / columns per thread (8 x 4 for p <= 129).
// kRow (p <= 129, A in shared memory; used up to p = 88): the fused pass is row-parallel instead -- four threads per row,
// each a strided quarter of the columns, reduced with two shuffles (the 16 x 32 layout's butterfly over
// 32 lanes and its 8 x 4 register tile made that pass a ~1400-cycle latency floor per step: measured with
// -DTSK_TRD_PROF, phase 2 of a p = 76 step took 1950 cycles of 4350).
template <bool kSmem, int KR, int KC, bool kRow = false>
__global__ void __launch_bounds__(kTrdThreads) trd_kernel(const double* __restrict__ H, int p,
                                                          double* __restrict__ refl, double* __restrict__ tau_out,
                                                          double* __restrict__ d_out, double* __restrict__ e_out,
                                                          double* __restrict__ gA, long long hs, long long wsz) {
  extern __shared__ double trd_sm[];
  {  // problem blockIdx.y of a batch: H [b][p][p], per-problem workspace stride wsz
    const long long b = blockIdx.y;
    H += b * hs;
    refl += b * wsz;
    tau_out += b * wsz;
    d_out += b * wsz;
    e_out += b * wsz;
    if (gA) gA += b * wsz;
  }
  __shared__ double vs[2][256], ws[2][256], pvs[256];
  __shared__ double sc[4];
  const int ld = kSmem ? p + 1 : p;
  double* A = kSmem ? trd_sm : gA;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int ty = warp, tx = lane;  // 16 x 32
  for (int e = tid; e < p * p; e += nt) {
    const int i = e / p, j = e - (e / p) * p;
    A[i * ld + j] = 0.5 * (H[(size_t)i * p + j] + H[(size_t)j * p + i]);
  }
  for (int i = tid; i < 256; i += nt) {
    vs[0][i] = vs[1][i] = 0.0;
    ws[0][i] = ws[1][i] = 0.0;
  }
  __syncthreads();
#ifdef TSK_TRD_PROF
  long long pf0 = 0, pf1 = 0, pf2 = 0, pc = clock64();
#endif
  for (int j = 0; j + 2 < p; ++j) {
    const int cur = j & 1, prv = cur ^ 1;
    const double* vp = vs[prv];  // pending update v_{j-1}, w_{j-1} (zero at j = 0), indices >= j
    const double* wp = ws[prv];
    if (warp == 0) {
      // column j with the pending update applied; v_j = x / (alpha - beta)
      const double vpj = vp[j], wpj = wp[j];
      double xi[8];
      double s2 = 0.0, alpha = 0.0, ajj = 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = j + lane + 32 * u;
        double a = 0.0;
        if (i < p) a = A[i * ld + j] - fma(vp[i], wpj, wp[i] * vpj);
        xi[u] = a;
        if (i >= j + 2) s2 = fma(a, a, s2);
        if (i == j + 1) alpha = a;
        if (i == j) ajj = a;
      }
      s2 = warp_sum_d(s2);
      alpha = __shfl_sync(0xffffffffu, xi[0], 1);  // rows j + 1 and j sit in lanes 1 and 0
      ajj = __shfl_sync(0xffffffffu, xi[0], 0);
      double tau = 0.0, beta = alpha, scal = 0.0;
      if (s2 > 0.0) {
        const double mu = fast_sqrt(fma(alpha, alpha, s2));
        beta = alpha <= 0.0 ? mu : -mu;
        tau = (beta - alpha) * fast_rcp(beta);
        scal = fast_rcp(alpha - beta);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = j + lane + 32 * u;
        if (i >= j + 1 && i < p) {
          const double v = i == j + 1 ? 1.0 : xi[u] * scal;
          vs[cur][i] = v;
          refl[(size_t)j * p + i] = v;
        }
      }
      if (lane == 0) {
        sc[0] = tau;
        e_out[j] = beta;
        d_out[j] = ajj;
        tau_out[j] = tau;
      }
    }
    __syncthreads();
#ifdef TSK_TRD_PROF
    { const long long c = clock64(); pf0 += c - pc; pc = c; }
#endif
    const double tau = sc[0];
    const double* v = vs[cur];
    // fused pass: A22 -= vp wp^T + wp vp^T (pending), pv = tau A22 v
    if constexpr (kRow) {
      const int i = j + 1 + (tid >> 2), sg = tid & 3;
      double acc0 = 0.0, acc1 = 0.0;
      if (i < p) {
        const double vpi = vp[i], wpi = wp[i];
        double* row = A + i * ld;
        int l = j + 1 + sg;
        for (; l + 4 < p; l += 8) {
          const double a0 = row[l] - fma(vpi, wp[l], wpi * vp[l]);
          const double a1 = row[l + 4] - fma(vpi, wp[l + 4], wpi * vp[l + 4]);
          row[l] = a0;
          row[l + 4] = a1;
          acc0 = fma(a0, v[l], acc0);
          acc1 = fma(a1, v[l + 4], acc1);
        }
        if (l < p) {
          const double a0 = row[l] - fma(vpi, wp[l], wpi * vp[l]);
          row[l] = a0;
          acc0 = fma(a0, v[l], acc0);
        }
      }
      double acc = acc0 + acc1;
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (sg == 0 && i < p) pvs[i] = tau * acc;
    } else {
      double vpc[KC], wpc[KC], vc[KC];
#pragma unroll
      for (int c = 0; c < KC; ++c) {
        const int l = j + 1 + tx + 32 * c;
        const bool ok = l < p;
        vpc[c] = ok ? vp[l] : 0.0;
        wpc[c] = ok ? wp[l] : 0.0;
        vc[c] = ok ? v[l] : 0.0;
      }
      double acc[KR];
#pragma unroll
      for (int r = 0; r < KR; ++r) {
        const int i = j + 1 + ty + 16 * r;
        acc[r] = 0.0;
        if (i < p) {
          const double vpi = vp[i], wpi = wp[i];
          double* row = A + i * ld;
#pragma unroll
          for (int c = 0; c < KC; ++c) {
            const int l = j + 1 + tx + 32 * c;
            if (l < p) {
              const double a = row[l] - fma(vpi, wpc[c], wpi * vpc[c]);
              row[l] = a;
              acc[r] = fma(a, vc[c], acc[r]);
            }
          }
        }
      }
      // butterfly reduce-scatter of the KR row sums over the 32 lanes: at each level a lane keeps
      // half of its rows and sends the other half to its partner (KR - 1 + log2(32 / KR) shuffles
      // instead of 5 KR); afterwards row r's total sits in the lanes whose high bits encode r
      int nrow = KR;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        if (nrow > 1) {
          const bool upper = (lane & o) != 0;
          const int h = nrow >> 1;
#pragma unroll
          for (int q = 0; q < KR / 2; ++q) {
            if (q < h) {
              const double send = upper ? acc[q] : acc[q + h];
              const double recv = __shfl_xor_sync(0xffffffffu, send, o);
              acc[q] = (upper ? acc[q + h] : acc[q]) + recv;
            }
          }
          nrow = h;
        } else {
          acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
        }
      }
      // the row index held by this lane: bits of (lane >> (5 - log2 KR)) read from the top level down
      {
        int r = 0, rows = KR;
#pragma unroll
        for (int o = 16; o >= 1 && rows > 1; o >>= 1) {
          rows >>= 1;
          if (lane & o) r += rows;
        }
        const int i = j + 1 + ty + 16 * r;
        const int owner_bits = 32 / KR;  // lanes sharing row r: the low log2(32 / KR) bits vary
        if ((lane & (owner_bits - 1)) == 0 && i < p) pvs[i] = tau * acc[0];
      }
    }
    __syncthreads();
#ifdef TSK_TRD_PROF
    { const long long c = clock64(); pf1 += c - pc; pc = c; }
#endif
    if (warp == 0) {
      double s = 0.0;
      for (int i = j + 1 + lane; i < p; i += 32) s = fma(pvs[i], v[i], s);
      s = warp_sum_d(s);
      const double K = -0.5 * tau * s;
      for (int i = j + 1 + lane; i < p; i += 32) ws[cur][i] = fma(K, v[i], pvs[i]);
      if (lane == 0) ws[cur][j] = 0.0;  // the pending vectors are read from index j + 1 on
      if (lane == 0) vs[cur][j] = 0.0;
    }
    __syncthreads();
#ifdef TSK_TRD_PROF
    { const long long c = clock64(); pf2 += c - pc; pc = c; }
#endif
  }
#ifdef TSK_TRD_PROF
  if (tid == 0 && blockIdx.y == 0) { trd_prof[0] = pf0; trd_prof[1] = pf1; trd_prof[2] = pf2; trd_prof[3] = p; }
#endif
  if (tid == 0) {
    if (p >= 3) {
      // the last 2 x 2 block with the pending update of step p - 3
      const double* vp = vs[(p - 3) & 1];
      const double* wp = ws[(p - 3) & 1];
      const int a = p - 2, b = p - 1;
      d_out[a] = A[a * ld + a] - 2.0 * vp[a] * wp[a];
      d_out[b] = A[b * ld + b] - 2.0 * vp[b] * wp[b];
      e_out[a] = A[b * ld + a] - fma(vp[b], wp[a], wp[b] * vp[a]);
    } else if (p == 2) {
      d_out[0] = A[0];
      d_out[1] = A[ld + 1];
      e_out[0] = A[ld];
    } else {
      d_out[0] = A[0];
    }
  }
}

// Register-resident variant for p <= 128 (the Rayleigh-Ritz sizes): thread (w, l) of the 16 x 32
// layout keeps A[w + 16 r][l + 32 c] (r < 8, c < 4) in registers for the whole reduction (fixed
// ownership by absolute index), so the matrix never goes through shared memory.  One barrier per
// step: every warp redundantly rebuilds the scalars it needs -- the pending update of step j - 1
// (v_{j-1} from vs, w_{j-1} = pv_{j-1} + K v_{j-1} with K = -tau/2 pv.v) and the Householder
// vector of column j (published raw by its owners at the end of the previous step) -- then applies
// the pending update to its elements while accumulating A v_j; row sums are reduced across the
// warp (butterfly) into pvs.  Buffers alternate by step parity, so the single barrier suffices.
__device__ __forceinline__ double trd_pending_w(const double* pv, const double* v, double K, int i) {
  return fma(K, v[i], pv[i]);
}
__global__ void __launch_bounds__(kTrdThreads) trd_reg_kernel(const double* __restrict__ H, int p,
                                                              double* __restrict__ refl,
                                                              double* __restrict__ tau_out,
                                                              double* __restrict__ d_out,
                                                              double* __restrict__ e_out, long long hs, long long ws) {
  {  // problem blockIdx.y of a batch
    const long long b = blockIdx.y;
    H += b * hs;
    refl += b * ws;
    tau_out += b * ws;
    d_out += b * ws;
    e_out += b * ws;
  }
  constexpr int KR = 8, KC = 4;
  __shared__ double colb[2][256], vs[2][256], pvs[2][256];
  __shared__ double taus[2];
  __shared__ double fin[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double a[KR][KC];
#pragma unroll
  for (int r = 0; r < KR; ++r)
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      const int i = warp + 16 * r, col = lane + 32 * c;
      a[r][c] = (i < p && col < p) ? 0.5 * (H[(size_t)i * p + col] + H[(size_t)col * p + i]) : 0.0;
    }
  for (int i = tid; i < 256; i += blockDim.x) {
    vs[1][i] = 0.0;
    pvs[1][i] = 0.0;
  }
  if (tid == 0) taus[1] = 0.0;
  // raw column 0 from its owners (lane 0, slot 0)
  if (lane == 0)
#pragma unroll
    for (int r = 0; r < KR; ++r) {
      const int i = warp + 16 * r;
      if (i < p) colb[0][i] = a[r][0];
    }
  __syncthreads();
  for (int j = 0; j + 2 < p; ++j) {
    const int cur = j & 1, prv = cur ^ 1;
    const double* vp = vs[prv];
    const double* pp = pvs[prv];
    // K of the pending update (step j - 1): -tau/2 * sum_{i >= j} pv_i v_i
    double Kp;
    {
      double t = 0.0;
      for (int i = j + lane; i < p; i += 32) t = fma(pp[i], vp[i], t);
      Kp = -0.5 * taus[prv] * warp_sum_d(t);
    }
    const double vpj = vp[j], wpj = trd_pending_w(pp, vp, Kp, j);
    // column j with the pending update: x_i = colb_i - (vp_i wp_j + wp_i vp_j), i >= j
    auto xcol = [&](int i) -> double {
      return colb[cur][i] - fma(vp[i], wpj, trd_pending_w(pp, vp, Kp, i) * vpj);
    };
    double s2 = 0.0;
    for (int i = j + 2 + lane; i < p; i += 32) {
      const double x = xcol(i);
      s2 = fma(x, x, s2);
    }
    s2 = warp_sum_d(s2);
    const double alpha = xcol(j + 1);
    double tau = 0.0, beta = alpha, scal = 0.0;
    if (s2 > 0.0) {
      const double mu = sqrt(fma(alpha, alpha, s2));
      beta = alpha <= 0.0 ? mu : -mu;
      tau = (beta - alpha) * fast_rcp(beta);
      scal = fast_rcp(alpha - beta);
    }
    auto vval = [&](int i) -> double {  // v_j at absolute index i (0 for i <= j)
      return i == j + 1 ? 1.0 : (i > j + 1 && i < p ? xcol(i) * scal : 0.0);
    };
    if (warp == 0) {
      for (int i = j + 1 + lane; i < p; i += 32) {
        const double v = vval(i);
        vs[cur][i] = v;
        refl[(size_t)j * p + i] = v;
      }
      if (lane == 0) {
        d_out[j] = xcol(j);
        e_out[j] = beta;
        tau_out[j] = tau;
        taus[cur] = tau;
      }
    }
    // registers: apply the pending update and accumulate pv = tau A v_j over the trailing block
    double vpc[KC], wpc[KC], vc[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      const int col = lane + 32 * c;
      const bool act = col > j && col < p;
      vpc[c] = act ? vp[col] : 0.0;
      wpc[c] = act ? trd_pending_w(pp, vp, Kp, col) : 0.0;
      vc[c] = act ? vval(col) : 0.0;
    }
    double acc[KR];
#pragma unroll
    for (int r = 0; r < KR; ++r) {
      const int i = warp + 16 * r;
      acc[r] = 0.0;
      if (i > j && i < p) {
        const double vpi = vp[i], wpi = trd_pending_w(pp, vp, Kp, i);
#pragma unroll
        for (int c = 0; c < KC; ++c) {
          const int col = lane + 32 * c;
          if (col > j && col < p) {
            a[r][c] -= fma(vpi, wpc[c], wpi * vpc[c]);
            acc[r] = fma(a[r][c], vc[c], acc[r]);
          }
        }
      }
    }
    // butterfly reduce-scatter of the 8 row sums over the 32 lanes (7 + 2 shuffles)
    {
      int nrow = KR;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        if (nrow > 1) {
          const bool upper = (lane & o) != 0;
          const int h = nrow >> 1;
#pragma unroll
          for (int q = 0; q < KR / 2; ++q)
            if (q < h) {
              const double send = upper ? acc[q] : acc[q + h];
              const double recv = __shfl_xor_sync(0xffffffffu, send, o);
              acc[q] = (upper ? acc[q + h] : acc[q]) + recv;
            }
          nrow = h;
        } else {
          acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
        }
      }
      const int r = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
      const int i = warp + 16 * r;
      if ((lane & 3) == 0 && i > j && i < p) pvs[cur][i] = tau * acc[0];
    }
    // raw column j + 1 (pending update of step j not applied) for the next step
    {
      const int col = j + 1, cs = col >> 5;
      if (lane == (col & 31))
#pragma unroll
        for (int c = 0; c < KC; ++c)
          if (c == cs)
#pragma unroll
            for (int r = 0; r < KR; ++r) {
              const int i = warp + 16 * r;
              if (i >= col && i < p) colb[prv][i] = a[r][c];
            }
    }
    __syncthreads();
  }
  // the last 2 x 2 block, with the pending update of step p - 3
  if (p >= 3) {
    const int ia = p - 2, ib = p - 1;
#pragma unroll
    for (int r = 0; r < KR; ++r)
#pragma unroll
      for (int c = 0; c < KC; ++c) {
        const int i = warp + 16 * r, col = lane + 32 * c;
        if (i == ia && col == ia) fin[0] = a[r][c];
        if (i == ib && col == ia) fin[1] = a[r][c];
        if (i == ib && col == ib) fin[2] = a[r][c];
      }
    __syncthreads();
    if (tid == 0) {
      const int q = (p - 3) & 1;
      const double* v = vs[q];
      const double* pv = pvs[q];
      const double K = -0.5 * taus[q] * (pv[ia] * v[ia] + pv[ib] * v[ib]);
      const double wa = fma(K, v[ia], pv[ia]), wb = fma(K, v[ib], pv[ib]);
      d_out[ia] = fin[0] - 2.0 * v[ia] * wa;
      d_out[ib] = fin[2] - 2.0 * v[ib] * wb;
      e_out[ia] = fin[1] - fma(v[ib], wa, wb * v[ia]);
    }
  } else {
#pragma unroll
    for (int r = 0; r < KR; ++r)
#pragma unroll
      for (int c = 0; c < KC; ++c) {
        const int i = warp + 16 * r, col = lane + 32 * c;
        if (i < p && col <= i) {
          if (i == col) d_out[i] = a[r][c];
          else e_out[col] = a[r][c];
        }
      }
  }
}

// Warp-per-problem tridiagonalisation (p <= 128): each warp reduces one matrix held in shared memory,
// warp-synchronous (no block barrier), lanes striding over rows.  Many small problems per SM (the SCW's
// batch of k x k Grams, the eigensolver's Rayleigh-Ritz matrix) run side by side; one problem on one
// warp is still faster than a whole CTA with a barrier per phase (measured: 26 vs 150 us at p = 60).
// Outputs as trd_kernel.  blockDim.x = 32 * problems per CTA; problem b = blockIdx.x * wpb + warp.
__global__ void __launch_bounds__(256) trd_warp_kernel(const double* __restrict__ H, int p, int batch,
                                                       double* __restrict__ refl, double* __restrict__ tau_out,
                                                       double* __restrict__ d_out, double* __restrict__ e_out,
                                                       long long hs, long long wsz) {
  extern __shared__ double tw_sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int ld = p | 1;
  const long long b = (long long)blockIdx.x * wpb + warp;
  if (b >= batch) return;  // whole warp
  double* A = tw_sm + (size_t)warp * ((size_t)p * ld + 2 * 128);
  double* v = A + (size_t)p * ld;  // [128]
  double* w = v + 128;             // [128]
  H += b * hs;
  refl += b * wsz;
  tau_out += b * wsz;
  d_out += b * wsz;
  e_out += b * wsz;
  for (int e = lane; e < p * p; e += 32) {
    const int i = e / p, j = e - (e / p) * p;
    A[i * ld + j] = 0.5 * (H[(size_t)i * p + j] + H[(size_t)j * p + i]);
  }
  __syncwarp();
  for (int j = 0; j + 2 < p; ++j) {
    // Householder vector of column j (rows j+1..p-1)
    double s2 = 0.0;
    for (int i = j + 2 + lane; i < p; i += 32) {
      const double x = A[i * ld + j];
      s2 = fma(x, x, s2);
    }
    s2 = warp_sum_d(s2);
    const double alpha = A[(j + 1) * ld + j];
    double tau = 0.0, beta = alpha, scal = 0.0;
    if (s2 > 0.0) {
      const double mu = sqrt(fma(alpha, alpha, s2));
      beta = alpha <= 0.0 ? mu : -mu;
      tau = (beta - alpha) * fast_rcp(beta);
      scal = fast_rcp(alpha - beta);
    }
    for (int i = j + 1 + lane; i < p; i += 32) {
      const double vi = i == j + 1 ? 1.0 : A[i * ld + j] * scal;
      v[i] = vi;
      refl[(size_t)j * p + i] = vi;
    }
    if (lane == 0) {
      d_out[j] = A[j * ld + j];
      e_out[j] = beta;
      tau_out[j] = tau;
    }
    __syncwarp();
    if (tau == 0.0) continue;
    // pv = tau A22 v (rows by lanes), K = -tau/2 pv.v, w = pv + K v
    double kp = 0.0;
    for (int i = j + 1 + lane; i < p; i += 32) {
      const double* row = A + i * ld;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int l = j + 1;
      for (; l + 3 < p; l += 4) {
        a0 = fma(row[l], v[l], a0);
        a1 = fma(row[l + 1], v[l + 1], a1);
        a2 = fma(row[l + 2], v[l + 2], a2);
        a3 = fma(row[l + 3], v[l + 3], a3);
      }
      for (; l < p; ++l) a0 = fma(row[l], v[l], a0);
      const double pv = tau * ((a0 + a1) + (a2 + a3));
      w[i] = pv;
      kp = fma(pv, v[i], kp);
    }
    const double K = -0.5 * tau * warp_sum_d(kp);
    __syncwarp();
    for (int i = j + 1 + lane; i < p; i += 32) w[i] = fma(K, v[i], w[i]);
    __syncwarp();
    // A22 -= v w^T + w v^T  (lanes over rows)
    for (int i = j + 1 + lane; i < p; i += 32) {
      double* row = A + i * ld;
      const double vi = v[i], wi = w[i];
#pragma unroll 4
      for (int l = j + 1; l < p; ++l) row[l] -= fma(vi, w[l], wi * v[l]);
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (p >= 2) {
      d_out[p - 2] = A[(p - 2) * ld + p - 2];
      e_out[p - 2] = A[(p - 1) * ld + p - 2];
    }
    d_out[p - 1] = A[(p - 1) * ld + p - 1];
  }
}

// number of eigenvalues of T (d, e2 = e^2) strictly below sig: sign changes of the Sturm
// sequence of leading principal minors P_i = (d_i - sig) P_{i-1} - e2_{i-1} P_{i-2}, rescaled
// by powers of two (exact) to stay in range; a zero minor takes the sign opposite to its
// predecessor (LAPACK's convention of perturbing the shift).
__device__ __forceinline__ int sturm_count(const double* __restrict__ d, const double* __restrict__ e2, int p,
                                           double sig) {
  double P0 = 1.0, P1 = d[0] - sig;
  if (P1 == 0.0) P1 = -0x1p-900;
  int cnt = P1 < 0.0 ? 1 : 0;
  int i = 1;
  // 8 steps per block: the d / e2 loads of a block are independent of the chain and issue together
  for (; i + 7 < p; i += 8) {
    double dd[8], ee[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      dd[u] = d[i + u] - sig;
      ee[u] = e2[i + u - 1];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      double P2 = fma(dd[u], P1, -ee[u] * P0);
      P2 = P2 == 0.0 ? (P1 < 0.0 ? 0x1p-900 : -0x1p-900) : P2;
      cnt += (P2 < 0.0) != (P1 < 0.0);
      P0 = P1;
      P1 = P2;
    }
    // rescale both by 2^-e (exact), e the exponent of the larger: no branch on the values
    const long long eb = (__double_as_longlong(fmax(fabs(P0), fabs(P1))) >> 52) & 0x7ff;
    const double scl = __longlong_as_double((long long)max(1LL, min(2046LL, 2046LL - eb)) << 52);
    P0 *= scl;
    P1 *= scl;
  }
  for (; i < p; ++i) {
    double P2 = fma(d[i] - sig, P1, -e2[i - 1] * P0);
    P2 = P2 == 0.0 ? (P1 < 0.0 ? 0x1p-900 : -0x1p-900) : P2;
    cnt += (P2 < 0.0) != (P1 < 0.0);
    P0 = P1;
    P1 = P2;
  }
  return cnt;
}

constexpr int kTevThreads = 128;
constexpr int kTevChunk = 24;
constexpr int kOrthWindow = 6;

// eigenpair i (i-th largest) of the tridiagonal (d, e), back-transformed to the eigenvector of H:
// W[:, i] (row-major W[row * ldw + i]) and lam[i]
__global__ void __launch_bounds__(kTevThreads) tev_kernel(const double* __restrict__ d_g, const double* __restrict__ e_g,
                                                          int p, const double* __restrict__ tau,
                                                          const double* __restrict__ refl, double* __restrict__ W,
                                                          int ldw, double* __restrict__ lam, int refl_whole,
                                                          long long ws, long long wstride, long long lstride) {
  {  // problem blockIdx.y of a batch
    const long long b = blockIdx.y;
    d_g += b * ws;
    e_g += b * ws;
    tau += b * ws;
    refl += b * ws;
    W += b * wstride;
    lam += b * lstride;
  }
  __shared__ double d[256], e[256], e2[256];
  __shared__ double Dp[256], Lp[256], Dm[256], Um[256], z[256];
  __shared__ double red[kTevThreads / 32];
  __shared__ int redi[kTevThreads / 32];
  __shared__ double lo_s, hi_s;
  __shared__ int r_s;
  __shared__ __align__(8) uint64_t rbar;
  extern __shared__ __align__(16) double rch[];  // all reflector rows (whole) or kTevChunk of them
  const bool whole = refl_whole != 0;
  if (whole && threadIdx.x == 0) {
    // the reflectors (rows 0..p-3 of refl) stream into shared memory while the eigenvalue is bisected
    mbar_init(&rbar, 1);
    fence_barrier_init();
    const uint32_t bytes = (uint32_t)((((size_t)(p - 2) * p * 8) + 15) & ~(size_t)15);
    mbar_arrive_expect_tx(&rbar, bytes);
    for (uint32_t off = 0; off < bytes; off += 32768)
      bulk_g2s(reinterpret_cast<char*>(rch) + off, reinterpret_cast<const char*>(refl) + off,
               min(32768u, bytes - off), &rbar);
  }
  const int i = blockIdx.x;
  const int s = p - 1 - i;  // index of lambda_i in ascending order
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
  for (int k = tid; k < p; k += nt) {
    d[k] = d_g[k];
    const double ek = k + 1 < p ? e_g[k] : 0.0;
    e[k] = ek;
    e2[k] = ek * ek;
  }
  __syncthreads();
  // Gershgorin interval
  double glo = INFINITY, ghi = -INFINITY, emax2 = 0.0;
  for (int k = tid; k < p; k += nt) {
    const double r = fabs(e[k]) + (k > 0 ? fabs(e[k - 1]) : 0.0);
    glo = fmin(glo, d[k] - r);
    ghi = fmax(ghi, d[k] + r);
    emax2 = fmax(emax2, e2[k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    glo = fmin(glo, __shfl_xor_sync(0xffffffffu, glo, o));
    ghi = fmax(ghi, __shfl_xor_sync(0xffffffffu, ghi, o));
  }
  if (lane == 0) {
    red[warp] = glo;
    Dp[warp] = ghi;  // scratch before the factorisation
  }
  __syncthreads();
  if (tid == 0) {
    double lo = red[0], hi = Dp[0];
    for (int w = 1; w < nt / 32; ++w) {
      lo = fmin(lo, red[w]);
      hi = fmax(hi, Dp[w]);
    }
    const double nrm = fmax(fabs(lo), fabs(hi));
    const double pad = 2.0 * DBL_EPSILON * nrm * p + DBL_MIN;
    lo_s = lo - pad;
    hi_s = hi + pad;
  }
  __syncthreads();
  // multisection: nt shifts per round (~7 bits); bracket [lo, hi] keeps count(lo) <= s < count(hi)
  for (int round = 0; round < 16; ++round) {
    const double lo = lo_s, hi = hi_s;
    const double nrm = fmax(fabs(lo), fabs(hi));
    if (hi - lo <= 2.0 * DBL_EPSILON * nrm || hi - lo <= DBL_MIN) break;
    const double sig = lo + (hi - lo) * ((double)(tid + 1) / (double)(nt + 1));
    const int c = sturm_count(d, e2, p, sig);
    const unsigned ball = __ballot_sync(0xffffffffu, c >= s + 1);
    if (lane == 0) redi[warp] = ball ? warp * 32 + __ffs(ball) - 1 : nt;
    __syncthreads();
    if (tid == 0) {
      int t = nt;
      for (int w = 0; w < nt / 32; ++w) t = min(t, redi[w]);
      const double step = (hi - lo) / (double)(nt + 1);
      const double nhi = t < nt ? lo + step * (double)(t + 1) : hi;
      const double nlo = t > 0 ? lo + step * (double)t : lo;
      lo_s = fmax(lo, nlo);
      hi_s = fmin(hi, nhi);
    }
    __syncthreads();
  }
  const double lm = 0.5 * (lo_s + hi_s);
  const double pivmin = DBL_MIN * fmax(1.0, emax2) * 1e10;
  // twisted factorisation: thread 0 forward, thread 32 backward (concurrently)
  if (tid == 0) {
    double D = d[0] - lm;
    Dp[0] = D;
    for (int k = 0; k + 1 < p; ++k) {
      if (fabs(D) < pivmin) D = -pivmin;
      const double L = e[k] * fast_rcp(D);
      Lp[k] = L;
      D = (d[k + 1] - lm) - L * e[k];
      Dp[k + 1] = D;
    }
  } else if (tid == 32) {
    double D = d[p - 1] - lm;
    Dm[p - 1] = D;
    for (int k = p - 1; k > 0; --k) {
      if (fabs(D) < pivmin) D = -pivmin;
      const double U = e[k - 1] * fast_rcp(D);
      Um[k - 1] = U;
      D = (d[k - 1] - lm) - U * e[k - 1];
      Dm[k - 1] = D;
    }
  }
  __syncthreads();
  // twist index r = argmin |gamma_r|, gamma_r = D+_r + D-_r - (d_r - lambda) (lowest index on ties)
  {
    double bv = INFINITY;
    int bi = p;
    for (int k = tid; k < p; k += nt) {
      const double g = fabs(Dp[k] + Dm[k] - (d[k] - lm));
      if (g < bv) { bv = g; bi = k; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) {
      red[warp] = bv;
      redi[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double b = red[0];
      int r = redi[0];
      for (int w = 1; w < nt / 32; ++w)
        if (red[w] < b || (red[w] == b && redi[w] < r)) { b = red[w]; r = redi[w]; }
      r_s = r < p ? r : 0;
    }
    __syncthreads();
  }
  const int r = r_s;
  if (tid == 0) {
    z[r] = 1.0;
    double zz = 1.0;
    for (int k = r - 1; k >= 0; --k) {
      zz = -Lp[k] * zz;
      z[k] = zz;
    }
  } else if (tid == 32) {
    double zz = 1.0;
    for (int k = r; k + 1 < p; ++k) {
      zz = -Um[k] * zz;
      z[k + 1] = zz;
    }
  }
  __syncthreads();
  // back-transformation x = H_0 H_1 ... H_{p-3} z (warp 0), reflectors from shared memory: all of
  // them (bulk copy issued at the start) or kTevChunk rows at a time staged by the whole CTA
  auto apply = [&](int j1, int j0, const double* base) {
    for (int j = j1; j >= j0; --j) {
      const double tj = tau[j];
      if (tj == 0.0) continue;
      const double* v = base + (size_t)(j - j0) * p;
      double sacc = 0.0;
      for (int k = j + 1 + lane; k < p; k += 32) sacc = fma(v[k], z[k], sacc);
      sacc = warp_sum_d(sacc) * tj;
      for (int k = j + 1 + lane; k < p; k += 32) z[k] = fma(-sacc, v[k], z[k]);
      __syncwarp();
    }
  };
  if (whole) {
    if (warp == 0) {
      mbar_wait(&rbar, 0);
      apply(p - 3, 0, rch);
    }
  } else {
    for (int j1 = p - 3; j1 >= 0; j1 -= kTevChunk) {
      const int j0 = max(0, j1 - kTevChunk + 1);
      const int nrow = j1 - j0 + 1;
      for (int e = tid; e < nrow * p; e += nt) rch[e] = refl[(size_t)j0 * p + e];
      __syncthreads();
      if (warp == 0) apply(j1, j0, rch);
      __syncthreads();
    }
  }
  if (warp == 0) {
    double n2 = 0.0;
    for (int k = lane; k < p; k += 32) n2 = fma(z[k], z[k], n2);
    n2 = warp_sum_d(n2);
    const double inv = n2 > 0.0 ? 1.0 / sqrt(n2) : 0.0;
    for (int k = lane; k < p; k += 32) W[(size_t)k * ldw + i] = z[k] * inv;
    if (lane == 0) lam[i] = lm;
  }
}

// One CTA per problem, one warp per wanted eigenpair (looping when nw > warps): 32-lane multisection
// of the Sturm count (5 bits per round), twisted factorisation by lanes 0 (forward) and 16 (backward),
// then the back-transformation with the problem's reflectors staged once into shared memory for all
// warps (tev_kernel stages them once per eigenpair).  Outputs as tev_kernel.
__global__ void __launch_bounds__(1024) tev_cta_kernel(const double* __restrict__ d_g,
                                                       const double* __restrict__ e_g, int p, int nw,
                                                       const double* __restrict__ tau_g,
                                                       const double* __restrict__ refl,
                                                       double* __restrict__ W, int ldw, double* __restrict__ lam,
                                                       long long wsz, long long wstride, long long lstride, int vmode,
                                                       const int* __restrict__ only) {
  extern __shared__ __align__(16) double tc_sm[];
  const long long b = blockIdx.x;
  if (vmode == 2 && only[b] == 0) return;  // vectors only for the problems the caller marks
  d_g += b * wsz;
  e_g += b * wsz;
  tau_g += b * wsz;
  refl += b * wsz;
  W += b * wstride;
  lam += b * lstride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  double* R = tc_sm;                                // [(p-2) * p] reflectors
  double* d = R + (size_t)max(p - 2, 0) * p;        // [p]
  double* e2 = d + p;                               // [p]
  double* e = e2 + p;                               // [p]
  double* tau = e + p;                              // [p]
  double* scratch = tau + p;                        // per warp: Dp, Lp, Dm, Um, z [5][p]
  if (vmode != 1)
    for (int x = tid; x < max(p - 2, 0) * p; x += blockDim.x) R[x] = refl[x];
  for (int k = tid; k < p; k += blockDim.x) {
    d[k] = d_g[k];
    const double ek = k + 1 < p ? e_g[k] : 0.0;
    e[k] = ek;
    e2[k] = ek * ek;
    tau[k] = k + 2 < p ? tau_g[k] : 0.0;
  }
  __syncthreads();
  // Gershgorin interval (every warp redundantly)
  double glo = INFINITY, ghi = -INFINITY, emax2 = 0.0;
  for (int k = lane; k < p; k += 32) {
    const double r = fabs(e[k]) + (k > 0 ? fabs(e[k - 1]) : 0.0);
    glo = fmin(glo, d[k] - r);
    ghi = fmax(ghi, d[k] + r);
    emax2 = fmax(emax2, e2[k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    glo = fmin(glo, __shfl_xor_sync(0xffffffffu, glo, o));
    ghi = fmax(ghi, __shfl_xor_sync(0xffffffffu, ghi, o));
    emax2 = fmax(emax2, __shfl_xor_sync(0xffffffffu, emax2, o));
  }
  const double pad = 2.0 * DBL_EPSILON * fmax(fabs(glo), fabs(ghi)) * p + DBL_MIN;
  const double pivmin = DBL_MIN * fmax(1.0, emax2) * 1e10;
  double* Dp = scratch + (size_t)warp * 5 * p;
  double* Lp = Dp + p;
  double* Dm = Lp + p;
  double* Um = Dm + p;
  double* z = Um + p;
  for (int i = warp; i < nw; i += nwarp) {
    const int s = p - 1 - i;
    double lo = glo - pad, hi = ghi + pad;
    for (int round = 0; round < 24; ++round) {
      const double nrm = fmax(fabs(lo), fabs(hi));
      if (hi - lo <= 2.0 * DBL_EPSILON * nrm || hi - lo <= DBL_MIN) break;
      const double step = (hi - lo) / 33.0;
      const double sig = lo + step * (double)(lane + 1);
      const int c = sturm_count(d, e2, p, sig);
      const unsigned ball = __ballot_sync(0xffffffffu, c >= s + 1);
      const int t = ball ? __ffs(ball) - 1 : 32;
      const double nhi = t < 32 ? lo + step * (double)(t + 1) : hi;
      const double nlo = t > 0 ? lo + step * (double)t : lo;
      lo = fmax(lo, nlo);
      hi = fmin(hi, nhi);
    }
    const double lm = 0.5 * (lo + hi);
    if (vmode == 1) {  // eigenvalues only (SCW's error path needs sum_{i<r} sigma_i^2, not the vectors)
      if (lane == 0) lam[i] = lm;
      continue;
    }
    if (lane == 0) {
      double D = d[0] - lm;
      Dp[0] = D;
      for (int k = 0; k + 1 < p; ++k) {
        if (fabs(D) < pivmin) D = -pivmin;
        const double L = e[k] * fast_rcp(D);
        Lp[k] = L;
        D = (d[k + 1] - lm) - L * e[k];
        Dp[k + 1] = D;
      }
    } else if (lane == 16) {
      double D = d[p - 1] - lm;
      Dm[p - 1] = D;
      for (int k = p - 1; k > 0; --k) {
        if (fabs(D) < pivmin) D = -pivmin;
        const double U = e[k - 1] * fast_rcp(D);
        Um[k - 1] = U;
        D = (d[k - 1] - lm) - U * e[k - 1];
        Dm[k - 1] = D;
      }
    }
    __syncwarp();
    double bv = INFINITY;
    int bi = p;
    for (int k = lane; k < p; k += 32) {
      const double g = fabs(Dp[k] + Dm[k] - (d[k] - lm));
      if (g < bv) { bv = g; bi = k; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    const int r = bi < p ? bi : 0;
    if (lane == 0) {
      z[r] = 1.0;
      double zz = 1.0;
      for (int k = r - 1; k >= 0; --k) {
        zz = -Lp[k] * zz;
        z[k] = zz;
      }
    } else if (lane == 16) {
      double zz = 1.0;
      for (int k = r; k + 1 < p; ++k) {
        zz = -Um[k] * zz;
        z[k + 1] = zz;
      }
    }
    __syncwarp();
    for (int j = p - 3; j >= 0; --j) {
      const double tj = tau[j];
      if (tj == 0.0) continue;
      const double* v = R + (size_t)j * p;
      double sacc = 0.0;
      for (int k = j + 1 + lane; k < p; k += 32) sacc = fma(v[k], z[k], sacc);
      sacc = warp_sum_d(sacc) * tj;
      for (int k = j + 1 + lane; k < p; k += 32) z[k] = fma(-sacc, v[k], z[k]);
      __syncwarp();
    }
    double n2 = 0.0;
    for (int k = lane; k < p; k += 32) n2 = fma(z[k], z[k], n2);
    n2 = warp_sum_d(n2);
    const double inv = n2 > 0.0 ? 1.0 / sqrt(n2) : 0.0;
    for (int k = lane; k < p; k += 32) W[(size_t)k * ldw + i] = z[k] * inv;
    if (lane == 0) lam[i] = lm;
    __syncwarp();
  }
}

// flag[0] = 1 if max_{a,b < nw} |(W^T W)_ab - delta_ab| > tol  (W [p][ldw], columns 0..nw-1)
__global__ void __launch_bounds__(512) orth_kernel(const double* __restrict__ W, int p, int nw, int ldw, double tol,
                                                   int* __restrict__ flag, int use_smem, long long wstride,
                                                   const int* __restrict__ only) {
  if (only && only[blockIdx.y] == 0) return;
  W += (long long)blockIdx.y * wstride;
  extern __shared__ double osm[];
  __shared__ double red[16];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int ldc = p | 1;  // columns stored contiguously with an odd pitch
  if (use_smem)
    for (int e = tid; e < p * nw; e += nt) {
      const int row = e / nw, c = e - (e / nw) * nw;
      osm[(size_t)c * ldc + row] = W[(size_t)row * ldw + c];
    }
  __syncthreads();
  double worst = 0.0;
  // pairs (a, a + o), o < kOrthWindow: eigenvectors lose orthogonality only between close
  // eigenvalues, which are adjacent in the sorted order (any cluster has adjacent members)
  const long long npairs = (long long)nw * kOrthWindow;
  for (long long q = tid; q < npairs; q += nt) {
    const int a = (int)(q / kOrthWindow), b = a + (int)(q % kOrthWindow);
    if (b >= nw) continue;
    double s0 = 0.0, s1 = 0.0;
    if (use_smem) {
      const double* x = osm + (size_t)a * ldc;
      const double* y = osm + (size_t)b * ldc;
      int k = 0;
      for (; k + 1 < p; k += 2) {
        s0 = fma(x[k], y[k], s0);
        s1 = fma(x[k + 1], y[k + 1], s1);
      }
      if (k < p) s0 = fma(x[k], y[k], s0);
    } else {
      for (int k = 0; k < p; ++k) s0 = fma(W[(size_t)k * ldw + a], W[(size_t)k * ldw + b], s0);
    }
    worst = fmax(worst, fabs((s0 + s1) - (a == b ? 1.0 : 0.0)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
  if ((tid & 31) == 0) red[tid >> 5] = worst;
  __syncthreads();
  if (tid == 0) {
    double w = red[0];
    for (int k = 1; k < nt / 32; ++k) w = fmax(w, red[k]);
    if (!(w <= tol)) flag[0] = 1;
  }
}

// batch of problems: H [batch][p][p], W [batch][p][ldw] (stride p * ldw), lam [batch][nw]
// per-problem workspace: refl [p][p], A scratch [p][p] (p > 160), tau, d, e [p] each
long long syev_ws_doubles(int p) {
  const size_t pp = (size_t)p * p;
  return (long long)((pp * 2 + 3 * (size_t)p + 16 + 1) & ~(size_t)1);  // even: 16-B aligned
}

tsk_status syev_top_batched(Ctx* ctx, const double* H, int p, int nw, int batch, double* W, int ldw, double* lam,
                            int* flag, double orth_tol, long long lstride, double* ws, int vmode, const int* only) {
  if (p < 1 || p > 256 || nw < 1 || nw > p || ldw < nw || batch < 0) return TSK_EINVAL;
  if (lstride <= 0) lstride = nw;
  if (batch == 0) return TSK_OK;
  cudaStream_t st = ctx->stream;
  const size_t pp = (size_t)p * p;
  const long long wsz = syev_ws_doubles(p);
  if (!ws) ws = reinterpret_cast<double*>(ctx->workspace(WS_SYEV, (size_t)wsz * batch * sizeof(double)));
  if (!ws) return TSK_ENOMEM;
  double* refl = ws;
  double* gA = ws + pp;
  double* tau = ws + 2 * pp;
  double* d = tau + p;
  double* e = d + p;
  const long long wstride = (long long)p * ldw;
  if (p == 1) {
    // 1 x 1: W = 1, lam = H
    for (int b = 0; b < batch; ++b) {
      cudaMemcpyAsync(lam + b * lstride, H + b, sizeof(double), cudaMemcpyDeviceToDevice, st);
      const double one = 1.0;
      cudaMemcpyAsync(W + b * wstride, &one, sizeof(double), cudaMemcpyHostToDevice, st);
    }
    return cudaPeekAtLastError() == cudaSuccess ? TSK_OK : TSK_ECUDA;
  }
  const bool small = p <= 128 && batch >= 8 && !getenv("TSK_SYEV_CTA");
  if (!small && vmode == 2) return TSK_OK;  // the vectors came with the values (vmode 1 == 0 there)
  if (!small) only = nullptr;
  static uint64_t attr = 0;
  if (!(attr & device_bit())) {
    cudaFuncSetAttribute(trd_kernel<true, 8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaFuncSetAttribute(trd_kernel<true, 8, 4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaFuncSetAttribute(trd_kernel<true, 16, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaFuncSetAttribute(orth_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(tev_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    cudaFuncSetAttribute(trd_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaFuncSetAttribute(tev_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    attr |= device_bit();
  }
  // tau is read for j <= p - 3 only (written by the tridiagonalisation for every such j)
  const size_t asmem = (size_t)p * (p + 1) * sizeof(double);
  const dim3 g1(1, batch);
  const long long hs = (long long)pp;
  // many problems: a CTA per tridiagonalisation (p <= 88; a warp per problem above) and a CTA per
  // problem's eigenpairs keep every SM busy with independent latency chains (SCW: 250 Grams per launch);
  // a single problem (the eigensolver's Rayleigh-Ritz matrix) takes the per-eigenpair CTAs of tev_kernel
  if (small) {
    // warp-per-problem geometry: as many problems per CTA as fit 200 KB of shared memory (<= 8)
    const size_t per = ((size_t)p * (p | 1) + 2 * 128) * sizeof(double);
    // spread the problems over the SMs first (each warp is one latency chain), then stack them
    const int want = (batch + ctx->num_sms - 1) / ctx->num_sms;
    const int wpb = (int)std::max<size_t>(1, std::min<size_t>(std::min(8, want), (200 * 1024) / per));
    const int nblk = (batch + wpb - 1) / wpb;
    if (vmode != 2) {
      // a CTA per tridiagonalisation up to p = 88 (row-parallel pass; C4 SCW, p = 60, 250 problems: 118 us
      // against 232 us for a warp per problem -- 250 one-warp latency chains leave the SMs mostly idle)
      static const bool warp_only = getenv("TSK_SYEV_TRD_WARP") != nullptr;
      if (!warp_only && p <= 88)
        trd_kernel<true, 8, 4, true><<<g1, kTrdThreads, asmem, st>>>(H, p, refl, tau, d, e, nullptr, hs, wsz);
      else
        trd_warp_kernel<<<nblk, 32 * wpb, per * wpb, st>>>(H, p, batch, refl, tau, d, e, hs, wsz);
      ctx->count_launch();
    }
    const size_t fixed = ((size_t)std::max(p - 2, 0) * p + 4 * (size_t)p) * sizeof(double);
    const size_t per_warp = (size_t)5 * p * sizeof(double);
    const int fit = (int)(((size_t)200 * 1024 - fixed) / per_warp);
    const int warps = std::max(1, std::min(std::min(32, nw), fit));
    const size_t tsm = fixed + (size_t)warps * per_warp;
    tev_cta_kernel<<<batch, 32 * warps, tsm, st>>>(d, e, p, nw, tau, refl, W, ldw, lam, wsz, p * (long long)ldw,
                                                   lstride, vmode, only);
    ctx->count_launch();
    if (vmode == 1) return launch_status("syev_top (values)");
  } else if (p <= 128 && getenv("TSK_TRD_REG"))
    trd_reg_kernel<<<g1, kTrdThreads, 0, st>>>(H, p, refl, tau, d, e, hs, wsz);
  else if (p <= 129) {
    // the row-parallel pass wins below ~p = 90 (p = 48: 1070 vs 1589 cycles per step, 76: 1394 vs 1950) and
    // loses above (96: 2614 vs 2249, 128: 4264 vs 2848; its 4-thread rows serialise (p - j) / 4 columns)
    if (p > 88 || getenv("TSK_TRD_TILE"))
      trd_kernel<true, 8, 4><<<g1, kTrdThreads, asmem, st>>>(H, p, refl, tau, d, e, nullptr, hs, wsz);
    else
      trd_kernel<true, 8, 4, true><<<g1, kTrdThreads, asmem, st>>>(H, p, refl, tau, d, e, nullptr, hs, wsz);
  } else if (p <= kTrdSmemMaxP)
    trd_kernel<true, 16, 8><<<g1, kTrdThreads, asmem, st>>>(H, p, refl, tau, d, e, nullptr, hs, wsz);
  else
    trd_kernel<false, 16, 8><<<g1, kTrdThreads, 0, st>>>(H, p, refl, tau, d, e, gA, hs, wsz);
  if (!small) {
    const size_t rbytes = (((size_t)(p - 2) * p * 8) + 15) & ~(size_t)15;
    const int whole = rbytes <= 140 * 1024;
    tev_kernel<<<dim3(nw, batch), kTevThreads, whole ? rbytes : (size_t)kTevChunk * p * sizeof(double), st>>>(
        d, e, p, tau, refl, W, ldw, lam, whole, wsz, wstride, lstride);
    ctx->count_launch(2);
  }
  if (flag) {
    const size_t wsm = (size_t)(p | 1) * nw * sizeof(double);
    const int use_smem = wsm <= 220 * 1024;
    orth_kernel<<<dim3(1, batch), 512, use_smem ? wsm : 0, st>>>(W, p, nw, ldw, orth_tol, flag, use_smem, wstride,
                                                                  only);
    ctx->count_launch();
  }
  return launch_status("syev_top");
}

tsk_status syev_top(Ctx* ctx, const double* H, int p, int nw, double* W, int ldw, double* lam, int* flag,
                    double orth_tol) {
  return syev_top_batched(ctx, H, p, nw, 1, W, ldw, lam, flag, orth_tol, nw);
}

}  // namespace tsk
#ifdef TSK_TRD_PROF
extern "C" int tsk_trd_prof_read(long long* out) {
  return cudaMemcpyFromSymbol(out, tsk::trd_prof, sizeof(long long) * 4) == cudaSuccess ? 0 : -4;
}
#endif
