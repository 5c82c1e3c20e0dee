// Small fp64 / layout kernels of the eigensolver (defined in eig.cu), shared with the matrix-free
// sketch (matrix_free.cu).  Row-major [m][p] blocks throughout.
#pragma once
#include "tsk_internal.h"

namespace tsk {
// Y (=|+=) scale * uniform(-1, 1) from a counter-based hash of (idx, salt)
__global__ void hash_fill_kernel(double* Y, int m, int p, uint64_t salt, double scale, int add);
// Q [m][p] fp64 -> Qt [p][ms] fp32 (transposed), Q <- fp64(fp32(Q))
__global__ void q_to_f32t_kernel(double* __restrict__ Q, int m, int p, int ms, float* __restrict__ Qt);
// S[c][:] = sign-normalised, normalised column c of V [m][ldv], c < gridDim.x (reading c5)
__global__ void write_sketch_kernel(const double* __restrict__ V, int m, int ldv, float* __restrict__ S);
// Yn = alpha (Z - c Yc) - beta Yp  (n elements)
__global__ void cheb_step_kernel(const double* __restrict__ Z, const double* __restrict__ Yc,
                                 const double* __restrict__ Yp, long long n, double c, double alpha, double beta,
                                 double* __restrict__ Yn);
// dst[:, d0:d0+nc] = src[:, c0:c0+nc]
__global__ void copy_cols_kernel(const double* __restrict__ src, int lds, int c0, double* __restrict__ dst, int ldd,
                                 int d0, int m, int nc);
// Q = orthonormal basis of range(Y) by fp64 CholQR twice (Y, Q1, Q: [m][p]); flags[0..1] = first
// failed pivot + 1 of each pass (device, sticky; 0 = success)
tsk_status cholqr2(Ctx* ctx, const double* Y, double* Q1, double* Q, int m, int p, double* C, double* R,
                   int* flags);
}  // namespace tsk
