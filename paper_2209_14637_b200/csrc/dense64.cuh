// fp64 helper kernels (dense64.cu)
#pragma once
#include "tsk_internal.h"

namespace tsk {
// C[b] = X[b]^T Y[b]  (X: m x p, Y: m x q, row-major with leading dims; batch strides sx, sy, sc).
// sym: C = (C + C^T)/2 (p == q).  Split over m with fixed-order reduction.
tsk_status gemm_tn_f64(Ctx* ctx, const double* X, long long ldx, long long sx, const double* Y, long long ldy,
                       long long sy, int m, int p, int q, int batch, double* C, long long ldc, long long sc, int sym,
                       int ws_id);
// Y[b] = (Z[b] W[b]) diag(colscale[b])   (Z: m x p, W: p x q; sw = 0 shares one W; colscale may be null)
tsk_status gemm_nn_f64(Ctx* ctx, const double* Z, long long ldz, long long sz, const double* W, long long ldw,
                       long long sw, int m, int p, int q, int batch, const double* colscale, double* Y, long long ldy,
                       long long sy);
// Cholesky C[b] = L L^T (L lower, row-major); on failure flag[b] = first failed pivot + 1 (sticky)
tsk_status chol(Ctx* ctx, const double* C, int p, int batch, double rel_tol, double* L, int* flag, int ws_id);
// Q = Y L^{-T} (Y, Q: m x p row-major; L: p x p lower), i.e. Q R = Y with R = L^T; p <= ~150
tsk_status trsm_rlt(Ctx* ctx, const double* Y, const double* L, int m, int p, double* Q);
// Cholesky C = L L^T and Rinv = L^{-T} (upper) in one CTA (p <= 116); flag as chol
tsk_status chol_inv2(Ctx* ctx, const double* C, int p, int batch, double rel_tol, double* Rinv, int* flag);
}  // namespace tsk
