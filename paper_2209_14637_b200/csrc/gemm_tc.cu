// Split-TF32 ("3xTF32") NT GEMM on tcgen05 tensor cores, the Gram hot loop of the
// tensor-based sketch (G = A_(1) A_(1)^T = sum_d A_d A_d^T).
//
//   C[M x N] = sum_{z < D} X_z[M x n] * Y_z[N x n]^T          (fp64 result)
//
// X and Y are fp32, K-major (row-major with the contracted index contiguous) and are
// addressed through 3-D TMA tensor maps [D][rows][n]; the contraction runs over the pair
// (z, j) -- for the mode-1 Gram z = d (the stream index) and X = Y = the training stack,
// so A_(1) is never materialised (its column order does not matter for G; reading c3).
//
// Precision: each 32-column K-chunk x is split into
//   H = trunc_tf32(x) (the tensor core's own fp32->tf32 conversion),  L = x - H (exact)
// and the tile accumulates H_X H_Y^T + H_X L_Y^T + L_X H_Y^T (L L^T dropped, ~2^-21 rel).
// TMEM fp32 accumulation (truncating) runs over bounded chains of `chain` chunks, is folded
// into fp32 registers (round-to-nearest), and every `fold` chains into an fp64 partial.
//
// Work decomposition: the output is cut into 128x128 tiles (lower-triangle tiles only when
// `sym`), K into S equal splits; unit u = s*T + t is handled by CTA (u mod grid).  A round
// of `grid` consecutive units touches at most a few K-splits, so the CTAs of a round read the
// same K window and the operands are served from L2 (HBM traffic ~1x the input).
// A finalize kernel sums the S partials of each tile in fixed order (deterministic) and
// mirrors the lower triangle for `sym`.
#include <cudaTypedefs.h>

#include <algorithm>
#include <vector>
#include <cmath>

#include "ptx.cuh"
#include "tsk_internal.h"

namespace tsk {

constexpr int kBM = 128;            // tile rows (UMMA M)
constexpr int kBN = 128;            // tile cols (UMMA N)
constexpr int kBK = 32;             // fp32 elements per K-chunk = 128 B = one SW128 row
constexpr int kRawStages = 5;       // TMA ring: raw fp32 tiles of X and Y (the raw tile IS the hi part)
constexpr int kLoStages = 2;        // transform ring: lo parts L = x - trunc_tf32(x)
constexpr int kTileBytes = kBM * kBK * 4;  // 16 KB
constexpr int kThreads = 512;
constexpr int kTmemCols = 512;      // 2 buffers x {H H^T, cross} x 128 fp32 columns
constexpr int kSmemBytes = (kRawStages + kLoStages) * 2 * kTileBytes + 1024 /*align*/ + 256 /*barriers*/;

struct GemmArgs {
  int T;         // tiles
  int nb;        // column blocks (general layout)
  int sym;       // lower-triangle tiles of X X^T
  int cps;       // K-chunks per slice = ceil(n / 32)
  int S;         // K splits
  long long Kc;  // chunks per tile = D * cps
  int U;         // units = S * T
  int chain;     // chunks per TMEM accumulation chain
  int fold;      // chains per fp64 fold
  int products;  // 3 = split-TF32 (production); 1 = H*H only (precision probe)
  int raw;       // diagnostics: 1 = skip the split transform (the lo buffers are not written)
  int lag;       // drift throttle: max chunks a unit may run ahead of its K-split peers (0 = off)
  double* part;  // [U][128][128] fp64 partials
  unsigned* progress;  // [U] chunks issued per unit (drift throttle)
  int batch;     // 0: the D slices are contracted; 1: D independent problems (slice z = problem b)
  int T0;        // tiles per problem (batched)
  int bn;        // MMA N: 128, or 64 for narrow outputs (TS kernel)
  int Mv, Nv;    // valid output extents (direct output)
  float* dout;   // direct fp32 output, transposed: dout[b * dstride + col * ldd + row] (requires S == 1)
  int xt;        // X operand stored transposed ([z][K][M], M contiguous): the transform reads tile columns
  int ybc;       // Y broadcast: every slice z uses Y slice 0
  int drow;      // direct output row-major: dout[b * dstride + row * ldd + col]
  const float* resA;  // residual epilogue: tile partials of sum (resA_b[row][col] - D[row][col])^2 (fp64)
  long long res_stride;
  int res_ld;
  double* res_part;   // [units][8] (one partial per epilogue warp, fixed order)
  long long dstride;
  int ldd;
  const int* only;   // batch mode: problems b with only[b] == 0 are skipped by every role (null: all)
  const int* only_any;  // optional device count of problems with only[b] != 0: 0 => the whole grid exits at once
  int spin;  // TS kernel mbarrier waits without suspend hint: bit 0 TMA producer, 1 transform, 2 MMA issuer
  unsigned long long* trace;  // diagnostics (TSK_TS_TRACE): per-chunk globaltimer stamps of CTA 0, [8][trace_n]
  int trace_n;
  double* sq_part;   // TS kernel: [U][8] fp64 sums of the squared X elements of each unit (transform warps)
};

// batch mode with a problem mask: unit u belongs to a skipped problem (same test in every role, so the
// ring / accumulator phases stay in step).  The mask is copied to shared memory in the prologue when the
// batch has <= kOnlyMax problems (a CTA walks ~U / 148 units; one dependent global load per unit cost
// ~65 us on a launch whose units were all skipped).
constexpr int kOnlyMax = 256;  // 1 KB: the kYT variant has 225 KB of dynamic shared memory
__device__ __forceinline__ void ts_wait(uint64_t* bar, uint32_t parity, bool spin) {
  if (spin) mbar_wait_spin(bar, parity);
  else mbar_wait(bar, parity);
}
__device__ __forceinline__ void ts_stamp(const GemmArgs& a, int slot, long long i) {
  if (a.trace && blockIdx.x == 0 && i < a.trace_n) a.trace[(size_t)slot * a.trace_n + i] = globaltimer_ns();
}
__device__ __forceinline__ bool unit_skipped(const GemmArgs& a, const int* s_only, int u) {
  if (a.only == nullptr) return false;
  const int b = (u % a.T) / a.T0;
  return (s_only ? s_only[b] : a.only[b]) == 0;
}

__device__ __forceinline__ void tile_coords(const GemmArgs& a, int t, int& bi, int& bj) {
  if (a.batch) t %= a.T0;
  if (a.sym) {
    int i = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
    while ((i + 1) * (i + 2) / 2 <= t) ++i;
    while (i * (i + 1) / 2 > t) --i;
    bi = i;
    bj = t - i * (i + 1) / 2;
  } else {
    bi = t / a.nb;
    bj = t % a.nb;
  }
}

__device__ __forceinline__ void unit_range(const GemmArgs& a, int u, int& t, long long& q0, long long& q1) {
  t = u % a.T;
  int s = u / a.T;
  // batched: tile t belongs to problem b = t / T0, whose K range is the chunks of slice b only
  const long long base = a.batch ? (long long)(t / a.T0) * a.cps : 0;
  if (a.S == 1) {  // batched problems: no 64-bit division per unit
    q0 = base;
    q1 = base + a.Kc;
    return;
  }
  q0 = base + (long long)s * a.Kc / a.S;
  q1 = base + (long long)(s + 1) * a.Kc / a.S;
}

// Warp roles (16 warps): 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 3 idle,
// 4-7 split transform, 8-15 epilogue.
//
// The tensor core reads fp32 operands of kind::tf32 by TRUNCATING them to tf32 (measured on
// B200, scripts/gram_probe.py), so the raw TMA tile is used directly as the hi part
// H = trunc_tf32(x) and only L = x - H (exact in fp32) is produced in shared memory.
// Products go to two TMEM accumulators per buffer: ACC_HH += H_X H_Y^T and
// ACC_X += H_X L_Y^T + L_X H_Y^T (2^-10-scaled terms: their truncating accumulation error is
// negligible), which divides the dominant accumulation error by three at equal chain length.
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapY,
                       const GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* raw_base = smem;                                        // [kRawStages][X|Y]
  uint8_t* lo_base = smem + kRawStages * 2 * kTileBytes;           // [kLoStages][XL|YL]
  uint64_t* bars = reinterpret_cast<uint64_t*>(lo_base + kLoStages * 2 * kTileBytes);
  uint64_t* rfull = bars;                        // TMA -> transform / MMA
  uint64_t* rempty = rfull + kRawStages;         // MMA -> TMA
  uint64_t* lfull = rempty + kRawStages;         // transform -> MMA
  uint64_t* lempty = lfull + kLoStages;          // MMA -> transform
  uint64_t* accf = lempty + kLoStages;           // MMA -> epilogue (2 buffers)
  uint64_t* acce = accf + 2;                     // epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapX);
    tma_prefetch_desc(&mapY);
    for (int i = 0; i < kRawStages; ++i) {
      mbar_init(&rfull[i], 1);
      mbar_init(&rempty[i], 1);
    }
    for (int i = 0; i < kLoStages; ++i) {
      mbar_init(&lfull[i], 4);
      mbar_init(&lempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&accf[i], 1);
      mbar_init(&acce[i], 8);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto raw_ptr = [&](int st, int which) { return raw_base + (st * 2 + which) * kTileBytes; };
  auto lo_ptr = [&](int st, int which) { return lo_base + (st * 2 + which) * kTileBytes; };

  if (warp == 0) {
    // ===================== TMA producer (lane 0 issues; the warp runs the drift throttle) =====================
    // Units of the same K-split s in the same round read the same K window; if they drift apart
    // the window leaves L2 and every tile re-reads its rows from HBM (measured 6x over-read).
    // Every 32 chunks each unit publishes its progress and waits while it is more than `lag`
    // chunks ahead of the slowest such peer (the slowest never waits: no deadlock).
    int st = 0;
    uint32_t ph = 0;
    for (int u = blockIdx.x; u < a.U; u += gridDim.x) {
      int t, bi, bj;
      long long q0, q1;
      unit_range(a, u, t, q0, q1);
      tile_coords(a, t, bi, bj);
      const bool diag = a.sym && bi == bj;
      const int s_split = u / a.T;
      const int round = u / gridDim.x;
      for (long long q = q0; q < q1; ++q) {
        if (lane == 0) {
          mbar_wait(&rempty[st], ph ^ 1);
          mbar_arrive_expect_tx(&rfull[st], diag ? kTileBytes : 2 * kTileBytes);
          const int z = (int)(q / a.cps);
          const int kc = (int)(q % a.cps) * kBK;
          tma_load_3d(raw_ptr(st, 0), &mapX, &rfull[st], kc, bi * kBM, z);
          if (!diag) tma_load_3d(raw_ptr(st, 1), &mapY, &rfull[st], kc, bj * kBN, z);
        }
        if (++st == kRawStages) { st = 0; ph ^= 1; }
        const unsigned done = (unsigned)(q - q0 + 1);
        if (a.lag > 0 && ((done & 31u) == 0 || q + 1 == q1)) {
          if (lane == 0) st_volatile_u32(&a.progress[u], q + 1 == q1 ? 0xFFFFFFFFu : done);
          if (q + 1 < q1) {
            while (true) {
              unsigned mn = 0xFFFFFFFFu;
              for (int tp = lane; tp < a.T; tp += 32) {
                const int up = s_split * a.T + tp;
                if (up != u && up / (int)gridDim.x == round) mn = min(mn, ld_volatile_u32(&a.progress[up]));
              }
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
              if (mn == 0xFFFFFFFFu || done <= mn + (unsigned)a.lag) break;
              __nanosleep(1000);
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread) =====================
    if (elect_one()) {
      const uint32_t idesc = idesc_tf32(kBM, kBN);
      int rs = 0, ls = 0;
      uint32_t rph = 0, lph = 0;
      int ab = 0;
      uint32_t aph = 0;
      for (int u = blockIdx.x; u < a.U; u += gridDim.x) {
        int t, bi, bj;
        long long q0, q1;
        unit_range(a, u, t, q0, q1);
        tile_coords(a, t, bi, bj);
        const bool diag = a.sym && bi == bj;
        int cpos = 0;
        for (long long q = q0; q < q1; ++q) {
          if (cpos == 0) {
            mbar_wait(&acce[ab], aph ^ 1);
            tc_fence_after();
          }
          if (a.products == 3) mbar_wait(&lfull[ls], lph);  // implies the raw stage landed
          else mbar_wait(&rfull[rs], rph);
          tc_fence_after();
          const uint32_t d_hh = tmem_base + (uint32_t)(ab * 2 * kBN);
          const uint32_t d_x = d_hh + kBN;
          const uint64_t xh = sw128_kmajor_desc(smem_u32(raw_ptr(rs, 0)));
          const uint64_t yh = diag ? xh : sw128_kmajor_desc(smem_u32(raw_ptr(rs, 1)));
          const uint64_t xl = sw128_kmajor_desc(smem_u32(lo_ptr(ls, 0)));
          const uint64_t yl = diag ? xl : sw128_kmajor_desc(smem_u32(lo_ptr(ls, 1)));
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk) {
            const uint64_t adv = (uint64_t)(kk * 32 >> 4);  // +32 B per K=8 step inside the swizzle atom
            const uint32_t acc = (cpos > 0 || kk > 0) ? 1u : 0u;
            mma_tf32_ss(d_hh, xh + adv, yh + adv, idesc, acc);
            if (a.products == 3) {
              mma_tf32_ss(d_x, xh + adv, yl + adv, idesc, acc);
              mma_tf32_ss(d_x, xl + adv, yh + adv, idesc, 1u);
            }
          }
          mma_commit(&rempty[rs]);
          if (++rs == kRawStages) { rs = 0; rph ^= 1; }
          if (a.products == 3) {
            mma_commit(&lempty[ls]);
            if (++ls == kLoStages) { ls = 0; lph ^= 1; }
          }
          if (++cpos == a.chain || q + 1 == q1) {
            mma_commit(&accf[ab]);
            cpos = 0;
            if (++ab == 2) { ab = 0; aph ^= 1; }
          }
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ===================== split transform: L = x - trunc_tf32(x) =====================
    if (a.products == 3) {
      const int tt = threadIdx.x - 128;  // 0..127
      int rs = 0, ls = 0;
      uint32_t rph = 0, lph = 0;
      for (int u = blockIdx.x; u < a.U; u += gridDim.x) {
        int t, bi, bj;
        long long q0, q1;
        unit_range(a, u, t, q0, q1);
        tile_coords(a, t, bi, bj);
        const bool diag = a.sym && bi == bj;
        for (long long q = q0; q < q1; ++q) {
          mbar_wait(&rfull[rs], rph);
          mbar_wait(&lempty[ls], lph ^ 1);
          const int ntiles = a.raw ? 0 : (diag ? 1 : 2);
          for (int w = 0; w < ntiles; ++w) {
            const float4* xp = reinterpret_cast<const float4*>(raw_ptr(rs, w));
            float4* lp = reinterpret_cast<float4*>(lo_ptr(ls, w));
            float4 v[kTileBytes / 16 / 128];
#pragma unroll
            for (int i = 0; i < kTileBytes / 16 / 128; ++i) v[i] = xp[i * 128 + tt];
#pragma unroll
            for (int i = 0; i < kTileBytes / 16 / 128; ++i) {
              float4 l;
              l.x = v[i].x - __uint_as_float(__float_as_uint(v[i].x) & 0xFFFFE000u);
              l.y = v[i].y - __uint_as_float(__float_as_uint(v[i].y) & 0xFFFFE000u);
              l.z = v[i].z - __uint_as_float(__float_as_uint(v[i].z) & 0xFFFFE000u);
              l.w = v[i].w - __uint_as_float(__float_as_uint(v[i].w) & 0xFFFFE000u);
              lp[i * 128 + tt] = l;
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&lfull[ls]);
          if (++rs == kRawStages) { rs = 0; rph ^= 1; }
          if (++ls == kLoStages) { ls = 0; lph ^= 1; }
        }
      }
    }
  } else if (warp >= 8) {
    // ===================== epilogue: TMEM chains -> fp32 registers -> fp64 partials =====================
    const int e = warp - 8;
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int col0 = (e >> 2) * 64;
    const int row = quad * 32 + lane;
    int ab = 0;
    uint32_t aph = 0;
    for (int u = blockIdx.x; u < a.U; u += gridDim.x) {
      int t;
      long long q0, q1;
      unit_range(a, u, t, q0, q1);
      const long long nchunks = q1 - q0;
      const long long nchains = (nchunks + a.chain - 1) / a.chain;
      float sum[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) sum[i] = 0.f;
      // staggered folds: epilogue warp e folds (fp32 -> fp64 reductions at L2) at chains offset by
      // e * fold / 8, so no single accumulator drain carries all the L2 reductions of a fold
      int cin = (e * a.fold) / 8;
      bool first_fold = true;
      double* prow = a.part + (size_t)u * (kBM * kBN) + (size_t)row * kBN + col0;
      for (long long c = 0; c < nchains; ++c) {
        mbar_wait(&accf[ab], aph);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(ab * 2 * kBN + col0);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + h * 32, r);
          tmem_ld_wait();
          if (a.products == 3) {
            uint32_t x[32];
            tmem_ld_32x32b_x32(taddr + kBN + h * 32, x);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) sum[h * 32 + i] += __uint_as_float(r[i]) + __uint_as_float(x[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) sum[h * 32 + i] += __uint_as_float(r[i]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acce[ab]);
        if (++ab == 2) { ab = 0; aph ^= 1; }
        if (++cin == a.fold || c + 1 == nchains) {
          // partial-sum lines are re-read every fold: keep them in L2 against the streaming operands
          const uint64_t pol = l2_policy_evict_last();
          if (first_fold) {
#pragma unroll
            for (int i = 0; i < 64; i += 2)
              st_f64x2_hint(reinterpret_cast<double2*>(prow + i), make_double2((double)sum[i], (double)sum[i + 1]), pol);
          } else {
#pragma unroll
            for (int i = 0; i < 64; ++i) red_add_f64_hint(prow + i, (double)sum[i], pol);
          }
#pragma unroll
          for (int i = 0; i < 64; ++i) sum[i] = 0.f;
          first_fold = false;
          cin = 0;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// ---------------------------------------------------------------------------------------------
// TS variant (production path): the A operand (hi and lo parts of the X rows) is written by the
// transform warps straight into tensor memory with tcgen05.st, so the MMAs read only their B
// operand from shared memory.  Per 32-column chunk of an off-diagonal 128x128 tile this moves
// 128 KB through shared memory (TMA 32 + transform 48 + MMA-B 48) instead of 192 KB.
// TMEM: two 128-column accumulators (double buffer; H H^T and the cross terms share one) + three
// 64-column A stages [H_X | L_X].  Shared memory: 5 raw TMA stages [X|Y] + 3 lo stages [L_Y].
// transform -> MMA ring depth (TMEM A stages [H_X | L_X] and smem lo stages): 4 (TMEM 2 x 128 + 4 x 64 = 512
// columns) unless the lo stages are [H_Y | L_Y] (kYT: 32 KB each, 3 fit shared memory)
template <bool kN64, bool kYT>
constexpr int ts_lo_stages() { return kYT ? 3 : 4; }
// Split rounding (TS kernel): hi(x) = x rounded to nearest tf32 for the X operand (written to TMEM), and
// lo = x - hi, which then has a random sign: the tensor core truncates its operands, so truncated hi
// parts leave lo with the sign of x and the dropped lo x lo' and the truncation of lo bias every product
// toward zero (~3e-7 relative on SCW's AV, which the Pythagorean error reads at first order, reading
// c17).  Y keeps the hardware-truncated raw tile as hi; its lo part is rounded to nearest.
constexpr bool kYLoRn = true;
// Ring geometry: [X | Y] raw stages and [L_Y] (or, kYT, [H_Y | L_Y]) lo stages.  With N = 64 the Y tiles
// are half size, so the raw ring packs 7 stages of 24 KB instead of 5 of 32 KB: the SCW products (SA, AV)
// stream A from HBM and are latency-bound on the bytes in flight per SM.
template <bool kN64, bool kYT>
constexpr int ts_raw_stages() { return kYT ? kRawStages - 1 : (kN64 ? 7 : kRawStages); }
template <bool kN64, bool kYT>
constexpr int ts_raw_stage_bytes() { return kYT ? 2 * kTileBytes : kTileBytes + (kN64 ? kTileBytes / 2 : kTileBytes); }
template <bool kN64, bool kYT>
constexpr int ts_lo_stage_bytes() { return kYT ? 2 * kTileBytes : (kN64 ? kTileBytes / 2 : kTileBytes); }
template <bool kN64, bool kYT>
constexpr int ts_smem_bytes() {
  return ts_raw_stages<kN64, kYT>() * ts_raw_stage_bytes<kN64, kYT>() +
         ts_lo_stages<kN64, kYT>() * ts_lo_stage_bytes<kN64, kYT>() +
         1024 + 256;
}
constexpr int kTsSmemBytes = ts_smem_bytes<false, false>();
constexpr uint32_t kTsAccCols = 128;
constexpr uint32_t kTsAStageCols = 64;

// kYT: the Y operand is stored transposed ([z][K][N], N contiguous); the transform then writes
// both H_Y and L_Y in the swizzled K-major layout (the lo ring holds both, the raw ring shrinks).
template <bool kN64, bool kYT>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tf32x3_ts_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapY,
                          const GemmArgs a) {
  // nothing to compute (e.g. no matrix marked for SCW's dense residual): leave before any setup
  if (a.only_any && *a.only_any == 0) return;
  constexpr int RS = ts_raw_stages<kN64, kYT>();          // raw ring depth
  constexpr int RSB = ts_raw_stage_bytes<kN64, kYT>();    // raw stage: [X | Y] (Y = bn x 32 fp32)
  constexpr int LB = ts_lo_stage_bytes<kN64, kYT>();      // lo stage: [L_Y] or [H_Y | L_Y]
  constexpr int kTsLoStages = ts_lo_stages<kN64, kYT>();
  // N = 64 (SCW's SA / AV products): the split transform is the critical path (one warp per SM
  // sub-partition, latency-bound), so warps 12-15 join it -- two warps per TMEM lane quadrant, each
  // converting 16 of the chunk's 32 K-columns -- and the 64-column epilogue runs on warps 8-11
  constexpr bool kSplitT = kN64 && !kYT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* raw_base = smem;                                 // [RS][X|Y]
  uint8_t* lo_base = smem + RS * RSB;                       // [kTsLoStages][LB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(lo_base + kTsLoStages * LB);
  uint64_t* rfull = bars;
  uint64_t* rempty = rfull + RS;
  uint64_t* lfull = rempty + RS;
  uint64_t* lempty = lfull + kTsLoStages;
  uint64_t* accf = lempty + kTsLoStages;
  uint64_t* acce = accf + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapX);
    tma_prefetch_desc(&mapY);
    for (int i = 0; i < RS; ++i) {
      mbar_init(&rfull[i], 2);  // X box + Y box (or the diagonal tile's plain arrive)
      mbar_init(&rempty[i], 1);
    }
    for (int i = 0; i < kTsLoStages; ++i) {
      mbar_init(&lfull[i], 4);  // the 4 transform warps of the group that converts the chunk
      mbar_init(&lempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&accf[i], 1);
      mbar_init(&acce[i], kSplitT ? 4 : 8);
    }
    fence_barrier_init();
  }
  __shared__ int s_only_buf[kOnlyMax];
  const int* s_only = nullptr;
  if (a.only && a.T / a.T0 <= kOnlyMax) {
    for (int i = threadIdx.x; i < a.T / a.T0; i += blockDim.x) s_only_buf[i] = a.only[i];
    s_only = s_only_buf;
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto raw_ptr = [&](int st, int which) { return raw_base + st * RSB + which * kTileBytes; };
  auto lo_ptr = [&](int st) { return lo_base + st * LB; };

  if (warp == 0) {
    // ===================== TMA producer + drift throttle =====================
    // Lanes 0-3 issue the X boxes and lanes 4-7 the Y boxes; lane j (mod 4) owns the chunks whose
    // CTA-wide index is j mod 4 and runs decoupled from the other lanes, each chunk issued as soon
    // as its stage is free (a thread's TMA boxes complete one after another, scripts/tma_bench.cu,
    // so one lane cannot keep the ring full; and lanes stepping in lock-step groups of 4 left at
    // most one free stage of lead: SA/AV at C4 ran one chunk per 0.69 us against 0.21 us of MMA).
    if (lane < 8) {
      const int j = lane & 3;
      const bool isx = lane < 4;
      const uint32_t ybytes = (uint32_t)(a.bn * kBK * 4);
      long long idx = 0;  // CTA-wide chunk index (stage = idx % RS, use = idx / RS)
      for (int u = blockIdx.x; u < a.U; u += gridDim.x) {
        if (unit_skipped(a, s_only, u)) continue;
        int t, bi, bj;
        long long q0, q1;
        unit_range(a, u, t, q0, q1);
        tile_coords(a, t, bi, bj);
        const bool diag = a.sym && bi == bj;
        const int s_split = u / a.T;
        const int round = u / gridDim.x;
        // first chunk of this unit owned by this lane
        long long q = q0 + ((((long long)j - idx) % 4) + 4) % 4;
        long long ci = idx + (q - q0);
        for (; q < q1; q += 4, ci += 4) {
          const int sl = (int)(ci % RS);
          const uint32_t use = (uint32_t)((ci / RS) & 1);
          ts_wait(&rempty[sl], use ^ 1, a.spin & 1);
          const int z = (int)(q / a.cps);
          const int kc = (int)(q % a.cps) * kBK;
          if (isx) {
            ts_stamp(a, 0, ci);
            mbar_arrive_expect_tx(&rfull[sl], (uint32_t)kTileBytes);
            if (a.xt) tma_load_3d(raw_ptr(sl, 0), &mapX, &rfull[sl], bi * kBM, kc, z);  // box {128 M, 32 K}
            else tma_load_3d(raw_ptr(sl, 0), &mapX, &rfull[sl], kc, bi * kBM, z);
          } else if (diag) {
            mbar_arrive(&rfull[sl]);  // the diagonal tile's Y is its X
          } else {
            mbar_arrive_expect_tx(&rfull[sl], ybytes);
            if (kYT) tma_load_3d(raw_ptr(sl, 1), &mapY, &rfull[sl], bj * a.bn, kc, a.ybc ? 0 : z);  // {bn N, 32 K}
            else tma_load_3d(raw_ptr(sl, 1), &mapY, &rfull[sl], kc, bj * a.bn, a.ybc ? 0 : z);   // {32 K, bn N}
          }
          // drift throttle (lane 0 alone; the other lanes are bounded by the ring): units of the
          // same K window in the same round read the same operands through L2
          const unsigned done = (unsigned)(q - q0 + 1);
          if (lane == 0 && a.lag > 0 && (done & 31u) < 4u && q + 4 < q1) {
            st_volatile_u32(&a.progress[u], done);
            while (true) {
              unsigned mn = 0xFFFFFFFFu;
              for (int tp = 0; tp < a.T; ++tp) {
                const int up = s_split * a.T + tp;
                if (up != u && up / (int)gridDim.x == round) mn = min(mn, ld_volatile_u32(&a.progress[up]));
              }
              if (mn == 0xFFFFFFFFu || done <= mn + (unsigned)a.lag) break;
              __nanosleep(1000);
            }
          }
        }
        if (lane == 0 && a.lag > 0) st_volatile_u32(&a.progress[u], 0xFFFFFFFFu);
        idx += q1 - q0;
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread) =====================
    if (elect_one()) {
      const uint32_t idesc = idesc_tf32(kBM, (uint32_t)a.bn);
      int rs = 0, ls = 0;
      uint32_t rph = 0, lph = 0;
      int ab = 0;
      uint32_t aph = 0;
      long long tci = 0;  // CTA-wide chunk index (trace)
      for (int u = blockIdx.x; u < a.U; u += gridDim.x) {
        if (unit_skipped(a, s_only, u)) continue;
        int t, bi, bj;
        long long q0, q1;
        unit_range(a, u, t, q0, q1);
        tile_coords(a, t, bi, bj);
        const bool diag = a.sym && bi == bj;
        int cpos = 0;
        for (long long q = q0; q < q1; ++q) {
          if (cpos == 0) {
            ts_wait(&acce[ab], aph ^ 1, a.spin & 4);
            tc_fence_after();
          }
          ts_wait(&lfull[ls], lph, a.spin & 4);  // transform done: implies the raw stage landed
          tc_fence_after();
          ts_stamp(a, 1, tci);
          // bn = 128: one accumulator per buffer; bn = 64: separate H H^T and cross accumulators
          // (the truncating accumulation error then comes from the H H^T chain only)
          const uint32_t d = tmem_base + (uint32_t)ab * kTsAccCols;
          const uint32_t dx = kN64 ? d + 64 : d;
          const uint32_t a_hi = tmem_base + 2 * kTsAccCols + (uint32_t)ls * kTsAStageCols;
          const uint32_t a_lo = a_hi + 32;
          const uint64_t yh = kYT ? sw128_kmajor_desc(smem_u32(lo_ptr(ls)))
                                  : sw128_kmajor_desc(smem_u32(raw_ptr(rs, diag ? 0 : 1)));
          const uint64_t yl = sw128_kmajor_desc(smem_u32(lo_ptr(ls)) + (kYT ? (uint32_t)kTileBytes : 0u));
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk) {
            const uint64_t adv = (uint64_t)(kk * 32 >> 4);  // +32 B per K=8 step inside the swizzle atom
            const uint32_t acc = (cpos > 0 || kk > 0) ? 1u : 0u;
            mma_tf32_ts(d, a_hi + kk * 8, yh + adv, idesc, acc);
            mma_tf32_ts(dx, a_hi + kk * 8, yl + adv, idesc, kN64 ? acc : 1u);
            mma_tf32_ts(dx, a_lo + kk * 8, yh + adv, idesc, 1u);
          }
          mma_commit(&rempty[rs]);
          if (++rs == RS) { rs = 0; rph ^= 1; }
          mma_commit(&lempty[ls]);
          ts_stamp(a, 2, tci++);
          if (++ls == kTsLoStages) { ls = 0; lph ^= 1; }
          if (++cpos == a.chain || q + 1 == q1) {
            mma_commit(&accf[ab]);
            cpos = 0;
            if (++ab == 2) { ab = 0; aph ^= 1; }
          }
        }
      }
    }
  } else if ((warp >= 4 && warp < 8) || (kSplitT && warp >= 12)) {
    // ===================== transform: X rows -> TMEM (H, L); Y tile -> L_Y in shared memory ========
    const int quad = warp & 3;         // the TMEM lane quadrant of this warp
    const int tt = quad * 32 + lane;   // 0..127 = tile row handled for the TMEM A operand
    // kSplitT (N = 64): two groups of 4 warps (4-7, 12-15) convert alternate chunks, all 32 K-columns each,
    // so two chunks' conversions overlap (the per-chunk chain load -> split -> tcgen05.st -> wait -> fence ->
    // arrive was ~420 ns of latency with both groups on the same chunk, 16 columns each; scripts/ts_trace.py)
    constexpr int NC = 32;
    const int grp = (kSplitT && warp >= 12) ? 1 : 0;
    constexpr int c0 = 0;
    int rs = 0, ls = 0;
    uint32_t rph = 0, lph = 0;
    long long tfi = 0;  // CTA-wide chunk index (trace)
    for (int u = blockIdx.x; u < a.U; u += gridDim.x) {
      if (unit_skipped(a, s_only, u)) continue;
      int t, bi, bj;
      long long q0, q1;
      unit_range(a, u, t, q0, q1);
      tile_coords(a, t, bi, bj);
      const bool diag = a.sym && bi == bj;
      double sq = 0.0;  // this thread's sum of squared X elements over the unit (a.sq_part)
      for (long long q = q0; q < q1; ++q) {
        if (kSplitT && (int)(tfi & 1) != grp) {  // the other group's chunk: advance the rings only
          ++tfi;
          if (++rs == RS) { rs = 0; rph ^= 1; }
          if (++ls == kTsLoStages) { ls = 0; lph ^= 1; }
          continue;
        }
        ts_wait(&rfull[rs], rph, a.spin & 2);
        if (tt == 0) ts_stamp(a, 3, tfi);
        ts_wait(&lempty[ls], lph ^ 1, a.spin & 2);
        if (tt == 0) ts_stamp(a, 4, tfi);
        tc_fence_after();
        // (1) row tt of X (128-B swizzled row: 16-B chunk c at position c ^ (tt & 7)); for a
        // transposed X the raw tile is [32 K][128 M] unswizzled and row tt of X is column tt
        {
          uint32_t hi[NC], lo[NC];
          if (a.xt) {
            // explicit shared loads (a generic float* compiled to LD.E), all issued before the split
            const uint32_t xcol = smem_u32(raw_ptr(rs, 0)) + (uint32_t)tt * 4u;
            float e[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) e[c] = lds_f32(xcol + (uint32_t)((c0 + c) * kBM) * 4u);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              const uint32_t h = tf32_rn(e[c]);
              hi[c] = h;
              lo[c] = __float_as_uint(e[c] - __uint_as_float(h));
            }
            if (a.sq_part) {  // fp32 within the chunk (<= 32 positive terms), fp64 across chunks
              float cs = 0.f;
#pragma unroll
              for (int c = 0; c < NC; ++c) cs = fmaf(e[c], e[c], cs);
              sq += (double)cs;
            }
          } else {
            const uint32_t xrow = smem_u32(raw_ptr(rs, 0)) + (uint32_t)tt * 128u;
#pragma unroll
            for (int c = 0; c < NC / 4; ++c) {
              const float4 v = lds_f4(xrow + (uint32_t)(((c0 / 4 + c) ^ (tt & 7)) * 16));
              const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint32_t h = tf32_rn(e[j]);
                hi[c * 4 + j] = h;
                lo[c * 4 + j] = __float_as_uint(e[j] - __uint_as_float(h));
              }
              if (a.sq_part) {
                float cs = 0.f;
#pragma unroll
                for (int j = 0; j < 4; ++j) cs = fmaf(e[j], e[j], cs);
                sq += (double)cs;
              }
            }
          }
          const uint32_t ta = tmem_base + ((uint32_t)(quad * 32) << 16) + 2 * kTsAccCols + (uint32_t)ls * kTsAStageCols;
          if constexpr (NC == 32) {
            tmem_st_32x32b_x32(ta, hi);
            tmem_st_32x32b_x32(ta + 32, lo);
          } else {
            tmem_st_32x32b_x16(ta + c0, hi);
            tmem_st_32x32b_x16(ta + 32 + c0, lo);
          }
        }
        // (2) the B-side lo part: L_Y (or L_X for a diagonal tile) in the swizzled smem layout; for
        // a transposed Y, row tt of Y is column tt of the raw [32 K][bn N] tile and both H_Y and
        // L_Y are written (row tt of the swizzled K-major tiles: 16-B chunk c at c ^ (tt & 7))
        if (kYT) {
          if (tt < a.bn) {
            const uint32_t ycol = smem_u32(raw_ptr(rs, diag ? 0 : 1)) + (uint32_t)tt * 4u;
            const int ys = diag ? kBM : a.bn;  // row pitch (floats) of the raw tile
            const uint32_t hrow = smem_u32(lo_ptr(ls)) + (uint32_t)tt * 128u;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              float4 h, l;
              float* hv = &h.x;
              float* lv = &l.x;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float e = lds_f32(ycol + (uint32_t)((c * 4 + j) * ys) * 4u);
                const float hh = __uint_as_float(__float_as_uint(e) & 0xFFFFE000u);
                hv[j] = hh;
                lv[j] = __uint_as_float(tf32_rn(e - hh));
              }
              const uint32_t off = (uint32_t)((c ^ (tt & 7)) * 16);
              sts_f4(hrow + off, h);
              sts_f4(hrow + (uint32_t)kTileBytes + off, l);
            }
          }
        } else {
          const uint32_t src = smem_u32(raw_ptr(rs, diag ? 0 : 1));
          const uint32_t dst = smem_u32(lo_ptr(ls));
          const int nyv = a.bn * (kBK * 4 / 16);  // float4 of the bn used rows
          constexpr int kTT = 128;  // transform threads of the group
          for (int i = tt; i < nyv; i += kTT) {
            const uint32_t off = (uint32_t)i * 16u;
            const float4 v = lds_f4(src + off);
            float4 l;
            if (kYLoRn) {
              l.x = __uint_as_float(tf32_rn(v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u)));
              l.y = __uint_as_float(tf32_rn(v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u)));
              l.z = __uint_as_float(tf32_rn(v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u)));
              l.w = __uint_as_float(tf32_rn(v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u)));
            } else {
              l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
              l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
              l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
              l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
            }
            sts_f4(dst + off, l);
          }
        }
        tmem_st_wait();
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&lfull[ls]);
        if (tt == 0) ts_stamp(a, 5, tfi);
        ++tfi;
        if (++rs == RS) { rs = 0; rph ^= 1; }
        if (++ls == kTsLoStages) { ls = 0; lph ^= 1; }
      }
      if (a.sq_part) {  // fixed-order warp reduction: one partial per (unit, transform warp), 8 per unit
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) {
          a.sq_part[(size_t)u * 8 + grp * 4 + quad] = sq;
          if (!kSplitT) a.sq_part[(size_t)u * 8 + 4 + quad] = 0.0;
        }
      }
    }
  } else if (warp >= 8) {
    // ===================== epilogue: TMEM chains -> fp32 registers -> fp64 partials =====================
    const int e = warp - 8;
    const int quad = warp & 3;
    // columns per epilogue warp: 64 of the 128-wide accumulator; for N = 64 all 64 (kSplitT: warps
    // 8-11 only, drained 16 columns at a time) or 32 (kYT: both warp groups drain) -- no spills
    constexpr int kEC = kN64 ? (kSplitT ? 64 : 32) : 64;
    const int col0 = kSplitT ? 0 : (e >> 2) * kEC;
    const int row = quad * 32 + lane;
    int ab = 0;
    uint32_t aph = 0;
    const bool has_cols = col0 < a.bn;
    for (int u = blockIdx.x; u < a.U; u += gridDim.x) {
      if (unit_skipped(a, s_only, u)) continue;
      int t;
      long long q0, q1;
      unit_range(a, u, t, q0, q1);
      const long long nchains = (q1 - q0 + a.chain - 1) / a.chain;
      if constexpr (!kN64) {
        if (a.resA && nchains == 1) {
          // residual epilogue (SCW error) with one accumulator drain per unit: this
          // thread's A row segment (64 columns) is requested BEFORE the accumulator is waited for,
          // so the loads overlap the unit's MMA instead of following the drain
          int bi, bj;
          tile_coords(a, t, bi, bj);
          const int b = t / a.T0;
          const int gr = bi * kBM + row;
          const int nv = (has_cols && gr < a.Mv) ? min(64, min(a.bn - col0, a.Nv - (bj * a.bn + col0))) : 0;
          const float* ar = a.resA + (size_t)b * a.res_stride + (size_t)(gr < a.Mv ? gr : 0) * a.res_ld +
                            (size_t)bj * a.bn + col0;
          float av[64];
          if (nv == 64 && ((reinterpret_cast<uintptr_t>(ar) & 15) == 0)) {
#pragma unroll
            for (int i = 0; i < 64; i += 4) {
              const float4 v = __ldg(reinterpret_cast<const float4*>(ar + i));
              av[i] = v.x;
              av[i + 1] = v.y;
              av[i + 2] = v.z;
              av[i + 3] = v.w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 64; ++i) av[i] = i < nv ? __ldg(ar + i) : 0.f;
          }
          mbar_wait(&accf[ab], aph);
          tc_fence_after();
          const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)ab * kTsAccCols + col0;
          // (a - s)^2 in fp32 (the difference is exact or correctly rounded, a 32-term sum of squares
          // carries ~1e-7 relative rounding), fp64 across halves and units: the fp64 version spent
          // ~70 % of the epilogue in F2F.F64 conversions
          double acc = 0.0;
          if (has_cols) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint32_t r[32];
              tmem_ld_32x32b_x32(taddr + h * 32, r);
              tmem_ld_wait();
              float s0 = 0.f, s1 = 0.f;
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                const float d0 = (h * 32 + i < nv) ? av[h * 32 + i] - __uint_as_float(r[i]) : 0.f;
                const float d1 = (h * 32 + i + 1 < nv) ? av[h * 32 + i + 1] - __uint_as_float(r[i + 1]) : 0.f;
                s0 = fmaf(d0, d0, s0);
                s1 = fmaf(d1, d1, s1);
              }
              acc += (double)s0 + (double)s1;
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acce[ab]);
          if (++ab == 2) { ab = 0; aph ^= 1; }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (lane == 0) a.res_part[(size_t)u * 8 + e] = acc;
          continue;
        }
      }
      float sum[kEC];
#pragma unroll
      for (int i = 0; i < kEC; ++i) sum[i] = 0.f;
      // staggered folds: epilogue warp e folds (fp32 -> fp64 reductions at L2) at chains offset by
      // e * fold / 8, so no single accumulator drain carries all the L2 reductions of a fold
      int cin = (e * a.fold) / 8;
      bool first_fold = true;
      double* prow = a.part + (size_t)u * (kBM * kBN) + (size_t)row * kBN + col0;
      for (long long c = 0; c < nchains; ++c) {
        mbar_wait(&accf[ab], aph);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)ab * kTsAccCols + col0;
        if (has_cols) {
          if constexpr (kSplitT) {  // separate accumulators: columns [0,64) = H H^T, [64,128) = cross terms
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              uint32_t r[16], x[16];
              tmem_ld_32x32b_x16(taddr + h * 16, r);
              tmem_ld_32x32b_x16(taddr + 64 + h * 16, x);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 16; ++i) sum[h * 16 + i] += __uint_as_float(r[i]) + __uint_as_float(x[i]);
            }
          } else if constexpr (kN64) {
            uint32_t r[32], x[32];
            tmem_ld_32x32b_x32(taddr, r);
            tmem_ld_32x32b_x32(taddr + 64, x);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) sum[i] += __uint_as_float(r[i]) + __uint_as_float(x[i]);
          } else {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint32_t r[32];
              tmem_ld_32x32b_x32(taddr + h * 32, r);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) sum[h * 32 + i] += __uint_as_float(r[i]);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acce[ab]);
        if (++ab == 2) { ab = 0; aph ^= 1; }
        if (a.dout || a.resA) continue;  // direct output / residual: keep summing in fp32, use once at the end
        if (++cin == a.fold || c + 1 == nchains) {
          const uint64_t pol = l2_policy_evict_last();
          if (first_fold) {
#pragma unroll
            for (int i = 0; i < kEC; i += 2)
              st_f64x2_hint(reinterpret_cast<double2*>(prow + i), make_double2((double)sum[i], (double)sum[i + 1]), pol);
          } else {
#pragma unroll
            for (int i = 0; i < kEC; ++i) red_add_f64_hint(prow + i, (double)sum[i], pol);
          }
#pragma unroll
          for (int i = 0; i < kEC; ++i) sum[i] = 0.f;
          first_fold = false;
          cin = 0;
        }
      }
      if (a.resA) {
        // residual epilogue (SCW error): this thread's row segment of A_b minus the
        // rank-r product D = L R^T of the tile, squared and summed in fp64, warp-reduced
        int bi, bj;
        tile_coords(a, t, bi, bj);
        const int b = t / a.T0;
        const int gr = bi * kBM + row;
        double acc = 0.0;
        if (has_cols && gr < a.Mv) {
          const float* ar = a.resA + (size_t)b * a.res_stride + (size_t)gr * a.res_ld + (size_t)bj * a.bn + col0;
          const int nv = min(kEC, min(a.bn - col0, a.Nv - (bj * a.bn + col0)));
          if (nv == kEC && ((reinterpret_cast<uintptr_t>(ar) & 15) == 0)) {
#pragma unroll
            for (int i = 0; i < kEC; i += 4) {
              const float4 v = __ldg(reinterpret_cast<const float4*>(ar + i));
              const double d0 = (double)v.x - (double)sum[i], d1 = (double)v.y - (double)sum[i + 1];
              const double d2 = (double)v.z - (double)sum[i + 2], d3 = (double)v.w - (double)sum[i + 3];
              acc += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
            }
          } else {
#pragma unroll
            for (int i = 0; i < kEC; ++i) {
              if (i < nv) {
                const double d = (double)__ldg(ar + i) - (double)sum[i];
                acc += d * d;
              }
            }
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) a.res_part[(size_t)u * 8 + e] = acc;
        // pull this thread's A segment of the CTA's next unit into L2 while its MMAs run
        const int un = u + (int)gridDim.x;
        if (un < a.U && has_cols) {
          int tn, bin, bjn;
          long long qa, qb;
          unit_range(a, un, tn, qa, qb);
          tile_coords(a, tn, bin, bjn);
          const int grn = bin * kBM + row;
          const int gcn = bjn * a.bn + col0;
          if (grn < a.Mv && gcn < a.Nv) {
            const float* an = a.resA + (size_t)(tn / a.T0) * a.res_stride + (size_t)grn * a.res_ld + gcn;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(an));
            if (gcn + 32 < a.Nv) asm volatile("prefetch.global.L2 [%0];" ::"l"(an + 32));
          }
        }
        continue;
      }
      if (a.dout && has_cols) {
        // transposed store: for a fixed column, the 32 lanes (consecutive rows) write contiguously
        int bi, bj;
        tile_coords(a, t, bi, bj);
        const int b = a.batch ? t / a.T0 : 0;
        const int gr = bi * kBM + row;
        float* ob = a.dout + (size_t)b * a.dstride;
        if (gr < a.Mv) {
          if (a.drow) {
#pragma unroll
            for (int i = 0; i < kEC; ++i) {
              const int gc = bj * a.bn + col0 + i;
              if (col0 + i < a.bn && gc < a.Nv) ob[(size_t)gr * a.ldd + gc] = sum[i];
            }
          } else {
#pragma unroll
            for (int i = 0; i < kEC; ++i) {
              const int gc = bj * a.bn + col0 + i;
              if (col0 + i < a.bn && gc < a.Nv) ob[(size_t)gc * a.ldd + gr] = sum[i];
            }
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// Sum the S partials of every tile in fixed order; write fp64 (and optionally fp32) output.
// sym: only i >= j is summed and mirrored to (j, i), so the result is exactly symmetric.
__global__ void gemm_finalize_kernel(const double* __restrict__ part, int M, int N, int T, int nb, int S, int sym,
                                     double* __restrict__ out64, long long ldo64, float* __restrict__ out32,
                                     long long ldo32, int accumulate) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= M || j >= N) return;
  if (sym && j > i) return;
  const int bi = i / kBM, bj = j / kBN;
  const int t = sym ? bi * (bi + 1) / 2 + bj : bi * nb + bj;
  const size_t off = (size_t)(i % kBM) * kBN + (j % kBN);
  double acc = 0.0;
  for (int s = 0; s < S; ++s) acc += part[(size_t)(s * T + t) * (kBM * kBN) + off];
  if (out64) {
    double v = accumulate ? out64[(size_t)i * ldo64 + j] + acc : acc;
    out64[(size_t)i * ldo64 + j] = v;
    if (sym && i != j) out64[(size_t)j * ldo64 + i] = v;
    acc = v;
  }
  if (out32) {
    out32[(size_t)i * ldo32 + j] = (float)acc;
    if (sym && i != j) out32[(size_t)j * ldo32 + i] = (float)acc;
  }
}

// ------------------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D map over [slices][rows][inner] fp32, box [1][128][32], 128-byte swizzle, OOB -> 0.
static bool make_map_3d(CUtensorMap* map, const float* base, int inner, int rows, long long slices,
                        long long row_stride_elems, long long slice_stride_elems, int box_rows = kBM) {
  auto enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)slices};
  cuuint64_t strides[2] = {(cuuint64_t)(row_stride_elems * 4), (cuuint64_t)(slice_stride_elems * 4)};
  cuuint32_t box[3] = {(cuuint32_t)kBK, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Choose the number of K splits S so that S*T units fill the grid in near-equal rounds.
static int choose_splits(int T, long long Kc, int sms, int min_chunks) {
  int best_s = 1;
  double best_eff = -1.0;
  const long long smax = std::max(1LL, std::min<long long>(Kc / std::max(1, min_chunks), 256));
  for (int s = 1; s <= smax; ++s) {
    long long U = (long long)s * T;
    long long rounds = (U + sms - 1) / sms;
    double eff = (double)U / (double)(rounds * sms);
    if (eff > best_eff + 0.01) {
      best_eff = eff;
      best_s = s;
    }
  }
  return best_s;
}

tsk_status gemm_tf32x3(Ctx* ctx, const GemmProblem& p) {
  if (p.M <= 0 || p.N <= 0 || p.n <= 0 || p.D <= 0) return TSK_EINVAL;
  if ((p.x_row_stride % 4) || (p.y_row_stride % 4) || (p.x_slice_stride % 4) ||
      (p.y_slice_stride % 4) || (reinterpret_cast<uintptr_t>(p.X) & 15) || (reinterpret_cast<uintptr_t>(p.Y) & 15))
    return TSK_ESHAPE;
  if (p.sym && (p.X != p.Y || p.M != p.N)) return TSK_EINVAL;
  // production symmetric Gram: CTA pairs (gram_pair.cu)
  if (p.sym && p.products == 3 && !p.raw && !p.ss && !p.one_cta && !p.batch && !p.xt) return gram_pair(ctx, p);
  CUtensorMap mx, my;
  if (p.xt) {
    // transposed X: [D][K = n][M] with M contiguous (x_row_stride = stride between K rows);
    // box {128 M, 32 K}, no swizzle (the transform reads tile columns, 4-byte lanes: no conflicts)
    if ((p.sym && !p.yt) || p.ss || p.products != 3 || p.raw || (p.x_row_stride % 4) || (p.M % 4)) return TSK_EINVAL;
    auto enc = get_encode_fn();
    if (!enc) return TSK_ECUDA;
    cuuint64_t dims[3] = {(cuuint64_t)p.M, (cuuint64_t)p.n, (cuuint64_t)p.D};
    cuuint64_t strides[2] = {(cuuint64_t)(p.x_row_stride * 4), (cuuint64_t)(p.x_slice_stride * 4)};
    cuuint32_t box[3] = {(cuuint32_t)kBM, (cuuint32_t)kBK, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(p.X), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      if (getenv("TSK_DEBUG")) fprintf(stderr, "[tsk] gemm: transposed X tensor map rejected\n");
      return TSK_ECUDA;
    }
  } else if (!make_map_3d(&mx, p.X, p.n, p.M, p.D, p.x_row_stride, p.x_slice_stride)) {
    if (getenv("TSK_DEBUG")) fprintf(stderr, "[tsk] gemm: X tensor map rejected\n");
    return TSK_ECUDA;
  }
  if (p.yt) {
    // transposed Y: [D][K = n][N] with N contiguous; box {bn N, 32 K}, no swizzle
    if (p.ss || p.products != 3 || p.raw || (p.y_row_stride % 4) || (p.N % 4)) return TSK_EINVAL;
    auto enc = get_encode_fn();
    if (!enc) return TSK_ECUDA;
    const int bnv = (p.bn == 64 && !p.sym) ? 64 : 128;
    cuuint64_t dims[3] = {(cuuint64_t)p.N, (cuuint64_t)p.n, (cuuint64_t)p.D};
    cuuint64_t strides[2] = {(cuuint64_t)(p.y_row_stride * 4), (cuuint64_t)(p.y_slice_stride * 4)};
    cuuint32_t box[3] = {(cuuint32_t)bnv, (cuuint32_t)kBK, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&my, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(p.Y), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      if (getenv("TSK_DEBUG")) fprintf(stderr, "[tsk] gemm: transposed Y tensor map rejected\n");
      return TSK_ECUDA;
    }
  } else if (!make_map_3d(&my, p.Y, p.n, p.N, p.D, p.y_row_stride, p.y_slice_stride,
                          (p.bn == 64 && !p.sym) ? 64 : kBM)) {
    if (getenv("TSK_DEBUG")) fprintf(stderr, "[tsk] gemm: Y tensor map rejected\n");
    return TSK_ECUDA;
  }

  GemmArgs a{};
  a.bn = (p.bn == 64 && !p.sym) ? 64 : 128;
  const int mb = (p.M + kBM - 1) / kBM;
  const int nb = (p.N + a.bn - 1) / a.bn;
  a.sym = p.sym;
  a.nb = nb;
  a.cps = (p.n + kBK - 1) / kBK;
  if (p.batch) {
    // D independent problems; one unit per (problem, tile), results stored directly (fp32)
    if (p.sym || (!p.dout && !p.resA)) return TSK_EINVAL;
    a.batch = 1;
    a.T0 = mb * nb;
    a.T = (int)(p.D * a.T0);
    a.Kc = a.cps;
    a.S = 1;
  } else {
    a.T = p.sym ? mb * (mb + 1) / 2 : mb * nb;
    a.Kc = (long long)p.D * a.cps;
    a.S = p.splits > 0 ? p.splits : choose_splits(a.T, a.Kc, ctx->num_sms, p.min_chunks_per_unit > 0 ? p.min_chunks_per_unit : 8);
    if (a.S > a.Kc) a.S = (int)a.Kc;
  }
  a.Mv = p.M;
  a.Nv = p.N;
  a.xt = p.xt;
  a.ybc = p.ybc;
  a.drow = p.drow;
  a.resA = p.resA;
  a.res_stride = p.res_stride;
  a.res_ld = p.res_ld;
  a.res_part = p.res_part;
  a.only = p.only;
  a.only_any = p.only_any;
  a.spin = getenv("TSK_TS_SPIN") ? atoi(getenv("TSK_TS_SPIN")) : 0;
  a.trace = nullptr;
  a.trace_n = 0;
  const char* ts_trace = getenv("TSK_TS_TRACE");  // diagnostics: scripts/ts_trace.py
  if (ts_trace) {
    a.trace_n = 8192;
    if (cudaMalloc(&a.trace, (size_t)8 * a.trace_n * 8) != cudaSuccess) return TSK_ENOMEM;
    cudaMemsetAsync(a.trace, 0, (size_t)8 * a.trace_n * 8, ctx->stream);
  }
  a.sq_part = p.sq_part;
  if ((p.only || p.sq_part) && !p.batch) return TSK_EINVAL;
  a.dout = p.dout;
  a.dstride = p.dstride;
  a.ldd = p.ldd;
  a.U = a.S * a.T;
  a.chain = p.chain > 0 ? p.chain : 4;
  a.fold = p.fold > 0 ? p.fold : 64;
  a.products = p.products == 1 ? 1 : 3;
  a.raw = p.raw;
  a.lag = a.batch ? 0 : (p.lag >= 0 ? p.lag : 64);
  const size_t part_bytes = (a.dout || a.resA) ? 256 : (size_t)a.U * kBM * kBN * sizeof(double);
  double* part = reinterpret_cast<double*>(ctx->workspace(WS_GEMM_PARTIAL, part_bytes));
  if (!part) return TSK_ENOMEM;
  a.part = part;
  unsigned* prog = reinterpret_cast<unsigned*>(ctx->workspace(WS_GEMM_PROGRESS, (size_t)a.U * sizeof(unsigned)));
  if (!prog) return TSK_ENOMEM;
  a.progress = prog;
  if (cudaMemsetAsync(prog, 0, (size_t)a.U * sizeof(unsigned), ctx->stream) != cudaSuccess) return TSK_ECUDA;

  constexpr int kTsYtSmemBytes = ts_smem_bytes<false, true>();
  constexpr int kTs64SmemBytes = ts_smem_bytes<true, false>();
  static_assert(ts_smem_bytes<true, true>() == kTsYtSmemBytes, "kYT geometry does not depend on N");
  static uint64_t attr_set = 0;
  if (!(attr_set & device_bit())) {
    if (cudaFuncSetAttribute(gemm_tf32x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes) !=
            cudaSuccess ||
        cudaFuncSetAttribute(gemm_tf32x3_ts_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kTsSmemBytes) != cudaSuccess ||
        cudaFuncSetAttribute(gemm_tf32x3_ts_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kTs64SmemBytes) != cudaSuccess ||
        cudaFuncSetAttribute(gemm_tf32x3_ts_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kTsYtSmemBytes) != cudaSuccess ||
        cudaFuncSetAttribute(gemm_tf32x3_ts_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kTsYtSmemBytes) != cudaSuccess)
      return TSK_ECUDA;
    attr_set |= device_bit();
  }
  const int grid = std::min(a.U, ctx->num_sms);
  // production: TS variant (A operand from TMEM); the SS variant serves the diagnostic modes
  if (a.products == 3 && !a.raw && !p.ss) {
    if (p.yt) {
      if (a.bn == 64)
        gemm_tf32x3_ts_kernel<true, true><<<grid, kThreads, kTsYtSmemBytes, ctx->stream>>>(mx, my, a);
      else
        gemm_tf32x3_ts_kernel<false, true><<<grid, kThreads, kTsYtSmemBytes, ctx->stream>>>(mx, my, a);
    } else if (a.bn == 64) {
      gemm_tf32x3_ts_kernel<true, false><<<grid, kThreads, kTs64SmemBytes, ctx->stream>>>(mx, my, a);
    } else {
      gemm_tf32x3_ts_kernel<false, false><<<grid, kThreads, kTsSmemBytes, ctx->stream>>>(mx, my, a);
    }
  } else {
    if (a.batch || a.bn != 128 || a.dout || p.xt || p.yt) return TSK_EINVAL;  // diagnostic SS kernel: plain problems only
    gemm_tf32x3_kernel<<<grid, kThreads, kSmemBytes, ctx->stream>>>(mx, my, a);
  }
  if (launch_status("gemm_tf32x3") != TSK_OK) return TSK_ECUDA;
  ctx->count_launch();
  if (ts_trace) {
    std::vector<unsigned long long> h((size_t)8 * a.trace_n);
    cudaStreamSynchronize(ctx->stream);
    cudaMemcpy(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost);
    cudaFree(a.trace);
    if (FILE* f = fopen(ts_trace, "ab")) {
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  if (a.dout || a.resA) {
    if (p.info) {
      p.info->splits = a.S;
      p.info->units = a.U;
      p.info->grid = grid;
      p.info->tiles = a.T;
    }
    return TSK_OK;
  }

  dim3 fb(32, 8);
  dim3 fg((p.N + 31) / 32, (p.M + 7) / 8);
  gemm_finalize_kernel<<<fg, fb, 0, ctx->stream>>>(part, p.M, p.N, a.T, nb, a.S, p.sym, p.out64, p.ldo64, p.out32,
                                                   p.ldo32, p.accumulate);
  if (cudaPeekAtLastError() != cudaSuccess) return TSK_ECUDA;
  ctx->count_launch();
  if (p.info) {
    p.info->splits = a.S;
    p.info->units = a.U;
    p.info->grid = grid;
    p.info->tiles = a.T;
  }
  return TSK_OK;
}

}  // namespace tsk
