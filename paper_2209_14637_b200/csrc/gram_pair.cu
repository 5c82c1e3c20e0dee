// Symmetric split-TF32 Gram on CTA PAIRS (tcgen05 cta_group::2) -- the production kernel of the
// mode-1 Gram G = sum_d A_d A_d^T, lower-triangle tiles only.
//
// Why pairs: with 1-CTA 128x128 tiles every K=8 MMA reads a 4 KB B operand from shared memory
// per 64 MMA cycles, and together with the TMA fill and the hi/lo split transform the tile needs
// ~128 KB of shared-memory traffic per 32-column chunk against 768 MMA cycles -- shared-memory
// bound (ncu, profiles/: tensor pipe 50 %, shared memory ~75 % busy).  A cta_group::2 MMA
// (M = 256 = two 128-row A blocks, one per CTA, A read from each CTA's TMEM) shares ONE B tile
// between the two SMs, each holding half of its rows: per CTA and chunk the traffic drops to
// ~80 KB (TMA 24 + transform 24 + 8 + MMA-B 24) for the same 768 MMA cycles.
//
// Tile pairing.  The output is cut in 128-row blocks; a pair computes the two tiles (I0, J) and
// (I1, J) that share the column block J (the B operand).  An off-diagonal tile {I, J} may be
// computed either as G_IJ (B = J) or as G_JI = G_IJ^T (B = I); the host orients the tiles so
// every block is the B side of an even number of tiles (flip one edge between two odd blocks),
// which leaves at most one unpaired tile (paired with a dummy A block whose result is dropped).
// A last block with <= 64 valid rows is always the B side with MMA N = 64 (half the MMA work), so
// the 1080 = 8*128 + 56 rows of C4 waste no MMA work on the padding of that block.
// Units = (pair, K window), all windows of equal length.
//
// Precision exactly as the 1-CTA kernel (gemm_tc.cu): H = trunc_tf32(x) is the raw tile (the
// tensor core truncates fp32 operands), L = x - H (exact); D += H_X H_Y^T + H_X L_Y^T + L_X H_Y^T
// in TMEM over chains of `chain` chunks, drained to fp32 registers (round to nearest), folded
// every `fold` chains into fp64 partials; a finalize kernel sums the partials of each tile in a
// fixed order (deterministic), transposing where a tile was computed as G_JI, and mirrors.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptx.cuh"
#include "tsk_internal.h"

namespace tsk {

namespace {

constexpr int kBM = 128;                 // rows of the A block held by each CTA
constexpr int kBK = 32;                  // fp32 per K-chunk row = 128 B (one SW128 row)
constexpr int kZ = 2;                    // slices per TMA box: one stage = kZ chunks (z, z+1 at column kc)
constexpr int kXSub = kBM * kBK * 4;     // 16 KB: one chunk of the A block
constexpr int kYSub = 64 * kBK * 4;      // 8 KB: one chunk of this CTA's half of the B rows (N/2 <= 64)
constexpr int kXBytes = kZ * kXSub;      // 32 KB per stage
constexpr int kYBytes = kZ * kYSub;      // 16 KB per stage
constexpr int kStageBytes = kXBytes + kYBytes;  // 48 KB (multiple of 1024: SW128 alignment)
constexpr int kRaw = 4;                  // TMA ring (stages of kZ chunks)
constexpr int kLo = 4;                   // transform ring, per CHUNK (L_Y in smem + [H_X | L_X] in TMEM)
constexpr int kThreads = 512;
constexpr int kAccCols = 128;            // one accumulator buffer
constexpr int kAccBufs = 2;              // accumulator buffers (double-buffered: drains overlap the MMA;
                                         // 1 buffer + 6 A stages measured no faster)
constexpr int kAStageCols = 64;          // per chunk: H_X 32 cols + L_X 32 cols
constexpr int kTmemCols = 512;           // kAccBufs * 128 + kLo * 64
constexpr int kSmemBytes = kRaw * kStageBytes + kLo * kYSub + 1024 + 256;
static_assert(kAccBufs * kAccCols + kLo * kAStageCols <= kTmemCols, "TMEM budget");
static_assert(kSmemBytes <= 232448, "shared memory budget");

struct PairUnit {
  int I[2];   // A row block of CTA 0 / 1 (I[1] = I[0] for a dummy slot)
  int J;      // B block
  int nb;     // MMA N: 128 or 64
  int grp;    // drift-throttle group (K window), -1 = none
  int pad;
  long long q0, q1;  // global stage range (a stage = kZ slices x 32 columns)
};

struct PairArgs {
  const PairUnit* units;
  int U;
  int cps;              // 32-column chunks per slice
  int chain, fold, lag;
  double* part;         // [U][2][128][128]
  unsigned* progress;   // [U]
  int diag;             // diagnostics: bit 0 = skip the split transform, bit 1 = H*H^T product only,
                        // bit 2 = skip the TMA loads
  unsigned long long* trace;  // diagnostics: per-chunk globaltimer stamps of cluster 0 (nullptr = off)
  int trace_n;
};

__device__ __forceinline__ void tstamp(const PairArgs& a, int cid, int slot, long long i) {
  // every 8th chunk of cluster 0
  if (a.trace && cid == 0 && (i & 7) == 0 && (i >> 3) < a.trace_n)
    a.trace[(size_t)slot * a.trace_n + (i >> 3)] = globaltimer_ns();
}

template <bool kSpin>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gram_pair_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapY64,
                     const __grid_constant__ CUtensorMap mapY32, const PairArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* raw_base = smem;                            // [kRaw][X kZ x 16 KB | Y-half kZ x <= 8 KB]
  uint8_t* lo_base = smem + kRaw * kStageBytes;        // [kLo][L_Y-half <= 8 KB] (one chunk each)
  uint64_t* bars = reinterpret_cast<uint64_t*>(lo_base + kLo * kYSub);
  uint64_t* rfull = bars;              // TMA -> transform (own CTA)
  uint64_t* rempty = rfull + kRaw;     // MMA commit (multicast) -> TMA
  uint64_t* lfull = rempty + kRaw;     // transforms of BOTH CTAs -> MMA (leader's copy used)
  uint64_t* lempty = lfull + kLo;      // MMA commit (multicast) -> transform
  uint64_t* accf = lempty + kLo;       // MMA commit (multicast) -> epilogue
  uint64_t* acce = accf + 2;           // epilogues of BOTH CTAs -> MMA (leader's copy used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const int cid = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapX);
    tma_prefetch_desc(&mapY64);
    tma_prefetch_desc(&mapY32);
    for (int i = 0; i < kRaw; ++i) {
      mbar_init(&rfull[i], 2);   // one arrive.expect_tx per box (A block, B half)
      mbar_init(&rempty[i], 1);
    }
    for (int i = 0; i < kLo; ++i) {
      mbar_init(&lfull[i], 12);  // 6 transform warps x 2 CTAs
      mbar_init(&lempty[i], 1);
    }
    for (int i = 0; i < kAccBufs; ++i) {
      mbar_init(&accf[i], 1);
      mbar_init(&acce[i], 16);   // 8 epilogue warps x 2 CTAs
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc2<kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto x_ptr = [&](int st) { return raw_base + st * kStageBytes; };
  auto y_ptr = [&](int st) { return raw_base + st * kStageBytes + kXBytes; };
  auto l_ptr = [&](int st) { return lo_base + st * kYSub; };

  if (warp == 0) {
    // ===================== TMA producer (own CTA: its A block + its half of the B rows) ==========
    // One box = kZ slices: the TMA engine's cost is per box (~1 us each, serial per issuing
    // thread; scripts/tma_bench.cu), so boxes are made as large as the swizzle allows and are
    // issued by 8 lanes (lanes 0-3: A boxes, 4-7: B boxes of 4 consecutive stages).
    int st = 0;
    uint32_t ph = 0;
    long long tq = 0;
    for (int u = cid; u < a.U; u += nclusters) {
      const PairUnit pu = a.units[u];
      const int xi = crank ? pu.I[1] : pu.I[0];
      const int yrows = pu.nb >> 1;
      const uint32_t ybytes = (uint32_t)(kZ * yrows * kBK * 4);
      const int yrow0 = pu.J * kBM + (int)crank * yrows;
      const CUtensorMap* my = pu.nb == 128 ? &mapY64 : &mapY32;
      const int round = u / nclusters;
      // group of kGrp consecutive stages per pass: never two lanes on the same stage (a lane waiting
      // for a phase that another lane of its own warp must produce could stall the warp)
      constexpr int kGrp = kRaw < 4 ? kRaw : 4;
      for (long long qb = pu.q0; qb < pu.q1; qb += kGrp) {
        const int j = lane % kGrp;
        const long long q = qb + j;
        if (lane < 2 * kGrp && q < pu.q1) {
          const int sl = (st + j) % kRaw;
          const uint32_t pl = ph ^ (uint32_t)(((st + j) / kRaw) & 1);
          (kSpin ? mbar_wait_spin : mbar_wait)(&rempty[sl], pl ^ 1);
          const int z = (int)(q / a.cps) * kZ;
          const int kc = (int)(q % a.cps) * kBK;
          if (a.diag & 4) {  // diagnostics: no loads (operands are whatever the ring holds)
            mbar_arrive(&rfull[sl]);
          } else if (lane < kGrp) {
            mbar_arrive_expect_tx(&rfull[sl], (uint32_t)kXBytes);
            tma_load_3d(x_ptr(sl), &mapX, &rfull[sl], kc, xi * kBM, z);
          } else {
            mbar_arrive_expect_tx(&rfull[sl], ybytes);
            tma_load_3d(y_ptr(sl), my, &rfull[sl], kc, yrow0, z);
          }
        }
        __syncwarp();
        const int nq = (int)min((long long)kGrp, pu.q1 - qb);
        tq += nq;
        ph ^= (uint32_t)(((st + nq) / kRaw) & 1);
        st = (st + nq) % kRaw;
        // drift throttle (CTA 0 only; CTA 1 cannot run ahead of the shared MMA by more than
        // the ring): units of the same K window in the same round read the same operands
        const unsigned done = (unsigned)(qb - pu.q0 + nq);
        if (crank == 0 && a.lag > 0 && pu.grp >= 0 && ((done & 15u) == 0 || qb + nq == pu.q1)) {
          if (lane == 0) st_volatile_u32(&a.progress[u], qb + nq == pu.q1 ? 0xFFFFFFFFu : done);
          if (qb + nq < pu.q1) {
            while (true) {
              unsigned mn = 0xFFFFFFFFu;
              for (int up = round * nclusters + lane; up < min(a.U, (round + 1) * nclusters); up += 32)
                if (up != u && a.units[up].grp == pu.grp) {
                  const unsigned pg = ld_volatile_u32(&a.progress[up]);
                  if (pg != 0u) mn = min(mn, pg);  // a peer that has not started yet is not waited for
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
    // tail: every stage's last commit has landed before this CTA may exit
    if (lane == 0)
      for (int i = 0; i < kRaw; ++i) {
        (kSpin ? mbar_wait_spin : mbar_wait)(&rempty[st], ph ^ 1);
        if (++st == kRaw) { st = 0; ph ^= 1; }
      }
  } else if (warp == 1) {
    // ===================== MMA issuer: leader CTA, one thread =====================
    if (crank == 0 && elect_one()) {
      int rs = 0, ls = 0;
      uint32_t rph = 0, lph = 0;
      int ab = 0;
      uint32_t aph = 0;
      long long ti = 0;
      if (a.trace) a.trace[(size_t)11 * a.trace_n + 2 * cid] = globaltimer_ns();
      for (int u = cid; u < a.U; u += nclusters) {
        const PairUnit pu = a.units[u];
        const uint32_t idesc = idesc_tf32(256, (uint32_t)pu.nb);
        const uint32_t ysub = (uint32_t)(pu.nb >> 1) * kBK * 4;  // bytes of one chunk of the B half
        int cpos = 0;
        for (long long q = pu.q0; q < pu.q1; ++q) {
#pragma unroll
          for (int zs = 0; zs < kZ; ++zs, ++ti) {
            tstamp(a, cid, 0, ti);
            if (cpos == 0) {
              (kSpin ? mbar_wait_cluster_spin : mbar_wait_cluster)(&acce[ab], aph ^ 1);
              tc_fence_after();
            }
            // both CTAs' transforms of this chunk done (which implies its raw stage landed)
            (kSpin ? mbar_wait_cluster_spin : mbar_wait_cluster)(&lfull[ls], lph);
            tc_fence_after();
            tstamp(a, cid, 1, ti);
            const uint32_t d = tmem_base + (uint32_t)ab * kAccCols;
            const uint32_t a_hi = tmem_base + kAccBufs * kAccCols + (uint32_t)ls * kAStageCols;
            const uint32_t a_lo = a_hi + 32;
            const uint64_t yh = sw128_kmajor_desc(smem_u32(y_ptr(rs)) + zs * ysub);
            const uint64_t yl = sw128_kmajor_desc(smem_u32(l_ptr(ls)));
#pragma unroll
            for (int kk = 0; kk < kBK / 8; ++kk) {
              const uint64_t adv = (uint64_t)(kk * 32 >> 4);
              const uint32_t acc = (cpos > 0 || kk > 0) ? 1u : 0u;
              mma2_tf32_ts(d, a_hi + kk * 8, yh + adv, idesc, acc);
              if (!(a.diag & 2)) {
                mma2_tf32_ts(d, a_hi + kk * 8, yl + adv, idesc, 1u);
                mma2_tf32_ts(d, a_lo + kk * 8, yh + adv, idesc, 1u);
              }
            }
            mma2_commit_mc(&lempty[ls], 3);
            if (++ls == kLo) { ls = 0; lph ^= 1; }
            tstamp(a, cid, 2, ti);
            if (++cpos == a.chain || (q + 1 == pu.q1 && zs + 1 == kZ)) {
              mma2_commit_mc(&accf[ab], 3);
              cpos = 0;
              if (++ab == kAccBufs) { ab = 0; aph ^= 1; }
            }
          }
          mma2_commit_mc(&rempty[rs], 3);
          if (++rs == kRaw) { rs = 0; rph ^= 1; }
        }
      }
      if (a.trace) a.trace[(size_t)11 * a.trace_n + 2 * cid + 1] = globaltimer_ns();
    }
  } else if (warp >= 2 && warp < 8) {
    // ===================== transform (own CTA) =====================
    // warps 4-7: X rows -> TMEM [H | L] (warp w may only reach TMEM lanes 32 (w % 4) .. +31);
    // warps 2-3: Y-half -> L_Y in shared memory.  Both halves run concurrently (the transform
    // latency is on the critical path of the ring, scripts/gram_pair_trace.py).
    const bool xw = warp >= 4;
    const int tt = xw ? (int)threadIdx.x - 128 : (int)threadIdx.x - 64;
    const int quad = warp & 3;
    const uint32_t lfull_leader = mapa_shared(smem_u32(&lfull[0]), 0);
    long long ti = 0;
    int rs = 0, ls = 0;
    uint32_t rph = 0, lph = 0;
    for (int u = cid; u < a.U; u += nclusters) {
      const int ychunks = (a.units[u].nb >> 1) * (kBK * 4 / 16);  // float4 per chunk of the Y-half
      const uint32_t ysub = (uint32_t)ychunks * 16u;
      const long long nq = a.units[u].q1 - a.units[u].q0;
      for (long long q = 0; q < nq; ++q) {
        (kSpin ? mbar_wait_spin : mbar_wait)(&rfull[rs], rph);
#pragma unroll
        for (int zs = 0; zs < kZ; ++zs, ++ti) {
          if (xw && tt == 0) tstamp(a, cid, 3 + 3 * (int)crank, ti);
          (kSpin ? mbar_wait_spin : mbar_wait)(&lempty[ls], lph ^ 1);
          if (xw && tt == 0) tstamp(a, cid, 4 + 3 * (int)crank, ti);
          tc_fence_after();
          if (!(a.diag & 1)) {
            if (xw) {
              const uint32_t xrow = smem_u32(x_ptr(rs)) + (uint32_t)(zs * kXSub) + (uint32_t)tt * 128u;
              uint32_t hi[32], lo[32];
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const float4 v = lds_f4(xrow + (uint32_t)((c ^ (tt & 7)) * 16));
                const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                  const uint32_t h = __float_as_uint(e[jj]) & 0xFFFFE000u;
                  hi[c * 4 + jj] = h;
                  lo[c * 4 + jj] = __float_as_uint(e[jj] - __uint_as_float(h));
                }
              }
              const uint32_t ta =
                  tmem_base + ((uint32_t)(quad * 32) << 16) + kAccBufs * kAccCols + (uint32_t)ls * kAStageCols;
              tmem_st_32x32b_x32(ta, hi);
              tmem_st_32x32b_x32(ta + 32, lo);
            }
            // L_Y over all 192 transform threads (X warps take their share after issuing the STTMs)
            const uint32_t src = smem_u32(y_ptr(rs)) + (uint32_t)zs * ysub;
            const uint32_t dst = smem_u32(l_ptr(ls));
            const int g = xw ? tt : 128 + tt;
            // <= 3 float4 per thread (ychunks <= 512): all loads issued before the first use, so one shared-
            // memory latency is paid per chunk instead of one per item (the compiler reused one register
            // quadruple for a rolled loop and serialised load -> split -> store)
            float4 v[3];
#pragma unroll
            for (int q = 0; q < 3; ++q)
              if (g + 192 * q < ychunks) v[q] = lds_f4(src + (uint32_t)(g + 192 * q) * 16u);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              if (g + 192 * q < ychunks) {
                float4 l;
                l.x = v[q].x - __uint_as_float(__float_as_uint(v[q].x) & 0xFFFFE000u);
                l.y = v[q].y - __uint_as_float(__float_as_uint(v[q].y) & 0xFFFFE000u);
                l.z = v[q].z - __uint_as_float(__float_as_uint(v[q].z) & 0xFFFFE000u);
                l.w = v[q].w - __uint_as_float(__float_as_uint(v[q].w) & 0xFFFFE000u);
                sts_f4(dst + (uint32_t)(g + 192 * q) * 16u, l);
              }
            }
            if (xw) tmem_st_wait();
          }
          fence_proxy_async_smem();
          tc_fence_before();
          __syncwarp();
          if (xw && tt == 0) tstamp(a, cid, 5 + 3 * (int)crank, ti);
          if (lane == 0) mbar_arrive_cluster(lfull_leader + (uint32_t)ls * 8u);
          if (++ls == kLo) { ls = 0; lph ^= 1; }
        }
        if (++rs == kRaw) { rs = 0; rph ^= 1; }
      }
    }
    if (lane == 0)
      for (int i = 0; i < kLo; ++i) {
        (kSpin ? mbar_wait_spin : mbar_wait)(&lempty[ls], lph ^ 1);
        if (++ls == kLo) { ls = 0; lph ^= 1; }
      }
  } else if (warp >= 8) {
    // ===================== epilogue (own CTA): TMEM -> fp32 registers -> fp64 partials ============
    const int e = warp - 8;
    const int quad = warp & 3;
    const int col0 = (e >> 2) * 64;
    const int row = quad * 32 + lane;
    const uint32_t acce_leader = mapa_shared(smem_u32(&acce[0]), 0);
    long long tc = 0;
    int ab = 0;
    uint32_t aph = 0;
    for (int u = cid; u < a.U; u += nclusters) {
      const bool has_cols = col0 < a.units[u].nb;
      const long long nchains = ((a.units[u].q1 - a.units[u].q0) * kZ + a.chain - 1) / a.chain;
      float sum[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) sum[i] = 0.f;
      // staggered folds: epilogue warp e folds (fp32 -> fp64 reductions at L2) at chains offset by
      // e * fold / 8, so no single accumulator drain carries all the L2 reductions of a fold
      int cin = (e * a.fold) / 8;
      bool first_fold = true;
      double* prow = a.part + ((size_t)u * 2 + crank) * (kBM * kBM) + (size_t)row * kBM + col0;
      for (long long c = 0; c < nchains; ++c) {
        (kSpin ? mbar_wait_spin : mbar_wait)(&accf[ab], aph);
        tc_fence_after();
        if (e == 0 && lane == 0 && crank == 0) tstamp(a, cid, 9, tc * 8);
        const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)ab * kAccCols + col0;
        if (has_cols) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(taddr + h * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) sum[h * 32 + i] += __uint_as_float(r[i]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (e == 0 && lane == 0 && crank == 0) tstamp(a, cid, 10, tc * 8);
        ++tc;
        if (lane == 0) mbar_arrive_cluster(acce_leader + (uint32_t)ab * 8u);
        if (++ab == kAccBufs) { ab = 0; aph ^= 1; }
        if (++cin == a.fold || c + 1 == nchains) {
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
      if (nchains == 0) {  // empty K range: the partial is zero
#pragma unroll
        for (int i = 0; i < 64; i += 2) reinterpret_cast<double2*>(prow + i)[0] = make_double2(0.0, 0.0);
      }
    }
  }

  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc2<kTmemCols>(tmem_base);
  }
}

// G[i][j] (i >= j) = sum over the units of tile t of its partial (transposed where the tile was
// computed as G_JI); fixed order => deterministic.  Mirrors to (j, i).
struct TileRef {
  int first;   // index into unit_list
  int count;
  int slot;    // CTA slot of the pair that holds the tile
  int trans;   // partial holds G_JI = G_IJ^T
};

// One CTA per lower 32 x 32 block of G (a block lies inside one 128-row tile): each element sums its
// tile's K-window partials in the fixed unit order; the thread -> element map follows the partial's
// layout (row-major, or transposed for a tile computed as G_JI) so the partial reads are coalesced, and the
// block goes through shared memory so both the lower write and its mirror are row-contiguous.  (The
// element-per-thread kernel this replaces read transposed tiles and wrote the mirror at a stride of m:
// 100 us per C4 launch under ncu; this kernel 61 us, the tile's unit bases staged in shared memory and the
// thread's 4 elements summed together.)  Same sums in the same order: bit-identical output.
__global__ void __launch_bounds__(256) gram_pair_finalize_kernel(const double* __restrict__ part,
                                                                 const TileRef* __restrict__ tiles,
                                                                 const int* __restrict__ unit_list, int M,
                                                                 double* __restrict__ out64, long long ldo64,
                                                                 float* __restrict__ out32, long long ldo32,
                                                                 int accumulate) {
  __shared__ double t[32][33];
  __shared__ long long ubase[64];  // the tile's partial bases, in the fixed unit order
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  if (j0 > i0) return;
  const int bi = i0 / kBM, bj = j0 / kBM;
  const TileRef tr = tiles[bi * (bi + 1) / 2 + bj];
  const int tx = threadIdx.x, tid = threadIdx.y * 32 + tx;
  const int cnt = min(tr.count, 64);
  for (int e = tid; e < cnt; e += 256) ubase[e] = ((long long)unit_list[tr.first + e] * 2 + tr.slot) * (kBM * kBM);
  __syncthreads();
  // the thread's 4 elements: rows yy = threadIdx.y + 8 q of the block (in the partial's orientation)
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int off[4];
  bool ok[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int yy = threadIdx.y + 8 * q;
    const int li = tr.trans ? tx : yy, lj = tr.trans ? yy : tx;  // element (i0 + li, j0 + lj)
    const int i = i0 + li, j = j0 + lj;
    ok[q] = i < M && j < M && j <= i;
    off[q] = tr.trans ? (j % kBM) * kBM + (i % kBM) : (i % kBM) * kBM + (j % kBM);
  }
  for (int e = 0; e < tr.count; ++e) {
    const long long b = e < 64 ? ubase[e] : ((long long)unit_list[tr.first + e] * 2 + tr.slot) * (kBM * kBM);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (ok[q]) acc[q] += part[b + off[q]];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int yy = threadIdx.y + 8 * q;
    const int li = tr.trans ? tx : yy, lj = tr.trans ? yy : tx;
    const int i = i0 + li, j = j0 + lj;
    double v = 0.0;
    if (ok[q]) v = (out64 && accumulate) ? out64[(size_t)i * ldo64 + j] + acc[q] : acc[q];
    t[li][lj] = v;
  }
  __syncthreads();
  for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
    // lower element (i0 + yy, j0 + tx) and the mirror (j0 + yy, i0 + tx) = lower element (i0 + tx, j0 + yy)
    const int i = i0 + yy, j = j0 + tx;
    if (i < M && j < M && j <= i) {
      if (out64) out64[(size_t)i * ldo64 + j] = t[yy][tx];
      if (out32) out32[(size_t)i * ldo32 + j] = (float)t[yy][tx];
    }
    const int mi = i0 + tx, mj = j0 + yy;  // lower element whose mirror is (mj, mi)
    if (mi < M && mj < M && mj < mi) {
      if (out64) out64[(size_t)mj * ldo64 + mi] = t[tx][yy];
      if (out32) out32[(size_t)mj * ldo32 + mi] = (float)t[tx][yy];
    }
  }
}

// ------------------------------------------------------------------------------ host schedule
struct Sched : HostCache {
  int m = -1, nsm = -1;
  long long Kc = -1;
  int splits_req = -1;
  std::vector<PairUnit> units;
  std::vector<TileRef> tiles;
  std::vector<int> unit_list;
  int S = 0;
  long long ver = 0;
};

// Orient the lower-triangle tiles, pair them by B block, and cut K into windows.
static void build_sched(Sched& s, int m, long long Kc, int nsm, int splits_req, int min_chunks) {
  const int nbk = (m + kBM - 1) / kBM;
  const int vlast = m - kBM * (nbk - 1);
  const int narrow = vlast <= 64 ? nbk - 1 : -1;
  const int T = nbk * (nbk + 1) / 2;
  // orientation: bsel[t] = the B block of tile t
  std::vector<int> ti(T), tj(T), bsel(T);
  for (int I = 0, t = 0; I < nbk; ++I)
    for (int J = 0; J <= I; ++J, ++t) {
      ti[t] = I;
      tj[t] = J;
      bsel[t] = (I == narrow) ? I : J;  // the narrow block is always B (MMA N = 64)
    }
  std::vector<int> cnt(nbk, 0);
  for (int t = 0; t < T; ++t) cnt[bsel[t]]++;
  std::vector<int> odd;
  for (int b = 0; b < nbk; ++b)
    if (b != narrow && (cnt[b] & 1)) odd.push_back(b);
  for (size_t k = 0; k + 1 < odd.size(); k += 2) {  // flip the edge between two odd blocks
    const int u = std::max(odd[k], odd[k + 1]), v = std::min(odd[k], odd[k + 1]);
    const int t = u * (u + 1) / 2 + v;
    cnt[bsel[t]]--;
    bsel[t] = (bsel[t] == u) ? v : u;
    cnt[bsel[t]]++;
  }
  // pairs
  struct Pair { int I[2]; int J; int nb; int t[2]; };
  std::vector<Pair> pairs;
  for (int b = 0; b < nbk; ++b) {
    std::vector<int> mine;
    for (int t = 0; t < T; ++t)
      if (bsel[t] == b) mine.push_back(t);
    for (size_t k = 0; k < mine.size(); k += 2) {
      Pair p;
      p.J = b;
      p.nb = (b == narrow) ? 64 : 128;
      for (int c = 0; c < 2; ++c) {
        const size_t kk = std::min(k + c, mine.size() - 1);
        const int t = mine[kk];
        p.I[c] = (bsel[t] == tj[t]) ? ti[t] : tj[t];  // the A block = the other block of the tile
        p.t[c] = (k + c < mine.size()) ? t : -1;       // -1: dummy slot
      }
      pairs.push_back(p);
    }
  }
  // K windows: every pair gets S units of equal K range.  (An N = 64 pair issues half the MMA work
  // per chunk, but the kernel is paced by the per-chunk TMA / transform work, which is the same.)
  const int ncl = std::max(1, nsm / 2);
  const int P = (int)pairs.size();
  int S = 1;
  if (splits_req > 0) {
    S = splits_req;
  } else {
    double best = -1.0;
    const long long smax = std::max(1LL, std::min<long long>(Kc / std::max(1, min_chunks), 512));
    for (int sc = 1; sc <= smax; ++sc) {
      const long long U = (long long)P * sc;
      const long long rounds = (U + ncl - 1) / ncl;
      const double eff = (double)U / (double)(rounds * ncl);
      if (eff > best + 0.005) {
        best = eff;
        S = sc;
      }
    }
  }
  if (Kc < S) S = (int)std::max(1LL, Kc);
  s.units.clear();
  s.S = S;
  std::vector<std::vector<int>> pair_units(pairs.size());
  for (int w = 0; w < S; ++w)
    for (size_t pi = 0; pi < pairs.size(); ++pi) {
      const Pair& p = pairs[pi];
      PairUnit u{};
      u.I[0] = p.I[0];
      u.I[1] = p.I[1];
      u.J = p.J;
      u.nb = p.nb;
      u.grp = w;
      u.q0 = (long long)w * Kc / S;
      u.q1 = (long long)(w + 1) * Kc / S;
      pair_units[pi].push_back((int)s.units.size());
      s.units.push_back(u);
    }
  s.tiles.assign(T, TileRef{0, 0, 0, 0});
  s.unit_list.clear();
  for (size_t pi = 0; pi < pairs.size(); ++pi)
    for (int c = 0; c < 2; ++c) {
      const int t = pairs[pi].t[c];
      if (t < 0) continue;
      TileRef tr;
      tr.first = (int)s.unit_list.size();
      tr.count = (int)pair_units[pi].size();
      tr.slot = c;
      tr.trans = (bsel[t] == ti[t] && ti[t] != tj[t]) ? 1 : 0;  // computed as G_JI
      for (int u : pair_units[pi]) s.unit_list.push_back(u);
      s.tiles[t] = tr;
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

bool map3d(CUtensorMap* map, const float* base, int inner, int rows, long long slices, long long rs, long long ss,
           int box_rows, int box_z) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)slices};
  cuuint64_t strides[2] = {(cuuint64_t)(rs * 4), (cuuint64_t)(ss * 4)};
  cuuint32_t box[3] = {(cuuint32_t)kBK, (cuuint32_t)box_rows, (cuuint32_t)box_z};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

tsk_status gram_pair(Ctx* ctx, const GemmProblem& p) {
  if (!p.sym || p.X != p.Y || p.M != p.N) return TSK_EINVAL;
  const int m = p.M;
  const int cps = (p.n + kBK - 1) / kBK;
  const long long Kc = (p.D + kZ - 1) / kZ * cps;  // stages of kZ slices (an odd last slice: TMA zero fill)
  CUtensorMap mx, my64, my32;
  if (!map3d(&mx, p.X, p.n, m, p.D, p.x_row_stride, p.x_slice_stride, kBM, kZ) ||
      !map3d(&my64, p.X, p.n, m, p.D, p.x_row_stride, p.x_slice_stride, 64, kZ) ||
      !map3d(&my32, p.X, p.n, m, p.D, p.x_row_stride, p.x_slice_stride, 32, kZ))
    return TSK_ECUDA;

  static uint64_t attr = 0;
  if (!(attr & device_bit())) {
    if (cudaFuncSetAttribute(gram_pair_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes) !=
            cudaSuccess ||
        cudaFuncSetAttribute(gram_pair_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes) !=
            cudaSuccess)
      return TSK_ECUDA;
    attr |= device_bit();
  }
  // persistent clusters: no more than can be co-resident (the drift throttle assumes every unit of
  // a round is running)
  const int nsm = ctx->num_sms & ~1;
  static int max_clusters_dev[64] = {};  // per device (0 = not queried yet)
  int& max_clusters = max_clusters_dev[ctx->device & 63];
  if (max_clusters <= 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nsm);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, gram_pair_kernel<false>, &cfg) != cudaSuccess || nc < 1) {
      cudaGetLastError();
      nc = nsm / 2;
    }
    max_clusters = std::min(nc, nsm / 2);
    if (getenv("TSK_DEBUG"))
      fprintf(stderr, "[tsk] gram_pair: max active clusters %d (occupancy query %d)\n", max_clusters, nc);
  }
  int ncl = max_clusters;
  if (const char* ev = getenv("TSK_PAIR_CLUSTERS")) ncl = std::max(1, std::min(ncl, atoi(ev)));

  // host schedule cache, per ctx (depends on m, K chunks, clusters, requested splits)
  if (!ctx->gram_sched) ctx->gram_sched.reset(new Sched());
  Sched& sched = *static_cast<Sched*>(ctx->gram_sched.get());
  const int min_chunks = std::max(1, (p.min_chunks_per_unit > 0 ? p.min_chunks_per_unit : 8) / kZ);
  if (sched.m != m || sched.Kc != Kc || sched.nsm != 2 * ncl || sched.splits_req != p.splits) {
    build_sched(sched, m, Kc, 2 * ncl, p.splits, min_chunks);
    sched.m = m;
    sched.Kc = Kc;
    sched.nsm = 2 * ncl;
    sched.splits_req = p.splits;
    sched.ver++;
  }
  const int U = (int)sched.units.size();
  const size_t ub = sched.units.size() * sizeof(PairUnit);
  const size_t tb = sched.tiles.size() * sizeof(TileRef);
  const size_t lb = sched.unit_list.size() * sizeof(int);
  uint8_t* dsched = reinterpret_cast<uint8_t*>(ctx->workspace(WS_GRAM_SCHED, ub + tb + lb + 64));
  double* part = reinterpret_cast<double*>(ctx->workspace(WS_GEMM_PARTIAL, (size_t)U * 2 * kBM * kBM * 8));
  unsigned* prog = reinterpret_cast<unsigned*>(ctx->workspace(WS_GEMM_PROGRESS, (size_t)U * sizeof(unsigned)));
  if (!dsched || !part || !prog) return TSK_ENOMEM;
  // the schedule (a few KB) is uploaded once per shape (a synchronous copy, off the steady state)
  if (ctx->gram_sched_dev != dsched || ctx->gram_sched_ver != sched.ver) {
    std::vector<uint8_t> hs(ub + tb + lb);
    std::copy_n(reinterpret_cast<const uint8_t*>(sched.units.data()), ub, hs.data());
    std::copy_n(reinterpret_cast<const uint8_t*>(sched.tiles.data()), tb, hs.data() + ub);
    std::copy_n(reinterpret_cast<const uint8_t*>(sched.unit_list.data()), lb, hs.data() + ub + tb);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess ||
        cudaMemcpy(dsched, hs.data(), hs.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      return TSK_ECUDA;
    ctx->gram_sched_dev = dsched;
    ctx->gram_sched_ver = sched.ver;
  }
  if (cudaMemsetAsync(prog, 0, (size_t)U * sizeof(unsigned), ctx->stream) != cudaSuccess) return TSK_ECUDA;

  PairArgs a;
  a.units = reinterpret_cast<const PairUnit*>(dsched);
  a.U = U;
  a.cps = cps;
  // chain / fold / lag arrive in chunks (GemmProblem units); the kernel counts stages of kZ chunks
  a.chain = p.chain > 0 ? p.chain : 4;
  // fold every 1024 chains (round 2; was 64): the uncoalesced fp64 L2 reductions of a fold cost ~6 % of
  // the C4 launch at 64 (23.5 -> ~22.0 ms, scripts/gram_fold.py), while the Gram error is unchanged
  // (2.72e-6 rel-F at C2-C4 for every fold from 64 to one per unit: it is the tensor core's truncating
  // accumulation within a chain, not the round-to-nearest fp32 register sums, that sets it)
  a.fold = p.fold > 0 ? p.fold : 1024;
  a.lag = p.lag >= 0 ? (p.lag + kZ - 1) / kZ : 64 / kZ;
  // developer overrides (scripts/gram_pair_time.py sweeps)
  if (const char* ev = getenv("TSK_PAIR_FOLD")) a.fold = std::max(1, atoi(ev));
  if (const char* ev = getenv("TSK_PAIR_LAG")) a.lag = atoi(ev) <= 0 ? 0 : std::max(1, (atoi(ev) + kZ - 1) / kZ);  // 0: throttle off
  a.part = part;
  a.progress = prog;
  // diagnostics only (developer experiments, scripts/gram_pair_*.py): TSK_PAIR_DIAG bit 0 = skip
  // the split transform, bit 1 = H*H^T product only, bit 2 = skip the TMA loads
  a.diag = 0;
  if (const char* dv = getenv("TSK_PAIR_DIAG")) a.diag = atoi(dv) & 7;
  a.trace = nullptr;
  a.trace_n = 0;
  const char* trace_path = getenv("TSK_PAIR_TRACE");
  if (trace_path) {
    a.trace_n = 4096;
    if (cudaMalloc(&a.trace, ((size_t)11 * a.trace_n + 2 * 148) * 8) != cudaSuccess) return TSK_ENOMEM;
    cudaMemsetAsync(a.trace, 0, ((size_t)11 * a.trace_n + 2 * 148) * 8, ctx->stream);
  }
  const int grid = 2 * std::min(U, ncl);
  if (getenv("TSK_DEBUG"))
    fprintf(stderr, "[tsk] gram_pair: m=%d Kc=%lld S=%d units=%d grid=%d\n", m, Kc, sched.S, U, grid);
  if (p.spin_waits)
    gram_pair_kernel<true><<<grid, kThreads, kSmemBytes, ctx->stream>>>(mx, my64, my32, a);
  else
    gram_pair_kernel<false><<<grid, kThreads, kSmemBytes, ctx->stream>>>(mx, my64, my32, a);
  if (cudaPeekAtLastError() != cudaSuccess) return TSK_ECUDA;
  ctx->count_launch();
  if (trace_path) {
    std::vector<unsigned long long> h((size_t)11 * a.trace_n + 2 * 148);
    cudaStreamSynchronize(ctx->stream);
    cudaMemcpy(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost);
    cudaFree(a.trace);
    if (FILE* f = fopen(trace_path, "wb")) {
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  dim3 fb(32, 8);
  dim3 fg((m + 31) / 32, (m + 31) / 32);
  gram_pair_finalize_kernel<<<fg, fb, 0, ctx->stream>>>(
      part, reinterpret_cast<const TileRef*>(dsched + ub), reinterpret_cast<const int*>(dsched + ub + tb), m,
      p.out64, p.ldo64, p.out32, p.ldo32, p.accumulate);
  if (cudaPeekAtLastError() != cudaSuccess) return TSK_ECUDA;
  ctx->count_launch();
  if (p.info) {
    p.info->splits = sched.S;
    p.info->units = U;
    p.info->grid = grid;
    p.info->tiles = (int)sched.tiles.size();
  }
  return TSK_OK;
}

}  // namespace tsk
