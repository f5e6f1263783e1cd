// Register-resident fronts: one warp per (front, shift) for the small fronts
// (m <= 8 MT), the whole partial LDL^T in the DMMA accumulator layout.
//
// Replaces, for the deep levels of the dissection tree, the per-shift SuperLU
// factorization of the reference (solvers.py:383-393 -> sparse_direct.py:155-188)
// like factor_front_kernel does, but without shared memory for the front and
// without CTA barriers: the front's lower triangle lives in registers as
// 8 x 8 tiles in the C/D fragment layout of mma.sync m8n8k4 f64 (lane
// (g, t) holds rows g, columns 2t and 2t+1 of every tile), so a warp carries
// its front from assembly to write-out with shuffles only.
//
// Index permutation inside each 8-block. Rows and columns of a tile are stored
// in the order phys = rho(logical) with rho(k) = 2 (k & 3) + (k >> 2), i.e.
// lane (g, t) holds the logical entries (pi(g), t) and (pi(g), t + 4),
// pi = rho^-1 = [0, 4, 1, 5, 2, 6, 3, 7]. Its two accumulator registers are
// then exactly the A fragment of the tile for the K-slices {0..3} and
// {4..7}, and -- scaled by the pivots -- its B fragment: the rank-8 trailing
// updates S_IJ -= X_I D X_J^T run on DMMA straight from the registers that
// hold the panel, with no shuffles and no shared-memory round trip. The pivot
// order itself is the logical one (the permutation only changes where an
// entry is stored), so the factors are the same LDL^T as factor_front_kernel's
// up to rounding order.
//
// Per 8-pivot block:
//  (a) the diagonal tile is factored in place with shuffles; the same row
//      operations applied to an identity tile give L11^-1 in the same layout
//      (Gauss-Jordan style), so M = L11^-T D^-1 is a per-lane product, again
//      without shuffles;
//  (b) panel tiles: X = A M on DMMA (A fragment = the lane's own registers);
//  (c) trailing tiles: S_IJ -= X_I (X_J D)^T on DMMA (4 real MMAs per K-slice,
//      accumulating in place).
// Assembly pulls each child's update block through the child's parent-row map
// (cmap), children in order (deterministic sums): the child's lower update
// block is first staged in a per-warp shared-memory buffer by cp.async (the
// whole block in flight at once without holding registers), then read by
// one LDS per register entry; the originals (M + lambda A on the pivot columns)
// come from a per-CTA dense shared-memory image built from the front's
// original-entry list, shared by the CTA's four shifts.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace {

#ifndef KH_WF_WARPS
#define KH_WF_WARPS 4
#endif
constexpr int WF_WARPS = KH_WF_WARPS;  // shifts per CTA (one warp each)
constexpr int WF_KMAP = WF_WARPS < 4 ? WF_WARPS : 4;  // children whose pull maps are tabulated in shared memory (by warp k)
// packed (lower, by columns) update-block index in 32-bit arithmetic (q <= 64)
KH_DEV int upk32(int q, int i, int j) { return i + j * (2 * q - j - 1) / 2; }
// per-warp child staging buffer: packed lower triangle of a q <= 8 MT update
// block followed by a zero slot
KH_HD constexpr int WF_CHILD_MAX(int mt) { return 4 * mt * (8 * mt + 1) + 2; }  // + zero slot (+ pad)

KH_DEV int perm8(int g) { return (g >> 1) + 4 * (g & 1); }           // phys -> logical
KH_HD constexpr int rho8(int k) { return 2 * (k & 3) + (k >> 2); }   // logical -> phys

KH_DEV double2 shfl2w(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

KH_HD constexpr int tix(int I, int J) { return I * (I + 1) / 2 + J; }

// Blocked LDL^T of the register-resident tile triangle S (lower, MT x MT
// tiles in the permuted accumulator layout) over its first p of m rows, one
// 8-pivot block per iteration of a runtime loop: the body works on the
// triangle relative to the current diagonal tile (S[tix(0, 0)]); after a
// block, col(kb, nt, w, dk, Mr, Mi) writes out the finished tile column
// (tiles S[tix(I, 0)], I < nt: L with D on the diagonal; dk = the lane's
// pivots d_t, d_{t+4}; Mr / Mi = the block's M_j B fragments) and the
// triangle shifts up-left by one tile (register moves): one copy of the
// block code instead of MT. Returns the first index not eliminated (the
// trailing triangle is then the Schur complement); minp = min |d|^2 or -1.
template <int MT, class ColFn>
KH_DEV int tile_ldlt(double2 (&S)[MT * (MT + 1) / 2][2], int p, int m, double& minp, ColFn col) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int rl = perm8(g);
  const int M8 = (m + 7) >> 3;
  int kb = 0;
#pragma unroll 1
  for (; kb < p; kb += 8) {
    const int w = min(8, p - kb);
    const int nt = M8 - (kb >> 3);  // tile rows left (>= 1)
    double2(&Dg)[2] = S[0];
    // E: identity in the same layout; receives the row operations -> L11^-1
    double2 E[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) E[h] = make_double2(rl == t + 4 * h ? 1.0 : 0.0, 0.0);
    double2 dk[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};  // d_{t}, d_{t+4}
    double2 dinv_row = make_double2(0.0, 0.0);                           // 1 / d_{rl}
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k < w) {
        const int rk = rho8(k), sk = rk & 1, qk4 = rk >> 1;  // phys index, slot, quad lane
        const double2 d = shfl2w(Dg[sk], rk * 4 + qk4);
        const double2 colk = shfl2w(Dg[sk], (lane & ~3) | qk4);  // S[rl][k]
        double2 sc[2], ek[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          sc[h] = shfl2w(Dg[sk], (2 * t + h) * 4 + qk4);  // S[t + 4h][k]
          ek[h] = shfl2w(E[h], rk * 4 + t);               // E[k][t + 4h]
        }
        const double2 di = cinv(d);
        const double2 l = cmul(colk, di);
        const bool below = rl > k;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = t + 4 * h;
          if (below && c > k && rl >= c) Dg[h] = cfms(Dg[h], l, sc[h]);
          if (below) E[h] = cfms(E[h], l, ek[h]);
        }
        if (below && t == qk4) Dg[sk] = l;
        if (t == (k & 3)) dk[k >> 2] = d;
        if (rl == k) dinv_row = di;
        const double a2 = cabs2(d);
        minp = (a2 != a2 || minp < 0.0) ? -1.0 : fmin(minp, a2);
      }
    }
    // M = L11^-T D^-1 as B fragments: lane (g, t), slice s holds
    // M[t + 4s][rl] = L11^-1[rl][t + 4s] / d_rl (zero outside the w pivots)
    double Mr[2], Mi[2], nMi[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const bool ok = rl < w && t + 4 * s < w;
      const double2 v = ok ? cmul(E[s], dinv_row) : make_double2(0.0, 0.0);
      Mr[s] = v.x;
      Mi[s] = v.y;
      nMi[s] = -v.y;
    }
    // B fragments of the diagonal tile's Schur rows (partial block only):
    // L[rl][t + 4s] d_{t+4s} for t + 4s < w
    const bool partial = w < 8;
    double2 Bd[2];
#pragma unroll
    for (int s = 0; s < 2; ++s)
      Bd[s] = (partial && t + 4 * s < w) ? cmul(Dg[s], dk[s]) : make_double2(0.0, 0.0);
    // (b) panel tiles I >= 1: X = A M; columns >= w keep A and get the Schur
    //     update by the block's first w pivots
#pragma unroll
    for (int I = 1; I < MT; ++I) {
      if (I < nt) {
        double2(&A)[2] = S[tix(I, 0)];
        double xr[2] = {0.0, 0.0}, xi[2] = {0.0, 0.0};
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          dmma884(xr[0], xr[1], A[s].x, Mr[s]);
          dmma884(xr[0], xr[1], A[s].y, nMi[s]);
          dmma884(xi[0], xi[1], A[s].x, Mi[s]);
          dmma884(xi[0], xi[1], A[s].y, Mr[s]);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (t + 4 * h < w) A[h] = make_double2(xr[h], xi[h]);
        if (partial) {
          // A[:, w:] -= X[:, :w] (L[w:, :w] D)^T
          double zr[2] = {0.0, 0.0}, zi[2] = {0.0, 0.0};
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const bool ks = t + 4 * s < w;
            const double ar = ks ? A[s].x : 0.0, ai = ks ? A[s].y : 0.0;
            dmma884(zr[0], zr[1], ar, Bd[s].x);
            dmma884(zr[0], zr[1], -ai, Bd[s].y);
            dmma884(zi[0], zi[1], ar, Bd[s].y);
            dmma884(zi[0], zi[1], ai, Bd[s].x);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (t + 4 * h >= w) A[h] = make_double2(A[h].x - zr[h], A[h].y - zi[h]);
        }
      }
    }
    // (c) trailing tiles (I, J), 1 <= J <= I: S_IJ -= X_I (X_J D)^T, accumulated
    //     in place: re += Ar (-Br) + Ai Bi, im += Ar (-Bi) + Ai (-Br)
#pragma unroll
    for (int J = 1; J < MT; ++J) {
      if (J < nt) {
        double nBr[2], Bi[2], nBi[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const bool ks = t + 4 * s < w;
          const double2 bx = ks ? cmul(S[tix(J, 0)][s], dk[s]) : make_double2(0.0, 0.0);
          nBr[s] = -bx.x;
          Bi[s] = bx.y;
          nBi[s] = -bx.y;
        }
#pragma unroll
        for (int I = J; I < MT; ++I) {
          if (I < nt) {
            double2(&C)[2] = S[tix(I, J)];
            double cr[2] = {C[0].x, C[1].x}, ci[2] = {C[0].y, C[1].y};
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const bool ks = t + 4 * s < w;
              const double ar = ks ? S[tix(I, 0)][s].x : 0.0, ai = ks ? S[tix(I, 0)][s].y : 0.0;
              dmma884(cr[0], cr[1], ar, nBr[s]);
              dmma884(cr[0], cr[1], ai, Bi[s]);
              dmma884(ci[0], ci[1], ar, nBi[s]);
              dmma884(ci[0], ci[1], ai, nBr[s]);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) C[h] = make_double2(cr[h], ci[h]);
          }
        }
      }
    }
    col(kb, nt, w, dk, Mr, Mi);
    // (e) shift the trailing triangle to the origin
#pragma unroll
    for (int I = 1; I < MT; ++I)
#pragma unroll
      for (int J = 1; J <= I; ++J)
#pragma unroll
        for (int h = 0; h < 2; ++h) S[tix(I - 1, J - 1)][h] = S[tix(I, J)][h];
  }
  return kb;
}

#ifdef KH_PHASE_TIMING
// debug builds only (profiles/probes/phase_timing.py): clock64 cycles per phase
// of warp_front_kernel, summed over warps, [MT][phase], phase 7 = warp count
__device__ unsigned long long g_wphase[8 * 8];
#endif

template <int MT>
__global__ void __launch_bounds__(32 * WF_WARPS, (MT <= 5 ? 12 : 8) / WF_WARPS) warp_front_kernel(
    KhTree T, const int32_t* __restrict__ level_fronts, const double2* __restrict__ lam, double2* panels,
    double2* upd_cur, int64_t upd_stride_cur, const double2* __restrict__ upd_child, int64_t upd_stride_child,
    double* minpiv, const int32_t* __restrict__ wdst, int32_t nshift) {
  constexpr int NTL = MT * (MT + 1) / 2;
  extern __shared__ __align__(16) double2 O[];  // originals image: [panel tile][h][lane] = (M, A)
  __shared__ __align__(8) uint64_t wbar[WF_WARPS];  // per-warp child-staging barriers
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef KH_PHASE_TIMING
  long long tph = clock64();
  auto wphase = [&](int i) {
    if (lane == 0) {
      const long long t1 = clock64();
      atomicAdd(&g_wphase[MT * 8 + i], (unsigned long long)(t1 - tph));
      if (i == 0) atomicAdd(&g_wphase[MT * 8 + 7], 1ull);
      tph = t1;
    }
  };
#else
  auto wphase = [](int) {};
#endif
  if (tid < WF_WARPS) mbar_init(&wbar[tid], 1);
  mbar_fence_init();
  const int g = lane >> 2, t = lane & 3;
  const KhDevFront F = T.lf_fronts[(level_fronts - T.lf_base) + blockIdx.x];
  const int f = F.pad, p = F.p, q = F.q, m = p + q;
  const int M8 = (m + 7) >> 3, PJ = (p + 7) >> 3;
  KH_ASSERT(m <= 8 * MT);
  const int b = blockIdx.y * WF_WARPS + warp;
  const int nkids = F.child_end - F.child_begin;
  double2* cs = O + NTL * 64 + warp * WF_CHILD_MAX(MT);  // this warp's child buffer
  // the first child's update block starts streaming in right away
  auto stage_child = [&](int k) {
    const KhKid C = T.kids[F.child_begin + k];
    if (lane == 0 && C.q > 0) {
      // order earlier generic-proxy reads of the buffer before the async-proxy writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const uint32_t bytes = 8u * (uint32_t)(C.q * (C.q + 1));
      mbar_arrive_expect_tx(&wbar[warp], bytes);
      bulk_g2s(cs, upd_child + (int64_t)b * upd_stride_child + C.upd_off, bytes, &wbar[warp]);
    }
  };
  __syncthreads();  // barriers initialized
  if (b < nshift && nkids > 0) stage_child(0);
  // child maps for the pulls, per lane (shared by the CTA's shifts, built once
  // by warp k for child k < WF_KMAP): child-local row of each parent row the
  // lane holds and packed column base of each parent column; entries outside
  // the child get a huge sentinel so that the sum of the two lands past the
  // zero slot and min() routes it there (branch-free pulls; the upper entries
  // of diagonal tiles are don't-care and may receive any child entry)
  constexpr int SENT = 1 << 24;
  int32_t* kmap = reinterpret_cast<int32_t*>(O + NTL * 64 + WF_WARPS * WF_CHILD_MAX(MT));
  auto child_maps = [&](int k, int (&ri)[MT], int (&cbase)[MT][2]) {
    const KhKid C = T.kids[F.child_begin + k];
    const int32_t* __restrict__ cm = T.cmap + C.cmap_begin;
    const int rl_ = perm8(g);
#pragma unroll
    for (int I = 0; I < MT; ++I) {
      const int r = 8 * I + rl_;
      const int v = r < m ? __ldg(cm + r) : -1;
      ri[I] = v >= 0 ? v : SENT;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 8 * I + t + 4 * h;
        const int cj = c < m ? __ldg(cm + c) : -1;
        cbase[I][h] = cj >= 0 ? cj * (2 * C.q - cj - 1) / 2 : SENT;
      }
    }
  };
  if (warp < nkids && warp < WF_KMAP) {
    int ri[MT], cbase[MT][2];
    child_maps(warp, ri, cbase);
    int32_t* km = kmap + warp * 3 * MT * 32 + lane;
#pragma unroll
    for (int I = 0; I < MT; ++I) {
      km[(3 * I) * 32] = ri[I];
      km[(3 * I + 1) * 32] = cbase[I][0];
      km[(3 * I + 2) * 32] = cbase[I][1];
    }
  }
  // ---- originals image (shared by the CTA's shifts)
  const int ntile = PJ * M8 - PJ * (PJ - 1) / 2;
  for (int i = tid; i < ntile * 64; i += 32 * WF_WARPS) O[i] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int64_t e = F.orig_begin + tid; e < F.orig_end; e += 32 * WF_WARPS) {
    const int d = wdst[e];
    KH_ASSERT(d >= 0 && d < ntile * 64);
    O[d] = make_double2(T.om[e], T.oa[e]);
  }
  __syncthreads();
  if (b >= nshift) return;
  wphase(0);

  const int rl = perm8(g);  // logical row of this lane inside every 8-block
  double2 S[NTL][2];
  {
    const double2 L = lam[b];
#pragma unroll
    for (int I = 0; I < MT; ++I)
#pragma unroll
      for (int J = 0; J <= I; ++J)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double2 v = make_double2(0.0, 0.0);
          if (J < PJ && I < M8) {
            const double2 o = O[(J * M8 - J * (J - 1) / 2 + I - J) * 64 + h * 32 + lane];
            v = make_double2(fma(L.x, o.y, o.x), L.y * o.y);
          }
          S[tix(I, J)][h] = v;
        }
  }
  wphase(1);
  // ---- children: each child's packed update block (one contiguous array) is
  // staged in the warp's shared-memory buffer by one bulk async copy, then
  // pulled through the child maps
  uint32_t phase = 0;
  for (int k = 0; k < nkids; ++k) {
    const int qk = T.kids[F.child_begin + k].q;
    KH_ASSERT(qk <= 8 * MT);
    if (k > 0) {
      __syncwarp();  // the previous child's pulls are done
      stage_child(k);
    }
    int ri[MT], cbase[MT][2];
    if (k < WF_KMAP) {
      const int32_t* km = kmap + k * 3 * MT * 32 + lane;
#pragma unroll
      for (int I = 0; I < MT; ++I) {
        ri[I] = km[(3 * I) * 32];
        cbase[I][0] = km[(3 * I + 1) * 32];
        cbase[I][1] = km[(3 * I + 2) * 32];
      }
    } else {
      child_maps(k, ri, cbase);
    }
    const int zslot = qk * (qk + 1) / 2;  // a zero entry right after the child block
    if (lane == 0) cs[zslot] = make_double2(0.0, 0.0);
    if (qk > 0) {
      mbar_wait(&wbar[warp], phase);
      phase ^= 1u;
    }
    __syncwarp();
#pragma unroll
    for (int I = 0; I < MT; ++I)
#pragma unroll
      for (int J = 0; J <= I; ++J)
#pragma unroll
        for (int h = 0; h < 2; ++h) S[tix(I, J)][h] = cadd(S[tix(I, J)][h], cs[min(cbase[J][h] + ri[I], zslot)]);
  }

  wphase(2);
  // ---- blocked LDL^T over the p pivots (tile_ldlt); the finished tile columns
  // go to the panel, the Schur columns of a partial block to the staged update
  // block
  double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  double2* Uo = upd_cur + (int64_t)b * upd_stride_cur + F.upd_off;
  double minp = DBL_MAX;  // min |d|^2 (-1: non-finite pivot)
  const int kb = tile_ldlt<MT>(S, p, m, minp, [&](int kb, int nt, int, const double2 (&)[2], const double (&)[2],
                                              const double (&)[2]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = kb + t + 4 * h;
      double2* pc = P + (int64_t)c * m;
#pragma unroll
      for (int I = 0; I < MT; ++I) {
        const int r = kb + 8 * I + rl;
        if (I < nt && r < m && (I > 0 || rl >= t + 4 * h)) {
          if (c < p) pc[r] = S[tix(I, 0)][h];
          else cs[upk32(q, r - p, c - p)] = S[tix(I, 0)][h];  // update block: staged, see below
        }
      }
    }
  });
  wphase(3);
  // ---- the rest is the update block (rows and columns >= kb >= p)
#pragma unroll
  for (int I = 0; I < MT; ++I)
#pragma unroll
    for (int J = 0; J <= I; ++J)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = kb + 8 * I + rl, c = kb + 8 * J + t + 4 * h;
        if (r < m && r >= c) cs[upk32(q, r - p, c - p)] = S[tix(I, J)][h];
      }
  // the packed update block is contiguous in global memory: it was assembled
  // in the warp's (now free) child buffer and leaves with one bulk copy
  __syncwarp();
  if (lane == 0 && q > 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(Uo),
                 "r"(smem_u32(cs)), "r"(8u * (uint32_t)(q * (q + 1)))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  if (lane == 0) {
    minpiv[(int64_t)b * T.nf + f] = minp < 0.0 ? -1.0 : sqrt(minp);
    // shared memory must outlive the bulk copy's reads of it
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  wphase(4);
}

// Pivot block of a large front's super-block (see pivot_block_kernel in
// frontal.cu for the shared-memory version and panel_trsm_kernel for the
// consumer): one warp per (front, shift), four shifts per CTA. The w x w
// diagonal block at (c0, c0) of the assembled panel (w <= 8 MT) is loaded
// into registers in the permuted accumulator layout, factored by tile_ldlt,
// and written back (L with D on the diagonal) together with the block's DMMA
// B image: for tile pair (j, k < j) the lane's own L_jk values times d_k, for
// (j, j) the M_j fragments of the Gauss-Jordan inverse -- both are already in
// the B-fragment layout in registers, so the image costs one store per value.
template <int MT>
__global__ void __launch_bounds__(32 * WF_WARPS, 8 / WF_WARPS) pivot_warp_kernel(KhTree T, const int32_t* __restrict__ tasks,
                                                                     int c0, double2* panels, double* minpiv,
                                                                     double2* img, int64_t img_stride,
                                                                     int32_t nshift) {
  constexpr int NTL = MT * (MT + 1) / 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3, rl = perm8(g);
  const int32_t f = tasks[2 * blockIdx.x];
  const int64_t off = tasks[2 * blockIdx.x + 1];
  const int b = blockIdx.y * WF_WARPS + warp;
  if (b >= nshift) return;
  const KhDevFront F = T.fronts[f];
  const int mf = F.p + F.q, w = min(8 * MT, F.p - c0);
  double2* P = panels + (int64_t)b * T.panel_total + F.panel_off + c0 + (int64_t)c0 * mf;
  double2 S[NTL][2];
#pragma unroll
  for (int I = 0; I < MT; ++I)
#pragma unroll
    for (int J = 0; J <= I; ++J)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 8 * I + rl, c = 8 * J + t + 4 * h;
        S[tix(I, J)][h] = (r < w && r >= c) ? P[r + (int64_t)c * mf] : make_double2(0.0, 0.0);
      }
  double2* im = img + (int64_t)b * img_stride + off + lane;
  double minp = DBL_MAX;
  tile_ldlt<MT>(S, w, w, minp, [&](int kb, int nt, int wb, const double2 (&dk)[2], const double (&Mr)[2],
                                   const double (&Mi)[2]) {
    const int KB = kb >> 3;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = kb + t + 4 * h;
      double2* pc = P + (int64_t)c * mf;
#pragma unroll
      for (int I = 0; I < MT; ++I) {
        const int r = kb + 8 * I + rl;
        if (I < nt && r < w && c < w && (I > 0 || rl >= t + 4 * h)) pc[r] = S[tix(I, 0)][h];
      }
    }
#pragma unroll
    for (int I = 0; I < MT; ++I) {
      if (I < nt) {
        const int tp = (KB + I) * (KB + I + 1) / 2 + KB;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          double2 v = make_double2(0.0, 0.0);
          if (t + 4 * s < wb) v = I == 0 ? make_double2(Mr[s], Mi[s]) : cmul(S[tix(I, 0)][s], dk[s]);
          im[(tp * 2 + s) * 32] = v;
        }
      }
    }
  });
  if (lane == 0) {
    double* mp = minpiv + (int64_t)b * T.nf + f;
    const double v = minp < 0.0 ? -1.0 : sqrt(minp);
    *mp = c0 == 0 ? v : fmin(*mp, v);
  }
}

}  // namespace

#ifdef KH_PHASE_TIMING
extern "C" int kh_debug_wphase_cycles(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, g_wphase, sizeof(unsigned long long) * 64) != cudaSuccess) return 4;
  static const unsigned long long zero[64] = {};
  return cudaMemcpyToSymbol(g_wphase, zero, sizeof zero) == cudaSuccess ? 0 : 4;
}
#endif

// shared-memory bytes of the originals image for a front class
static int warp_front_smem(int mt) {
  return 16 * (64 * (mt * (mt + 1) / 2) + WF_WARPS * WF_CHILD_MAX(mt)) + 4 * WF_KMAP * 3 * mt * 32;
}

int kh_warp_front_slot(int32_t m, int32_t p, int32_t r, int32_t c) {
  // destination of the original entry (r, c), r >= c, c < p, in the image
  const int M8 = (m + 7) >> 3, I = r >> 3, J = c >> 3;
  const int pr = rho8(r & 7), pc = rho8(c & 7);
  const int lane = pr * 4 + (pc >> 1), h = pc & 1;
  (void)p;
  return (J * M8 - J * (J - 1) / 2 + I - J) * 64 + h * 32 + lane;
}

cudaError_t kh_launch_pivot_warp(const KhTree& T, const int32_t* tasks, int32_t ntasks, int c0, int32_t batch,
                                 double2* panels, double* minpiv, double2* img, int64_t img_stride,
                                 cudaStream_t stream) {
  if (ntasks == 0 || batch == 0) return cudaSuccess;
  const dim3 grid(ntasks, (batch + WF_WARPS - 1) / WF_WARPS);
  pivot_warp_kernel<6><<<grid, 32 * WF_WARPS, 0, stream>>>(T, tasks, c0, panels, minpiv, img, img_stride, batch);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_warp_front(int mt, const KhTree& T, const int32_t* level_fronts, int32_t nlev,
                                 int32_t batch, const double2* lam, double2* panels, double2* upd_cur,
                                 int64_t upd_stride_cur, const double2* upd_child, int64_t upd_stride_child,
                                 double* minpiv, const int32_t* wdst, cudaStream_t stream) {
  if (nlev == 0 || batch == 0) return cudaSuccess;
  const dim3 grid(nlev, (batch + WF_WARPS - 1) / WF_WARPS);
  auto run = [&](auto kernel) -> cudaError_t {
    const int smem = warp_front_smem(mt);
    cudaError_t e = kh_smem_optin((const void*)kernel, smem);
    if (e != cudaSuccess) return e;
    kernel<<<grid, 32 * WF_WARPS, smem, stream>>>(T, level_fronts, lam, panels, upd_cur, upd_stride_cur,
                                                   upd_child, upd_stride_child, minpiv, wdst, batch);
    kh_note_launch();
    return cudaGetLastError();
  };
  switch (mt) {
    case 4: return run(warp_front_kernel<4>);
    case 5: return run(warp_front_kernel<5>);
    case 6: return run(warp_front_kernel<6>);
    default: return cudaErrorInvalidValue;
  }
}
