// Batched multifrontal complex-symmetric LDL^T (pivot-free) and its
// triangular solves (the register-resident m <= 48 fronts: warpfront.cu).
//
// Replaces the reference's per-shift SuperLU path
//   K = (Mc + lam[k] Ac).tocsr(); sparse_direct.factorize(sym, K).solve(G[:,k])
// (solvers.py:383-393 -> sparse_direct.py:155-209). All shifts share one
// symbolic analysis (symbolic.cpp) and are processed level by level of the
// dissection tree, deepest level first; every launch covers all fronts of a
// level (of one size class) for all shifts of a batch: grid (#fronts, #shifts).
//
// Per front (m = p + q rows, p pivots):
//   panel P (m x p, column-major, ld m) in the retained factor storage,
//   update U (q x q lower, packed by columns: kh_upk) in a depth-parity buffer
//   consumed by the parent.
// Fronts with m <= 128 (factor_front_kernel): the whole front is assembled in
//   shared memory (packed block-column layout, push extend-add of the
//   children), factored by blocked_ldlt (8-pivot blocks, DMMA trailing
//   updates) and written out once (m <= 48: warp_front_kernel instead).
// Larger fronts (level-synchronous kernels): big_assemble (panel), then per
//   64-pivot super-block pivot_block / panel_trsm / panel_update, then
//   schur_update_kernel, which pulls the children's contributions into its
//   64 x 64 tiles of U in the epilogue.
// Every GEMM-shaped step runs on DMMA (mma.sync m8n8k4 f64); complex products
// use three real MMAs in the tile engine (KH_3M) and four elsewhere.
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace {

constexpr int NT = 256;      // threads per CTA
constexpr int TB = 64;       // complex tile edge
#ifndef KH_TILE_KC
#define KH_TILE_KC 8
#endif
constexpr int KC = KH_TILE_KC;  // complex K chunk of the tile engine
constexpr int LDS = TB + 2;  // padded smem row (double2): conflict-free LDS.128 fragments
constexpr int NB = 32;       // pivot block width

// Complex products in the tile engine: KH_3M = 1 forms each 8x8x4 complex
// block product with three real DMMAs (Gauss: T1 = (Ar+Ai) Br,
// T2 = Ar (Bi-Br), T3 = Ai (Br+Bi); re = T1 - T3, im = T1 + T2) instead of
// four: 25% less FP64 tensor work, one more accumulator set.
#ifndef KH_3M
#define KH_3M 1
#endif
struct Acc {
  double r[4][2][2];
  double i[4][2][2];
#if KH_3M
  double t[4][2][2];
#endif
};

// Visit the accumulator: ep(row, col, value) with row, col in [0, 64).
template <class EP>
KH_DEV void tile_epilogue(const Acc& acc, EP ep) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wi = warp & 1, wj = warp >> 1;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        ep(wi * 32 + mt * 8 + g, wj * 16 + nt * 8 + 2 * t + h,
           make_double2(acc.r[mt][nt][h], acc.i[mt][nt][h]));
}

// ---- pull assembly ------------------------------------------------------------
// A parent entry (r, c) (parent-local rows, r >= c) is the sum over children
// k of U_k[ci + cj*q_k] with ci = cmap_k[r], cj = cmap_k[c] when both are
// present. Gathering instead of scattering needs no zeroing pass and no
// read-modify-write, keeps many independent loads in flight, and fixes the
// summation order (bitwise-deterministic factors).
constexpr int MAXC = 8;  // children cached in shared memory; more are read from global

struct ChildRef {
  const double2* U;
  const int32_t* cmap;
  int q;
};

struct Kids {
  ChildRef c[MAXC];
  int n;
};

KH_DEV void load_kids(const KhTree& T, const KhDevFront& F, const double2* upd_child, int64_t stride_child, int b,
                      Kids& K) {
  if (threadIdx.x == 0) K.n = F.child_end - F.child_begin;
  if (threadIdx.x < MAXC && threadIdx.x < F.child_end - F.child_begin) {
    const KhDevFront C = T.fronts[T.child_list[F.child_begin + threadIdx.x]];
    K.c[threadIdx.x] = {upd_child + (int64_t)b * stride_child + C.upd_off, T.cmap + C.cmap_begin, C.q};
  }
}

KH_DEV ChildRef kid(const KhTree& T, const KhDevFront& F, const double2* upd_child, int64_t stride_child, int b,
                    const Kids& K, int k) {
  if (k < MAXC) return K.c[k];
  const KhDevFront C = T.fronts[T.child_list[F.child_begin + k]];
  return {upd_child + (int64_t)b * stride_child + C.upd_off, T.cmap + C.cmap_begin, C.q};
}

// One pipeline stage of the cp.async tile engine: 16 K-columns of A and B
// (64 rows each, [k][row] with the conflict-free pad) and the 16 pivots d_k.
struct CpStage {
  double2 a[KC * LDS];
  double2 b[KC * LDS];
  double2 d[KC];
};

// acc(i, j) = sum_{k<K} A[i + k*lda] * s_k * B(j, k)   (i < rowsA, j < rowsB)
// on a 64 x (16 NWJ) tile computed by 2 x NWJ warps (64 NWJ threads).
//  MODE_SCALED: B(j, k) = B[j + k*ldb], s_k = d_k = D[k*ldd] (the pivots on the
//               panel diagonal): Schur complements and left-looking updates.
// cp.async ring of CP_STAGES chunks: the next ones stream in while DMMA
// consumes the current one; out-of-range operands are zero-filled by the copy itself. The
// pivot scaling is applied to the B fragments in registers.
constexpr int MODE_SCALED = 0;
// cp.async ring depth of the tile engine (chunks in flight ahead of the one
// being consumed: KH_CP_STAGES - 1)
#ifndef KH_CP_STAGES
#define KH_CP_STAGES 4
#endif
constexpr int CP_STAGES = KH_CP_STAGES;

// KH_TILE_BULK = 1: the A and B columns of a chunk arrive by bulk async copies
// (one TMA-engine transfer per 64-row column segment, issued by one warp and
// counted on the stage's mbarrier) instead of per-thread 16-byte cp.async;
// rows past rowsA / rowsB are left unwritten (they only reach accumulator rows
// / columns the epilogues discard) and k-columns past K are zeroed. Measured
// at c3: factorization 27.36 ms vs 26.41 ms with cp.async (32 small copies per
// stage serialize in the SM's TMA unit), so the default stays cp.async.
#ifndef KH_TILE_BULK
#define KH_TILE_BULK 0
#endif

template <int NWJ, int MODE>
KH_DEV void tile_mma_cp(Acc& acc, int K, const double2* __restrict__ A, int64_t lda, int rowsA,
                        const double2* __restrict__ B, int64_t ldb, int rowsB, const double2* __restrict__ D,
                        int64_t ldd, CpStage* st, bool idle = false, uint64_t* bars = nullptr) {
  // idle: this warp's 32 x 16 sub-tile is not needed (above the diagonal or
  // past the last row/column); it still stages operands and joins barriers
  constexpr int NTH = 64 * NWJ, TN = 16 * NWJ;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wi = warp & 1, wj = warp >> 1;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        acc.r[a][b][h] = acc.i[a][b][h] = 0.0;
#if KH_3M
        acc.t[a][b][h] = 0.0;
#endif
      }
  const int nch = (K + KC - 1) / KC;
#if KH_TILE_BULK
  const int ra = min(rowsA, TB), rb = min(rowsB, TN);
  if (tid == 0)
    for (int s0 = 0; s0 < CP_STAGES; ++s0) mbar_init(&bars[s0], 1);
  mbar_fence_init();
  __syncthreads();
  auto load = [&](int s, int c) {
    CpStage& S = st[s];
    const int kv = min(KC, K - c * KC);  // valid k-columns of the chunk
    if (kv < KC) {                       // zero the columns past K (both operands)
      for (int e = tid; e < (KC - kv) * LDS; e += NTH) {
        S.a[kv * LDS + e] = make_double2(0.0, 0.0);
        S.b[kv * LDS + e] = make_double2(0.0, 0.0);
      }
    }
    if (warp == 0) {
      // the stage was last read through the generic proxy: order those reads
      // before the async-proxy writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (lane == 0) mbar_arrive_expect_tx(&bars[s], 16u * (uint32_t)(kv * (ra + rb)));
      __syncwarp();
      const int k = lane & (KC - 1);
      if (k < kv) {
        const int64_t kk = (int64_t)c * KC + k;
        if (lane < KC) bulk_g2s(&S.a[k * LDS], A + kk * lda, 16u * ra, &bars[s]);
        else bulk_g2s(&S.b[k * LDS], B + kk * ldb, 16u * rb, &bars[s]);
      }
    }
    if (MODE == MODE_SCALED && tid < KC) {
      const int kk = c * KC + tid;
      cp_async16(&S.d[tid], kk < K ? D + (int64_t)kk * ldd : D, kk < K);
    }
  };
#else
  auto load = [&](int s, int c) {
    CpStage& S = st[s];
#pragma unroll
    for (int r = 0; r < (TB * KC) / NTH; ++r) {
      const int idx = tid + r * NTH;
      const int i = idx & (TB - 1), k = idx >> 6;
      const int kk = c * KC + k;
      const bool oa = kk < K && i < rowsA;
      cp_async16(&S.a[k * LDS + i], oa ? A + i + (int64_t)kk * lda : A, oa);
    }
#pragma unroll
    for (int r = 0; r < (TN * KC) / NTH; ++r) {
      const int idx = tid + r * NTH;
      const int j = idx % TN, k = idx / TN;
      const int kk = c * KC + k;
      const bool ob = kk < K && j < rowsB;
      cp_async16(&S.b[k * LDS + j], ob ? B + j + (int64_t)kk * ldb : B, ob);
    }
    if (MODE == MODE_SCALED && tid < KC) {
      const int kk = c * KC + tid;
      cp_async16(&S.d[tid], kk < K ? D + (int64_t)kk * ldd : D, kk < K);
    }
  };
#endif
#pragma unroll
  for (int s0 = 0; s0 < CP_STAGES - 1; ++s0) {
    if (s0 < nch) load(s0, s0);
    cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    if (c + CP_STAGES - 1 < nch) load((c + CP_STAGES - 1) % CP_STAGES, c + CP_STAGES - 1);
    cp_async_commit();
    cp_async_wait<CP_STAGES - 1>();
#if KH_TILE_BULK
    mbar_wait(&bars[c % CP_STAGES], (uint32_t)((c / CP_STAGES) & 1));
#endif
    __syncthreads();
    const CpStage& S = st[c % CP_STAGES];
#pragma unroll
    for (int kk = 0; kk < (idle ? 0 : KC); kk += 4) {
      double2 af[4], bf[2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) af[mt] = S.a[(kk + t) * LDS + wi * 32 + mt * 8 + g];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        bf[nt] = S.b[(kk + t) * LDS + wj * 16 + nt * 8 + g];
        if (MODE == MODE_SCALED) bf[nt] = cmul(bf[nt], S.d[kk + t]);
      }
#if KH_3M
      double bs[2], bd[2];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        bs[nt] = bf[nt].x + bf[nt].y;
        bd[nt] = bf[nt].y - bf[nt].x;
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const double as = af[mt].x + af[mt].y;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          dmma884(acc.t[mt][nt][0], acc.t[mt][nt][1], as, bf[nt].x);
          dmma884(acc.i[mt][nt][0], acc.i[mt][nt][1], af[mt].x, bd[nt]);
          dmma884(acc.r[mt][nt][0], acc.r[mt][nt][1], af[mt].y, bs[nt]);
        }
      }
#else
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const double nai = -af[mt].y;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          dmma884(acc.r[mt][nt][0], acc.r[mt][nt][1], af[mt].x, bf[nt].x);
          dmma884(acc.r[mt][nt][0], acc.r[mt][nt][1], nai, bf[nt].y);
          dmma884(acc.i[mt][nt][0], acc.i[mt][nt][1], af[mt].x, bf[nt].y);
          dmma884(acc.i[mt][nt][0], acc.i[mt][nt][1], af[mt].y, bf[nt].x);
        }
      }
#endif
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#if KH_3M
  // re = T1 - T3, im = T1 + T2
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double t1 = acc.t[a][b][h];
        acc.r[a][b][h] = t1 - acc.r[a][b][h];
        acc.i[a][b][h] = t1 + acc.i[a][b][h];
      }
#endif
}

KH_DEV double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

KH_DEV double2 shfl_xor2(double2 v, int o) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, o), __shfl_xor_sync(0xffffffffu, v.y, o));
}

// Warp transpose-reduction of 8 values per lane: returns, on lane l, the sum
// over all 32 lanes of v[u] with u = 4*bit4(l) + 2*bit3(l) + bit2(l).
KH_DEV double2 warp_sum8(double2 (&v)[8], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double2 send = b4 ? v[j] : v[j + 4], keep = b4 ? v[j + 4] : v[j];
    v[j] = cadd(keep, shfl_xor2(send, 16));
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double2 send = b3 ? v[j] : v[j + 2], keep = b3 ? v[j + 2] : v[j];
    v[j] = cadd(keep, shfl_xor2(send, 8));
  }
  {
    const double2 send = b2 ? v[0] : v[1], keep = b2 ? v[1] : v[0];
    v[0] = cadd(keep, shfl_xor2(send, 4));
  }
  v[0] = cadd(v[0], shfl_xor2(v[0], 2));
  v[0] = cadd(v[0], shfl_xor2(v[0], 1));
  return v[0];
}

// Schur complement of the large fronts of one level: one CTA per 64 x 64
// lower tile of U, per shift: U[i0:, j0:] = C - L21[i0:, :] D L21[j0:, :]^T
// (K = p), where C is the children's extend-add onto the tile, pulled in the
// epilogue (the update block is written exactly once: no separate assembly
// pass over U and no read-modify-write). Tasks are (front, tile row, tile
// col) triples built on the host.
#ifndef KH_SCHUR_MINB
#define KH_SCHUR_MINB 2
#endif
__global__ void __launch_bounds__(NT, KH_SCHUR_MINB) schur_update_kernel(KhTree T, const int32_t* __restrict__ tasks,
                                                             const double2* __restrict__ panels, double2* upd_cur,
                                                             int64_t upd_stride_cur,
                                                             const double2* __restrict__ upd_child,
                                                             int64_t upd_stride_child) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CpStage* st = reinterpret_cast<CpStage*>(smem_raw);
  __shared__ Kids kids;
  const int32_t f = tasks[3 * blockIdx.x];
  const int i0 = tasks[3 * blockIdx.x + 1] * TB, j0 = tasks[3 * blockIdx.x + 2] * TB;
  const int b = blockIdx.y;
  const KhDevFront F = T.fronts[f];
  const int p = F.p, q = F.q, m = p + q;
  const double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  double2* U = upd_cur + (int64_t)b * upd_stride_cur + F.upd_off;
  load_kids(T, F, upd_child, upd_stride_child, b, kids);
  Acc acc;
  // warps whose 32 x 16 sub-tile lies strictly above the diagonal (diagonal
  // tiles) or beyond row/column q skip their MMAs
  const int wrp = threadIdx.x >> 5, r0w = i0 + (wrp & 1) * 32, c0w = j0 + (wrp >> 1) * 16;
  const bool idle = c0w > r0w + 31 || r0w >= q || c0w >= q;
  __shared__ __align__(8) uint64_t bars[CP_STAGES];
  tile_mma_cp<4, MODE_SCALED>(acc, p, P + p + i0, m, q - i0, P + p + j0, m, q - j0, P, m + 1, st, idle, bars);
  // epilogue: the product goes to shared memory (the operand ring is free:
  // tile_mma_cp ends on a barrier after its last chunk), then the CTA pulls the
  // children's extend-add column by column -- a warp covers 32 consecutive
  // rows of one tile column, so both the child reads (rows of a child column
  // stay in order under cmap) and the U writes are coalesced; children in
  // order (deterministic sums)
  double2* Ct = reinterpret_cast<double2*>(smem_raw);  // [64 columns][TB + 1]
  tile_epilogue(acc, [&](int i, int j, double2 v) { Ct[j * (TB + 1) + i] = v; });
  __syncthreads();  // kids visible even when p = 0; the product tile complete
  // packed column base of every tile column in every (cached) child, once per CTA
  __shared__ int cbs[MAXC][TB];
  const int nkc = min(kids.n, MAXC);
  for (int e = threadIdx.x; e < nkc * TB; e += NT) {
    const int k = e / TB, j = e - k * TB, c = j0 + j;
    const ChildRef C = kids.c[k];
    const int cj = c < q ? C.cmap[p + c] : -1;
    cbs[k][j] = cj >= 0 ? cj * (2 * C.q - cj - 1) / 2 : -1;
  }
  __syncthreads();
  // thread: tile row i (fixed), columns jb, jb + 4, ..., jb + 60, in two passes
  // of 8; children two at a time with all their loads issued before the adds
  // (which stay in child order: deterministic sums)
  const int i = threadIdx.x & (TB - 1), jb = threadIdx.x >> 6;
  const int r = i0 + i;
  if (r >= q) return;
  constexpr int HU = TB / 8;
  auto colbase = [&](int k, int j) -> int {
    if (k < MAXC) return cbs[k][j];
    const ChildRef C = kid(T, F, upd_child, upd_stride_child, b, kids, k);
    const int c = j0 + j, cj = c < q ? C.cmap[p + c] : -1;
    return cj >= 0 ? cj * (2 * C.q - cj - 1) / 2 : -1;
  };
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    double2 v[HU];
#pragma unroll
    for (int u = 0; u < HU; ++u) v[u] = make_double2(0.0, 0.0);
    for (int k = 0; k < kids.n; k += 2) {
      const ChildRef C0 = kid(T, F, upd_child, upd_stride_child, b, kids, k);
      const bool two = k + 1 < kids.n;
      const ChildRef C1 = two ? kid(T, F, upd_child, upd_stride_child, b, kids, k + 1) : C0;
      const int ci0 = C0.cmap[p + r], ci1 = two ? C1.cmap[p + r] : -1;
      double2 a0[HU], a1[HU];
#pragma unroll
      for (int u = 0; u < HU; ++u) {
        const int j = jb + 4 * (half * HU + u), c = j0 + j;
        const int b0 = ci0 >= 0 && c <= r ? colbase(k, j) : -1;
        const int b1 = ci1 >= 0 && c <= r ? colbase(k + 1, j) : -1;
        a0[u] = b0 >= 0 ? C0.U[b0 + ci0] : make_double2(0.0, 0.0);
        a1[u] = b1 >= 0 ? C1.U[b1 + ci1] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < HU; ++u) v[u] = cadd(cadd(v[u], a0[u]), a1[u]);
    }
#pragma unroll
    for (int u = 0; u < HU; ++u) {
      const int j = jb + 4 * (half * HU + u), c = j0 + j;
      if (c <= r) U[kh_upk32(q, r, c)] = csub(v[u], Ct[j * (TB + 1) + i]);
    }
  }
}

// ---- large fronts, level-synchronous batched kernels ------------------------------
// For the fronts with m > 128 of one level, the factorization is a sequence of
// launches, each covering every (front, shift) of the level at once:
//   big_assemble        (front, 512-entry chunk): P = pulled children + originals
//   for each 64-pivot super-block at column c0 (see pivot_block_kernel below):
//     pivot_block       (front, shift): LDL^T of the diagonal block + its DMMA B image
//     panel_trsm        (front, 64-row tile): rows below, X = A L^-T D^-1      (DMMA)
//     panel_update      (front, 64x64 tile): later pivot columns -= X D X^T   (DMMA)
//   schur_update        (front, 64x64 tile of U): U = pulled children - L21 D L21^T (DMMA)
// Tasks are int32 tuples prepared on the host per level and super-block.
constexpr int ASM_CHUNK = KH_ASM_CHUNK;

__global__ void __launch_bounds__(NT) big_assemble_kernel(KhTree T, const int32_t* __restrict__ tasks,
                                                          const double2* __restrict__ lam, double2* panels,
                                                          const double2* __restrict__ upd_child,
                                                          int64_t upd_stride_child) {
  // index space: the panel P (column-major m x p, lower part) in chunks of
  // ASM_CHUNK entries; the update block is assembled by schur_update_kernel
  __shared__ Kids kids;
  const int tid = threadIdx.x;
  const int32_t f = tasks[4 * blockIdx.x];
  const int idx0 = tasks[4 * blockIdx.x + 1];
  const int64_t olo = tasks[4 * blockIdx.x + 2], ohi = tasks[4 * blockIdx.x + 3];
  const int b = blockIdx.y;
  const KhDevFront F = T.fronts[f];
  const int p = F.p, m = p + F.q;
  const int total = min(m * p, idx0 + ASM_CHUNK);
  double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  load_kids(T, F, upd_child, upd_stride_child, b, kids);
  __syncthreads();
  int rr[ASM_CHUNK / NT], cc[ASM_CHUNK / NT];  // front-local row / column
  double2 v[ASM_CHUNK / NT];
#pragma unroll
  for (int u = 0; u < ASM_CHUNK / NT; ++u) {
    const int idx = idx0 + tid + u * NT;
    cc[u] = idx / m;
    rr[u] = idx - cc[u] * m;
    v[u] = make_double2(0.0, 0.0);
  }
  for (int k = 0; k < kids.n; ++k) {
    const ChildRef C = kid(T, F, upd_child, upd_stride_child, b, kids, k);
#pragma unroll
    for (int u = 0; u < ASM_CHUNK / NT; ++u) {
      if (idx0 + tid + u * NT < total && rr[u] >= cc[u]) {
        const int ci = C.cmap[rr[u]], cj = C.cmap[cc[u]];
        if (ci >= 0 && cj >= 0) v[u] = cadd(v[u], C.U[kh_upk32(C.q, ci, cj)]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < ASM_CHUNK / NT; ++u) {
    const int idx = idx0 + tid + u * NT;
    if (idx < total && rr[u] >= cc[u]) P[idx] = v[u];
  }
  __syncthreads();
  // originals whose (sorted) destinations fall into this chunk (range from the host)
  const double2 L = lam[b];
  for (int64_t e = olo + tid; e < ohi; e += NT) {
    const int d = T.orig_dst[e];
    const double av = T.oa[e];
    KH_ASSERT(d >= 0 && d < m * p);
    P[d] = cadd(P[d], make_double2(fma(L.x, av, T.om[e]), L.y * av));
  }
}

// Lower-triangle tile index -> (bi, bj), bj <= bi, tiles numbered row by row.
KH_DEV void tri_index(int t, int& bi, int& bj) {
  int i = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
  if ((i + 1) * (i + 2) / 2 <= t) ++i;
  if (i * (i + 1) / 2 > t) --i;
  bi = i;
  bj = t - i * (i + 1) / 2;
}

// Blocked LDL^T of the m x m lower matrix S over its first p pivots, by
// 32*NW threads, leaving the Schur complement C - L21 D L21^T in S[p:, p:].
// Entry (r, c), r >= c, lives at S[cb[c] + r] (cb: per-column base offsets in
// shared memory, so dense and packed block-column layouts share the code).
//  * pivots in blocks of 8: warp 0 factors the 8 x 8 diagonal block with
//    shuffles; the rows below are solved one thread per row; the rank-8
//    trailing update runs on DMMA;
//  * for a large update block (q >= kDeferSyrk) the rank-8 updates cover the
//    panel columns only and S[p:, p:] is computed once with K = p afterwards
//    (deferred SYRK: accumulate in registers over all pivots, one read-
//    modify-write per 8 x 8 tile) instead of p/8 rank-8 passes.
// W (8 rows of ldw), dinv (8) and dg (p pivots) are shared scratch. Returns the
// smallest |d| (or -1 for a non-finite pivot) on thread 0.
#ifdef KH_PHASE_TIMING
// debug builds only (profiles/probes/phase_timing.py): clock64 cycles per
// phase of factor_front_kernel, summed over CTAs, [MS/16][phase]
__device__ unsigned long long g_phase[9 * 8];
#endif

#ifndef KH_DEFER_SYRK
#define KH_DEFER_SYRK 48
#endif
constexpr int kDeferSyrk = KH_DEFER_SYRK;
#ifndef KH_BULK_WRITE
#define KH_BULK_WRITE 1
#endif
#ifndef KH_LOOKAHEAD_MIN_NW
#define KH_LOOKAHEAD_MIN_NW 16
#endif
// look-ahead pays off when the CTA has warps enough to hide the serial (a) phase
KH_HD constexpr bool kLookAhead(int nw) { return nw >= KH_LOOKAHEAD_MIN_NW; }

// LDL^T of the w x w diagonal block at column kb by warp 0 (lane i holds row
// i, pivots broadcast with shuffles): L in the strict lower part, D on the
// diagonal, 1/d in dinv and d in dg; minp tracks min |d|^2 (or -1).
KH_DEV void diag_block_ldlt(double2* S, const int32_t* cb, double2* dinv, double2* dg, int kb, int w, int m,
                            double& minp) {  // minp: running min |d|^2
  constexpr int BK = 8;
  const int lane = threadIdx.x & 31;
  int cbk[BK];
#pragma unroll
  for (int j = 0; j < BK; ++j) cbk[j] = cb[min(kb + j, m - 1)];
  double2 a[BK];
#pragma unroll
  for (int j = 0; j < BK; ++j) a[j] = (lane < w && j <= lane) ? S[cbk[j] + kb + lane] : make_double2(0.0, 0.0);
  // branch-free over k (w is uniform; inactive pivots use d = 1 and write
  // nothing), so the broadcasts of column k are issued together, ahead of
  // the reciprocal on the dependency chain
#pragma unroll
  for (int k = 0; k < BK; ++k) {
    const bool act = k < w;
    double2 col[BK];
#pragma unroll
    for (int j = k; j < BK; ++j) col[j] = shfl2(a[k], j);
    const double2 dk = act ? col[k] : make_double2(1.0, 0.0);
    const double2 di = cinv(dk);
    const double2 lik = cmul(a[k], di);
#pragma unroll
    for (int j = k + 1; j < BK; ++j)
      if (act && lane > k && j <= lane && lane < w) a[j] = cfms(a[j], lik, col[j]);
    if (act && lane > k && lane < w) a[k] = lik;
    if (act && lane == 0) {
      dinv[k] = di;
      dg[kb + k] = dk;
    }
  }
  // pivot magnitudes off the dependency chain: min |d|^2 (-1 if non-finite);
  // blocked_ldlt takes the square root once
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < BK; ++k)
      if (k < w) {
        const double a2 = cabs2(dg[kb + k]);
        minp = (a2 != a2 || minp < 0.0) ? -1.0 : fmin(minp, a2);
      }
#pragma unroll
  for (int j = 0; j < BK; ++j)
    if (lane < w && j <= lane) S[cbk[j] + kb + lane] = a[j];
}

// One 8 x 8 tile (rows r0.., cols c0..) of the rank-8 update
// S[r][c] -= sum_k L[r][kb+k] W[c][k] (c < cl, c <= r < m) on DMMA, by one warp.
// HW = false: no W buffer; the scaled operand L[c][kb+k] d_{kb+k} is formed
// from the stored L and the pivots dg (saves 8 x MS x 16 B of shared memory).
template <bool HW = true>
KH_DEV void rank8_tile(double2* S, const int32_t* cb, const double2* W, int ldw, const double2* dg, int kb, int w,
                       int r0, int c0, int cl, int m) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int ca = cb[min(kb + t, m - 1)], cb4 = cb[min(kb + t + 4, m - 1)];
  const int ra = r0 + g, cbv = c0 + g;
  double2 af[2], bf[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int k = 4 * s + t;
    af[s] = (k < w && ra < m) ? S[(s ? cb4 : ca) + ra] : make_double2(0.0, 0.0);
    if (HW) bf[s] = (cbv < cl) ? W[k * ldw + cbv] : make_double2(0.0, 0.0);
    else bf[s] = (cbv < cl && k < w) ? cmul(S[(s ? cb4 : ca) + cbv], dg[kb + k]) : make_double2(0.0, 0.0);
  }
  // four independent accumulators (re*re, -im*im, re*im, im*re): MMA chains
  // of depth 2 instead of 4
  double rr[2] = {0.0, 0.0}, ii[2] = {0.0, 0.0}, ri[2] = {0.0, 0.0}, ir[2] = {0.0, 0.0};
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    dmma884(rr[0], rr[1], af[s].x, bf[s].x);
    dmma884(ii[0], ii[1], -af[s].y, bf[s].y);
    dmma884(ri[0], ri[1], af[s].x, bf[s].y);
    dmma884(ir[0], ir[1], af[s].y, bf[s].x);
  }
  const int row = r0 + g;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int cc = c0 + 2 * t + h;
    if (row < m && cc < cl && row >= cc) {
      double2* d = S + cb[cc] + row;
      *d = make_double2(d->x - (rr[h] + ii[h]), d->y - (ri[h] + ir[h]));
    }
  }
}

// Blocked LDL^T of the m x m lower matrix S over its first p pivots, by
// 32*NW threads, leaving the Schur complement C - L21 D L21^T in S[p:, p:].
// Entry (r, c), r >= c, lives at S[cb[c] + r] (cb: per-column base offsets in
// shared memory, so dense and packed block-column layouts share the code).
// Pivots go in blocks of 8:
//  (a) warp 0 factors the 8 x 8 diagonal block with shuffles;
//  (b) the rows below are solved one thread per row (W = L D of the block);
//  (c) rank-8 trailing update on DMMA, 8 x 8 tiles handed out through a
//      shared counter. Look-ahead: warp 0 first updates the next block's
//      diagonal tile and factors it (the next (a)) while the other warps work
//      through the remaining tiles, then joins them; the serial (a) chain is
//      thus hidden behind the update instead of idling the CTA.
// For a large update block (q >= kDeferSyrk) the rank-8 updates cover the
// panel columns only and S[p:, p:] is computed once with K = p at the end
// (deferred SYRK: one read-modify-write per tile instead of p/8).
// W (8 rows of ldw), dinv (8), dg (p pivots) and ctr (1 int) are shared
// scratch. Returns the smallest |d| (or -1 for a non-finite pivot) on thread 0.
template <int NW, bool LA, int TSLOT = 0, bool HW = true>
KH_DEV double blocked_ldlt(double2* S, const int32_t* cb, double2* W, int ldw, double2* dinv, double2* dg,
                           int* ctr, int m, int p) {
  constexpr int NTH = 32 * NW, BK = 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef KH_PHASE_TIMING
  long long ts0 = clock64();
  auto sub = [&](int i) {  // sub-phases 4 (a), 5 (b), 6 (c + SYRK) of the fused kernel
    if (TSLOT > 0 && tid == 0) {
      const long long t1 = clock64();
      atomicAdd(&g_phase[TSLOT * 8 + i], (unsigned long long)(t1 - ts0));
      ts0 = t1;
    }
  };
#else
  auto sub = [](int) {};
#endif
  const int g = lane >> 2, t = lane & 3;
  const bool defer = m - p >= kDeferSyrk;
  const int cl = defer ? p : m;  // columns updated inside the pivot loop
  double minp = DBL_MAX;
  if (LA) {
    if (p > 0 && warp == 0) diag_block_ldlt(S, cb, dinv, dg, 0, min(BK, p), m, minp);
    __syncthreads();
  }
  for (int kb = 0; kb < p; kb += BK) {
    const int w = min(BK, p - kb);
    if (!LA) {
      if (warp == 0) diag_block_ldlt(S, cb, dinv, dg, kb, w, m, minp);
      __syncthreads();
      sub(4);
    }
    // (b) rows below: v_j = a_rj - sum_{k<j} v_k L[kb+j][kb+k]; L[r][kb+j] = v_j / d_j
    const int s0 = kb + w;
    {
      int cbk[BK];
#pragma unroll
      for (int j = 0; j < BK; ++j) cbk[j] = cb[min(kb + j, m - 1)];
      for (int r = s0 + tid; r < m; r += NTH) {
        double2 v[BK];
#pragma unroll
        for (int j = 0; j < BK; ++j) v[j] = j < w ? S[cbk[j] + r] : make_double2(0.0, 0.0);
        // column-oriented (same subtraction order as the row form, depth BK)
#pragma unroll
        for (int j = 0; j < BK - 1; ++j)
#pragma unroll
          for (int i = j + 1; i < BK; ++i)
            if (i < w) v[i] = cfms(v[i], v[j], S[cbk[j] + kb + i]);
#pragma unroll
        for (int j = 0; j < BK; ++j) {
          if (j < w) {
            if (HW) W[j * ldw + r] = v[j];
            S[cbk[j] + r] = cmul(v[j], dinv[j]);
          } else if (HW) {
            W[j * ldw + r] = make_double2(0.0, 0.0);
          }
        }
      }
    }
    if (tid == 0) *ctr = 0;
    __syncthreads();
    sub(5);
    // (c) tiles (bi, bj), bj <= bi, of rows s0..m-1 x columns s0..cl-1,
    //     enumerated column block by column block; tile 0 is the next
    //     diagonal block
    if (!LA) {
      if (s0 < cl) {
        // tiles task = warp, warp + NW, ...: (bj, rem) advanced incrementally
        const int nrb = (m - s0 + 7) / 8, ncb = (cl - s0 + 7) / 8;
        int bj = 0, rem = warp;
        while (bj < ncb && rem >= nrb - bj) rem -= nrb - bj++;
        while (bj < ncb) {
          rank8_tile<HW>(S, cb, W, ldw, dg, kb, w, s0 + 8 * (bj + rem), s0 + 8 * bj, cl, m);
          rem += NW;
          while (bj < ncb && rem >= nrb - bj) rem -= nrb - bj++;
        }
      }
    } else if (s0 < cl) {
      const int nrb = (m - s0 + 7) / 8, ncb = (cl - s0 + 7) / 8;
      int first = 0;
      if (warp == 0 && s0 < p) {  // look-ahead
        rank8_tile<HW>(S, cb, W, ldw, dg, kb, w, s0, s0, cl, m);
        __syncwarp();
        diag_block_ldlt(S, cb, dinv, dg, s0, min(BK, p - s0), m, minp);
      }
      if (s0 < p) first = 1;
      for (;;) {
        int task = 0;
        if (lane == 0) task = atomicAdd(ctr, 1) + first;
        task = __shfl_sync(0xffffffffu, task, 0);
        int bj = 0, rem = task;
        while (bj < ncb && rem >= nrb - bj) rem -= nrb - bj++;
        if (bj >= ncb) break;
        rank8_tile<HW>(S, cb, W, ldw, dg, kb, w, s0 + 8 * (bj + rem), s0 + 8 * bj, cl, m);
      }
    }
    __syncthreads();
    sub(6);
  }
  // deferred SYRK: S[p:, p:] -= L21 D L21^T, K = p, one RMW per 8 x 8 tile
  const int q = m - p;
  if (defer && p > 0) {
    const int nb = (q + 7) / 8;
    for (int task = warp; task < nb * (nb + 1) / 2; task += NW) {
      int bi, bj;
      tri_index(task, bi, bj);
      const int r0 = p + 8 * bi, c0 = p + 8 * bj;
      const int ra = r0 + g, cv = c0 + g;
      // Gauss 3M form (see KH_3M): T1 = (Ar+Ai) Br, T2 = Ar (Bi-Br),
      // T3 = Ai (Br+Bi); re = T1 - T3, im = T1 + T2 -- three independent
      // accumulator chains
      double t1[2] = {0.0, 0.0}, t2[2] = {0.0, 0.0}, t3[2] = {0.0, 0.0};
#pragma unroll 2
      for (int ks = 0; ks < p; ks += 4) {
        const int k = ks + t;
        double2 af = make_double2(0.0, 0.0), bf = make_double2(0.0, 0.0);
        if (k < p) {
          const int ck = cb[k];
          if (ra < m) af = S[ck + ra];
          if (cv < m) bf = cmul(S[ck + cv], dg[k]);
        }
        dmma884(t1[0], t1[1], af.x + af.y, bf.x);
        dmma884(t2[0], t2[1], af.x, bf.y - bf.x);
        dmma884(t3[0], t3[1], af.y, bf.x + bf.y);
      }
      const int rr = r0 + g;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cc = c0 + 2 * t + h;
        if (rr < m && cc < m && rr >= cc) {
          double2* d = S + cb[cc] + rr;
          *d = make_double2(d->x - (t1[h] - t3[h]), d->y - (t1[h] + t2[h]));
        }
      }
    }
    __syncthreads();
    sub(6);
  }
  return minp < 0.0 ? -1.0 : sqrt(minp);  // min |d|
}

// ---- large fronts with p <= PIV_MAX: two launches for the whole panel ----------
// Instead of lupdate / diag / trsm per 32-pivot block:
//   pivot_block_kernel (front, shift): the p x p pivot block of the assembled
//     panel is loaded into shared memory, factored by blocked_ldlt (8-pivot
//     blocks, DMMA trailing updates) and written back; it also writes the
//     block's "B image": for every 8 x 8 tile pair (j, k), k < j, of L11 the
//     DMMA B fragments of D_k L_jk^T, and for k = j those of
//     M_j = L_jj^-T D_j^-1 (from the 8 x 8 unit-lower inverse), in lane order;
//   panel_trsm_kernel (front, 64-row tile of L21, shift): a warp per 8 rows
//     solves X = A21 L11^-T D^-1 by blocks of 8 columns,
//     X_j = (A_j - sum_{k<j} X_k D_k L_jk^T) M_j, on DMMA with its rows held in
//     registers in the permuted accumulator layout of warpfront.cu (lane
//     (g, t) holds logical rows pi(g), columns t and t + 4 of every tile, so
//     a finished X_k is directly an A fragment) and the B image staged in
//     shared memory by one bulk copy.
#ifndef KH_PIV_NW
#define KH_PIV_NW 4
#endif
constexpr int PIV_MAX = 64, PIV_NW = KH_PIV_NW, PIV_LD = PIV_MAX + 2, PIV_PT = PIV_MAX / 8;
constexpr int PIV_IMG = 64 * PIV_PT * (PIV_PT + 1) / 2;  // B image entries (double2) at p = PIV_MAX
KH_HD constexpr int piv_smem_bytes() { return 16 * (kh_packed_elems(PIV_MAX) + 8 * PIV_LD + 8 + PIV_MAX + 64 * PIV_PT) + 4 * PIV_MAX; }
KH_DEV int piv_perm8(int g) { return (g >> 1) + 4 * (g & 1); }  // phys -> logical inside an 8-block
KH_HD constexpr int piv_tp(int j, int k) { return j * (j + 1) / 2 + k; }

__global__ void __launch_bounds__(32 * PIV_NW) pivot_block_kernel(KhTree T, const int32_t* __restrict__ tasks,
                                                                  int c0, double2* panels, double* minpiv,
                                                                  double2* img, int64_t img_stride) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* S = reinterpret_cast<double2*>(smem_raw);  // packed p x p (L11, D)
  double2* W = S + kh_packed_elems(PIV_MAX);
  double2* dinv = W + 8 * PIV_LD;
  double2* dg = dinv + 8;
  double2* Ld = dg + PIV_MAX;  // inverses of the diagonal 8 x 8 blocks: Ld[j][i][c] = L_jj^-1[i][c]
  int32_t* cb = reinterpret_cast<int32_t*>(Ld + 64 * PIV_PT);
  __shared__ int ctr;
  constexpr int NTH = 32 * PIV_NW;
  const int tid = threadIdx.x;
  const int32_t f = tasks[2 * blockIdx.x];
  const int64_t off = tasks[2 * blockIdx.x + 1];
  const int b = blockIdx.y;
  const KhDevFront F = T.fronts[f];
  const int m = F.p + F.q;
  const int p = min(PIV_MAX, F.p - c0), PT = (p + 7) >> 3;  // this super-block's pivots
  // the super-block's diagonal block at (c0, c0): P[r + c m] below is entry (c0 + r, c0 + c)
  double2* P = panels + (int64_t)b * T.panel_total + F.panel_off + c0 + (int64_t)c0 * m;
  for (int c = tid; c < p; c += NTH) cb[c] = kh_packed_col_base(p, c);
  __syncthreads();
  for (int e = tid; e < p * p; e += NTH) {
    const int c = e / p, r = e - c * p;
    if (r >= c) S[cb[c] + r] = P[r + (int64_t)c * m];
  }
  __syncthreads();
  const double minp = blocked_ldlt<PIV_NW, kLookAhead(PIV_NW)>(S, cb, W, PIV_LD, dinv, dg, &ctr, p, p);
  for (int e = tid; e < p * p; e += NTH) {
    const int c = e / p, r = e - c * p;
    if (r >= c) P[r + (int64_t)c * m] = S[cb[c] + r];
  }
  // unit-lower inverses of the diagonal blocks, thread per (block, column)
  for (int e = tid; e < 8 * PT; e += NTH) {
    const int j = e >> 3, c = e & 7, base = 8 * j;
    double2 y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) y[i] = make_double2(i == c ? 1.0 : 0.0, 0.0);
#pragma unroll
    for (int i = 1; i < 8; ++i) {
      if (i > c && base + i < p) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < i; ++k)
          if (k >= c) acc = cfms(acc, S[cb[base + k] + base + i], y[k]);
        y[i] = acc;
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) Ld[j * 64 + i * 8 + c] = y[i];
  }
  __syncthreads();
  // B image: tile pair (j, k), slice s, lane (g, t) at [(tp * 2 + s) * 32 + lane]
  double2* im = img + (int64_t)b * img_stride + off;
  const int ntp = PT * (PT + 1) / 2;
  for (int e = tid; e < ntp * 64; e += NTH) {
    const int tp = e >> 6, s = (e >> 5) & 1, lane = e & 31;
    int j = 0;
    while (piv_tp(j + 1, 0) <= tp) ++j;
    const int k = tp - piv_tp(j, 0);
    const int g = lane >> 2, t = lane & 3;
    const int n = piv_perm8(g), kk = t + 4 * s;  // logical row of block j / column of block k
    const int rn = 8 * j + n, ck = 8 * k + kk;
    double2 v = make_double2(0.0, 0.0);
    if (rn < p && ck < p) {
      if (k < j) v = cmul(S[cb[ck] + rn], dg[ck]);                                    // d_k L_jk[n][kk]
      else if (kk <= n) v = cmul(Ld[j * 64 + n * 8 + kk], cinv(dg[rn]));             // L_jj^-1[n][kk] / d_n
    }
    im[e] = v;
  }
  if (tid == 0) {
    double* mp = minpiv + (int64_t)b * T.nf + f;
    *mp = c0 == 0 ? minp : fmin(*mp, minp);
  }
}

constexpr int PTR_NW = 8;  // warps (8-row slabs) per panel_trsm CTA
__global__ void __launch_bounds__(32 * PTR_NW) panel_trsm_kernel(KhTree T, const int32_t* __restrict__ tasks,
                                                                 int c0, double2* panels,
                                                                 const double2* __restrict__ img, int64_t img_stride) {
  __shared__ __align__(16) double2 Bs[PIV_IMG];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int32_t f = tasks[3 * blockIdx.x];
  const int i0 = tasks[3 * blockIdx.x + 1];
  const int64_t off = tasks[3 * blockIdx.x + 2];
  const int b = blockIdx.y;
  const KhDevFront F = T.fronts[f];
  const int m = F.p + F.q;
  const int p = min(kh_piv_max(), F.p - c0), PT = (p + 7) >> 3;  // this super-block's pivots
  // columns c0 .. c0 + p of the panel (rows keep their front numbering)
  double2* P = panels + (int64_t)b * T.panel_total + F.panel_off + (int64_t)c0 * m;
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    const uint32_t bytes = 16u * 64u * (uint32_t)(PT * (PT + 1) / 2);
    mbar_arrive_expect_tx(&bar, bytes);
    bulk_g2s(Bs, img + (int64_t)b * img_stride + off, bytes, &bar);
  }
  // this warp's 8 rows of A21, all p columns, in the permuted accumulator layout
  const int r = i0 + 8 * warp + piv_perm8(g);
  double2 a[PIV_PT][2];
#pragma unroll
  for (int j = 0; j < PIV_PT; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = 8 * j + t + 4 * h;
      a[j][h] = (j < PT && r < m && c < p) ? P[r + (int64_t)c * m] : make_double2(0.0, 0.0);
    }
  __syncthreads();  // barrier initialized before anyone waits on it
  mbar_wait(&bar, 0);
  if (i0 + 8 * warp >= m) return;
  const double2* B2 = Bs + lane;
#pragma unroll
  for (int j = 0; j < PIV_PT; ++j) {
    if (j < PT) {
      double cr[2] = {a[j][0].x, a[j][1].x}, ci[2] = {a[j][0].y, a[j][1].y};
      // A_j - sum_{k<j} X_k (D_k L_jk^T): re += Ar (-Br) + Ai Bi, im += Ar (-Bi) + Ai (-Br)
#pragma unroll
      for (int k = 0; k < j; ++k) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const double2 bv = B2[(piv_tp(j, k) * 2 + s) * 32];
          dmma884(cr[0], cr[1], a[k][s].x, -bv.x);
          dmma884(cr[0], cr[1], a[k][s].y, bv.y);
          dmma884(ci[0], ci[1], a[k][s].x, -bv.y);
          dmma884(ci[0], ci[1], a[k][s].y, -bv.x);
        }
      }
      // X_j = (.) M_j
      double xr[2] = {0.0, 0.0}, xi[2] = {0.0, 0.0};
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const double2 mv = B2[(piv_tp(j, j) * 2 + s) * 32];
        dmma884(xr[0], xr[1], cr[s], mv.x);
        dmma884(xr[0], xr[1], ci[s], -mv.y);
        dmma884(xi[0], xi[1], cr[s], mv.y);
        dmma884(xi[0], xi[1], ci[s], mv.x);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) a[j][h] = make_double2(xr[h], xi[h]);
    }
  }
  if (r < m) {
#pragma unroll
    for (int j = 0; j < PIV_PT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 8 * j + t + 4 * h;
        if (j < PT && c < p) P[r + (int64_t)c * m] = a[j][h];
      }
  }
}

// Right-looking update of the pivot columns after a super-block: for the 64 x 64
// tile (i0, j0) of the panel (j0 >= c0 + 64, rows i0.. >= j0, columns j0..< p),
// P[r][c] -= sum_{c0 <= k < c0 + 64} L[r][k] d_k L[c][k].
__global__ void __launch_bounds__(NT, KH_SCHUR_MINB) panel_update_kernel(KhTree T, const int32_t* __restrict__ tasks,
                                                                        int c0, double2* panels) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CpStage* st = reinterpret_cast<CpStage*>(smem_raw);
  const int32_t f = tasks[3 * blockIdx.x];
  const int i0 = tasks[3 * blockIdx.x + 1], j0 = tasks[3 * blockIdx.x + 2];
  const int b = blockIdx.y;
  const KhDevFront F = T.fronts[f];
  const int p = F.p, m = p + F.q;
  double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  const int wrp = threadIdx.x >> 5, r0w = i0 + (wrp & 1) * 32, c0w = j0 + (wrp >> 1) * 16;
  const bool idle = c0w > r0w + 31 || r0w >= m || c0w >= p;
  Acc acc;
  __shared__ __align__(8) uint64_t bars[CP_STAGES];
  const int64_t kc = (int64_t)c0 * m;
  tile_mma_cp<4, MODE_SCALED>(acc, kh_piv_max(), P + i0 + kc, m, m - i0, P + j0 + kc, m, p - j0, P + c0 + kc, m + 1, st,
                              idle, bars);
  tile_epilogue(acc, [&](int i, int j, double2 v) {
    const int r = i0 + i, c = j0 + j;
    if (r < m && c < p && r >= c) {
      double2* d = P + r + (int64_t)c * m;
      *d = csub(*d, v);
    }
  });
}

// ---- fused fronts (m <= MS): assemble + factor + Schur complement in one CTA ----
// The front's lower triangle lives in shared memory in the packed block-column
// layout of kernels.h (a 128-row front needs 140 KB instead of 260 KB). The
// whole LDL^T, including the update matrix U = C - L21 D L21^T, is done by
// blocked_ldlt; the panel and U are then written once, coalesced.
KH_HD constexpr int packed_elems(int m) { return kh_packed_elems(m); }
// classes whose residency is bounded by shared memory drop the W buffer
#ifndef KH_NOW_64
#define KH_NOW_64 0
#endif
KH_HD constexpr bool front_has_w(int ms) { return ms != 48 && !(KH_NOW_64 && ms == 64); }
KH_HD constexpr int front_smem_bytes(int ms) {
  return 16 * (packed_elems(ms) + (front_has_w(ms) ? 8 * (ms + 2) : 0) + 8 + 2 * ms) + 4 * ms + 4 * 4 * ms;
}

// the fourth fused class (m <= KH_CLASS4, between 64 and 128)
#ifndef KH_CLASS4
#define KH_CLASS4 96
#endif
// warps per CTA of the fused classes m <= 64, KH_CLASS4, 128
#ifndef KH_NW32
#define KH_NW32 2
#endif
#ifndef KH_NW48
#define KH_NW48 2
#endif
#ifndef KH_NW64
#define KH_NW64 4
#endif
#ifndef KH_NW96
#define KH_NW96 8
#endif
#ifndef KH_NW128
#define KH_NW128 16
#endif
#ifndef KH_F32_MINB
#define KH_F32_MINB 10
#endif
// resident CTAs per SM the register allocation must allow
KH_HD constexpr int front_min_blocks(int ms, int nw) {
  return ms <= 32 ? KH_F32_MINB : ((16 / nw) > 1 ? 16 / nw : 1);
}

// FWD: fused forward solve. The front's right-hand side (y of the pivot
// rows + the children's rhs updates, pushed in child order during the
// assembly) is kept in shared memory; after the LDL^T, warp 0 runs the
// forward sweep x_r -= L[r][k] x_k on the shared-memory panel (lanes own rows,
// pivots broadcast by shuffles; same operation order as fwd_small_kernel)
// while the other warps write the panel and the update block out. y and the
// parent's rhs update are then written like fwd_small_kernel would.
struct FwdArgs {
  double2* y;
  double2* ru_cur;
  int64_t ru_stride_cur;
  const double2* ru_child;
  int64_t ru_stride_child;
};

// child-update columns a warp loads per batch in the push assembly
#ifndef KH_ASM_CW
#define KH_ASM_CW 0
#endif
KH_HD constexpr int asm_cols(int ms) {
  return KH_ASM_CW > 0 ? KH_ASM_CW : (ms <= 32 ? 8 : ms <= 48 ? 6 : ms <= 64 ? 4 : ms <= 96 ? 4 : 2);
}

template <int MS, int NW, bool FWD>
__global__ void __launch_bounds__(32 * NW, front_min_blocks(MS, NW)) factor_front_kernel(
    KhTree T, const int32_t* __restrict__ level_fronts, const double2* __restrict__ lam, double2* panels,
    double2* upd_cur, int64_t upd_stride_cur, const double2* __restrict__ upd_child, int64_t upd_stride_child,
    double* minpiv, FwdArgs fw) {
  constexpr int NTH = 32 * NW, LDW = MS + 2, RK = 4;  // RK: children whose relind maps are staged
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* S = reinterpret_cast<double2*>(smem_raw);  // packed lower triangle (m + 1 rows)
  double2* W = S + packed_elems(MS);                  // W[k*LDW + r] = L[r][kb+k] d_{kb+k}
  double2* dinv = W + (front_has_w(MS) ? 8 * LDW : 0);  // 1/d of the current block
  double2* dg = dinv + 8;                              // pivots d_k
  double2* xs = dg + MS;                               // front rhs / forward-solved x (FWD)
  int32_t* cb = reinterpret_cast<int32_t*>(xs + MS);   // column bases
  int32_t* rel = cb + MS;                              // rel[k*MS + i]
  __shared__ int ctr;
  const int tid = threadIdx.x;
#ifdef KH_PHASE_TIMING
  long long t_0 = clock64();
  auto phase = [&](int i) {
    if (tid == 0) {
      const long long t1 = clock64();
      atomicAdd(&g_phase[(MS / 16) * 8 + i], (unsigned long long)(t1 - t_0));
      if (i == 0) atomicAdd(&g_phase[(MS / 16) * 8 + 7], 1ull);
      t_0 = t1;
    }
  };
#else
  auto phase = [](int) {};
#endif
  const int lane = tid & 31, warp = tid >> 5;
  const KhDevFront F = T.lf_fronts[(level_fronts - T.lf_base) + blockIdx.x];
  const int32_t f = F.pad;
  const int b = blockIdx.y;
  const int p = F.p, q = F.q, m = p + q;
  double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  double2* U = upd_cur + (int64_t)b * upd_stride_cur + F.upd_off;
  const int nkids = F.child_end - F.child_begin;
  __shared__ KhKid kinfo[RK];

  // ---- assembly: zero the front, add the originals (values pre-gathered in
  // front order, destinations pre-packed on the host: one coalesced stream),
  // then push each child's update block through its relind map (coalesced
  // column reads of the child's U, conflict-free within a child; children in
  // order, so the sums are deterministic)
  if (tid < RK && tid < nkids) kinfo[tid] = T.kids[F.child_begin + tid];
  const int ne = packed_elems(m);
  KH_ASSERT(m <= MS && ne <= packed_elems(MS));
  for (int idx = tid; idx < ne; idx += NTH) S[idx] = make_double2(0.0, 0.0);
  for (int c = tid; c < m; c += NTH) cb[c] = kh_packed_col_base(m, c);
  // FWD: the pivot rows' rhs, loaded now and stored to xs after the assembly
  // (the loads are in flight during it)
  constexpr int RY = (MS + NTH - 1) / NTH;
  double2 yreg[FWD ? RY : 1];
  if (FWD) {
    const double2* yb = fw.y + (int64_t)b * T.n + F.first;
#pragma unroll
    for (int u = 0; u < RY; ++u) {
      const int c = tid + u * NTH;
      yreg[u] = c < p ? yb[c] : make_double2(0.0, 0.0);
    }
  }
  __syncthreads();
  phase(0);
  // warm L2 with the children's update blocks (read after the originals)
  for (int k = 0; k < nkids && k < RK; ++k) {
    const char* base = reinterpret_cast<const char*>(upd_child + (int64_t)b * upd_stride_child + kinfo[k].upd_off);
    const int lines = (kinfo[k].q * (kinfo[k].q + 1) * 8 + 127) >> 7;
    for (int l = tid; l < lines; l += NTH) asm volatile("prefetch.global.L2 [%0];" ::"l"(base + 128 * l));
  }
  for (int idx = tid; idx < RK * MS; idx += NTH) {
    const int k = idx / MS, i = idx - k * MS;
    if (k < nkids && i < kinfo[k].q) rel[idx] = T.relind[kinfo[k].rows_begin + i];
  }
  {
    const double2 Lm = lam[b];
    for (int64_t e = F.orig_begin + tid; e < F.orig_end; e += NTH) {
      const int d = T.orig_dst[e];
      const double av = T.oa[e];
      KH_ASSERT(d >= 0 && d < ne);
      S[d] = cadd(S[d], make_double2(fma(Lm.x, av, T.om[e]), Lm.y * av));
    }
  }
  constexpr int R = (MS + 31) / 32;  // row passes per column
  for (int k = 0; k < nkids; ++k) {
    __syncthreads();
    if (FWD && k == 0) {
#pragma unroll
      for (int u = 0; u < RY; ++u) {
        const int c = tid + u * NTH;
        if (c < m) xs[c] = yreg[u];
      }
      __syncthreads();
    }
    int64_t upd_off, rows_begin, roff = 0;
    int qk;
    if (k < RK) {
      upd_off = kinfo[k].upd_off;
      rows_begin = kinfo[k].rows_begin;
      qk = kinfo[k].q;
      roff = kinfo[k].rupd_off;
    } else {
      const KhKid C = T.kids[F.child_begin + k];
      upd_off = C.upd_off;
      rows_begin = C.rows_begin;
      qk = C.q;
      roff = C.rupd_off;
    }
    // FWD: the child's rhs update, loaded ahead of its update block
    double2 rreg[FWD ? RY : 1];
    if (FWD) {
      const double2* rc = fw.ru_child + (int64_t)b * fw.ru_stride_child + roff;
#pragma unroll
      for (int u = 0; u < RY; ++u) {
        const int i = tid + u * NTH;
        rreg[u] = i < qk ? rc[i] : make_double2(0.0, 0.0);
      }
    }
    const double2* Uc = upd_child + (int64_t)b * upd_stride_child + upd_off;
    const int32_t* rk = k < RK ? rel + k * MS : T.relind + rows_begin;
    // warp w takes columns w, w + NW, ... CW at a time (all their loads in
    // flight before the adds); lanes walk the rows
    constexpr int CW = asm_cols(MS);
    for (int cj0 = warp; cj0 < qk; cj0 += CW * NW) {
      double2 v[CW][R];
      int dst[CW][R];
#pragma unroll
      for (int h = 0; h < CW; ++h) {
        const int cj = cj0 + h * NW;
        const int base = cj < qk ? cb[rk[cj]] : 0;
#pragma unroll
        for (int u = 0; u < R; ++u) {
          const int ci = cj + lane + 32 * u;
          const bool ok = cj < qk && ci < qk;
          v[h][u] = ok ? Uc[kh_upk32(qk, ci, cj)] : make_double2(0.0, 0.0);
          dst[h][u] = ok ? base + rk[ci] : -1;
        }
      }
#pragma unroll
      for (int h = 0; h < CW; ++h)
#pragma unroll
        for (int u = 0; u < R; ++u)
          if (dst[h][u] >= 0) {
            KH_ASSERT(dst[h][u] < ne);
            S[dst[h][u]] = cadd(S[dst[h][u]], v[h][u]);
          }
    }
    if (FWD) {  // the child's rhs update (rows distinct within a child)
#pragma unroll
      for (int u = 0; u < RY; ++u) {
        const int i = tid + u * NTH;
        if (i < qk) xs[rk[i]] = cadd(xs[rk[i]], rreg[u]);
      }
    }
  }
  if (FWD && nkids == 0) {
#pragma unroll
    for (int u = 0; u < RY; ++u) {
      const int c = tid + u * NTH;
      if (c < m) xs[c] = yreg[u];
    }
  }
  __syncthreads();
  phase(1);

  const double minp = blocked_ldlt<NW, kLookAhead(NW), MS / 16, front_has_w(MS)>(S, cb, W, LDW, dinv, dg, &ctr, m, p);
  phase(2);
  if (FWD && warp == 0) {
    // forward sweep on the shared-memory panel: lane owns rows lane + 32 v
    double2 x[R];
#pragma unroll
    for (int v = 0; v < R; ++v) {
      const int r = lane + 32 * v;
      x[v] = r < m ? xs[r] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      if (32 * u >= p) break;
      const int kend = min(32, p - 32 * u);
      for (int kk = 0; kk < kend; ++kk) {
        const int k = 32 * u + kk;
        const double2 xk = shfl2(x[u], kk);
        const int ck = cb[k];
#pragma unroll
        for (int v = 0; v < R; ++v) {
          const int r = lane + 32 * v;
          if (r > k && r < m) x[v] = cfms(x[v], S[ck + r], xk);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < R; ++v) {
      const int r = lane + 32 * v;
      if (r < m) xs[r] = x[v];
    }
  }
  // ---- write the panel and the update matrix (lower parts)
#if KH_BULK_WRITE
  // every column's lower part is contiguous both in the packed shared layout
  // and in global memory: one bulk async copy (TMA, async proxy) per column,
  // issued by the last warp's lanes, so the CTA does not spend issue slots
  // and registers on the stores (it only waits for the shared-memory reads)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const bool issuer = warp == NW - 1;
  if (issuer) {
    for (int c = lane; c < m; c += 32) {
      const double2* src;
      double2* dst;
      int rows;
      if (c < p) {
        src = S + cb[c] + c;
        dst = P + c + (int64_t)c * m;
        rows = m - c;
      } else {
        const int cc = c - p;
        src = S + cb[c] + c;
        dst = U + kh_upk32(q, cc, cc);
        rows = q - cc;
      }
      const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(src));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(saddr),
                   "r"(rows * 16)
                   : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
#else
  // coalesced: warp per column, lanes down the rows
  for (int c = warp; c < p; c += NW) {
    const int base = cb[c];
    for (int r = c + lane; r < m; r += 32) P[r + (int64_t)c * m] = S[base + r];
  }
  for (int c = warp; c < q; c += NW) {
    const int base = cb[p + c] + p;
    for (int r = c + lane; r < q; r += 32) U[kh_upk32(q, r, c)] = S[base + r];
  }
#endif
  if (FWD) {
    __syncthreads();
    double2* yb = fw.y + (int64_t)b * T.n + F.first;
    double2* ru = fw.ru_cur + (int64_t)b * fw.ru_stride_cur + F.rupd_off;
    for (int c = tid; c < m; c += NTH) {
      if (c < p) yb[c] = xs[c];
      else ru[c - p] = xs[c];
    }
  }
  if (tid == 0) minpiv[(int64_t)b * T.nf + f] = minp;
#if KH_BULK_WRITE
  // shared memory must outlive the bulk copies' reads of it
  if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
  phase(3);
}

// ---- forward solve: y <- L^{-1} b, fronts bottom-up ------------------------
// Large fronts of a wide level (many CTAs per SM): one CTA per (front,
// shift), blocks of 32 pivots solved by one warp in shared memory, rows below
// updated one thread per row.
__global__ void __launch_bounds__(NT) fwd_level_kernel(KhTree T, const int32_t* __restrict__ level_fronts,
                                                       const double2* __restrict__ panels, double2* y,
                                                       double2* ru_cur, int64_t ru_stride_cur,
                                                       const double2* __restrict__ ru_child,
                                                       int64_t ru_stride_child) {
  __shared__ double2 sL[NB * (NB + 1)];
  __shared__ double2 sy[NB];
  const int tid = threadIdx.x;
  const int32_t f = level_fronts[blockIdx.x];
  const int b = blockIdx.y;
  const KhDevFront F = T.fronts[f];
  const int p = F.p, q = F.q, m = p + q;
  const double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  double2* yy = y + (int64_t)b * T.n + F.first;
  double2* ru = ru_cur + (int64_t)b * ru_stride_cur + F.rupd_off;
  // pull the children's rhs updates (fixed child order: deterministic)
  __shared__ const double2* kru[MAXC];
  __shared__ const int32_t* kcm[MAXC];
  const int nk = F.child_end - F.child_begin;
  if (tid < MAXC && tid < nk) {
    const KhDevFront C = T.fronts[T.child_list[F.child_begin + tid]];
    kru[tid] = ru_child + (int64_t)b * ru_stride_child + C.rupd_off;
    kcm[tid] = T.cmap + C.cmap_begin;
  }
  __syncthreads();
  for (int r = tid; r < m; r += NT) {
    double2 v = make_double2(0.0, 0.0);
    for (int k = 0; k < nk; ++k) {
      const double2* rc;
      const int32_t* cm;
      if (k < MAXC) {
        rc = kru[k];
        cm = kcm[k];
      } else {
        const KhDevFront C = T.fronts[T.child_list[F.child_begin + k]];
        rc = ru_child + (int64_t)b * ru_stride_child + C.rupd_off;
        cm = T.cmap + C.cmap_begin;
      }
      const int ci = cm[r];
      if (ci >= 0) v = cadd(v, rc[ci]);
    }
    if (r < p) yy[r] = cadd(yy[r], v);
    else ru[r - p] = v;
  }
  __syncthreads();
  for (int kb = 0; kb < p; kb += NB) {
    const int w = min(NB, p - kb);
    for (int idx = tid; idx < w * w; idx += NT) {
      int i = idx % w, j = idx / w;
      sL[i * (NB + 1) + j] = P[(kb + i) + (int64_t)(kb + j) * m];
    }
    if (tid < w) sy[tid] = yy[kb + tid];
    __syncthreads();
    if (tid < 32) {  // one warp: unit-lower solve of the block
      for (int k = 0; k < w; ++k) {
        double2 yk = sy[k];
        __syncwarp();
        if (tid > k && tid < w) sy[tid] = cfms(sy[tid], sL[tid * (NB + 1) + k], yk);
        __syncwarp();
      }
    }
    __syncthreads();
    if (tid < w) yy[kb + tid] = sy[tid];
    // rows below the block
    for (int r = kb + w + tid; r < m; r += NT) {
      double2 s = make_double2(0.0, 0.0);
#pragma unroll 8
      for (int k = 0; k < w; ++k) {
        double2 l = P[r + (int64_t)(kb + k) * m];
        s = cadd(s, cmul(l, sy[k]));
      }
      if (r < p) yy[r] = csub(yy[r], s);
      else ru[r - p] = csub(ru[r - p], s);
    }
    __syncthreads();
  }
}

// Large fronts of a narrow level (top of the tree: fewer CTAs than SMs x 8),
// one CTA per (front, shift). The front's rhs segment x[0:m) is
// kept in shared memory. Per 32-column block: warp 0 loads the block's rows
// into registers (coalesced per column) and solves it with shuffles (no
// barriers on the chain), while warps 1..7 already load their rows' 32 panel
// entries below the block; after one barrier they finish the GEMV update
// x[r] -= L[r, blk] x[blk] from registers. Rows beyond 224 below the block
// take extra passes by all warps.
constexpr int FWD_W = 32;
// levels with at most this many (front, shift) CTAs use the narrow-level
// solves (crossover measured at c3: profiles/r1_solve_levels.md)
#ifndef KH_NARROW_FWD
#define KH_NARROW_FWD 1024
#endif
#ifndef KH_NARROW_BWD
#define KH_NARROW_BWD 2048
#endif
constexpr int64_t kNarrowLevelCtas = KH_NARROW_FWD, kNarrowLevelCtasBwd = KH_NARROW_BWD;
__global__ void __launch_bounds__(NT, 2) fwd_top_kernel(KhTree T, const int32_t* __restrict__ level_fronts,
                                                          const double2* __restrict__ panels, double2* y,
                                                          double2* ru_cur, int64_t ru_stride_cur,
                                                          const double2* __restrict__ ru_child,
                                                          int64_t ru_stride_child) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* xs = reinterpret_cast<double2*>(smem_raw);  // m + FWD_W entries
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t f = level_fronts[blockIdx.x];
  const int b = blockIdx.y;
  const KhDevFront F = T.fronts[f];
  const int p = F.p, q = F.q, m = p + q;
  const double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  double2* yy = y + (int64_t)b * T.n + F.first;
  double2* ru = ru_cur + (int64_t)b * ru_stride_cur + F.rupd_off;
  const double2 z = make_double2(0.0, 0.0);
  // gather: pivots' rhs plus the children's rhs updates (pull, fixed child order)
  __shared__ const double2* kru[MAXC];
  __shared__ const int32_t* kcm[MAXC];
  const int nk = F.child_end - F.child_begin;
  if (tid < MAXC && tid < nk) {
    const KhDevFront C = T.fronts[T.child_list[F.child_begin + tid]];
    kru[tid] = ru_child + (int64_t)b * ru_stride_child + C.rupd_off;
    kcm[tid] = T.cmap + C.cmap_begin;
  }
  __syncthreads();
  // xs[m, m + FWD_W) is zeroed: the GEMV below multiplies the L columns past the
  // block width (zeros) with xs entries up to kb + FWD_W, which must be finite
  for (int r = m + tid; r < m + FWD_W; r += NT) xs[r] = z;
  for (int r = tid; r < m; r += NT) {
    double2 v = r < p ? yy[r] : z;
    for (int k = 0; k < nk; ++k) {
      const double2* rc;
      const int32_t* cm;
      if (k < MAXC) {
        rc = kru[k];
        cm = kcm[k];
      } else {
        const KhDevFront C = T.fronts[T.child_list[F.child_begin + k]];
        rc = ru_child + (int64_t)b * ru_stride_child + C.rupd_off;
        cm = T.cmap + C.cmap_begin;
      }
      const int ci = cm[r];
      if (ci >= 0) v = cadd(v, rc[ci]);
    }
    xs[r] = v;
  }
  __syncthreads();
  for (int kb = 0; kb < p; kb += FWD_W) {
    const int w = min(FWD_W, p - kb), r0 = kb + w;
    constexpr int H = FWD_W / 2;  // register arrays hold half a block (2 CTAs per SM)
    double2 l[H];
    if (warp == 0) {
      // lane i: row kb+i of the block, L[kb+i][kb+k] for k < i; two halves
      const int i = lane;
      double2 xi = i < w ? xs[kb + i] : z;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
        for (int k = 0; k < H; ++k) {
          const int kk = hh * H + k;
          l[k] = (kk < i && i < w) ? P[(kb + i) + (int64_t)(kb + kk) * m] : z;
        }
#pragma unroll
        for (int k = 0; k < H; ++k) {
          const double2 xk = shfl2(xi, hh * H + k);
          xi = cfms(xi, l[k], xk);  // l[k] = 0 unless kk < i < w
        }
      }
      if (i < w) xs[kb + i] = xi;
    } else {
      const int r = r0 + tid - 32;
#pragma unroll
      for (int k = 0; k < H; ++k) l[k] = (r < m && k < w) ? P[r + (int64_t)(kb + k) * m] : z;
    }
    __syncthreads();
    if (warp > 0) {
      const int r = r0 + tid - 32;
      if (r < m) {
        double2 s0 = z, s1 = z;
#pragma unroll
        for (int k = 0; k < H; k += 2) {
          s0 = cadd(s0, cmul(l[k], xs[kb + k]));
          s1 = cadd(s1, cmul(l[k + 1], xs[kb + k + 1]));
        }
#pragma unroll
        for (int k = 0; k < H; ++k) l[k] = (H + k < w) ? P[r + (int64_t)(kb + H + k) * m] : z;
#pragma unroll
        for (int k = 0; k < H; k += 2) {
          s0 = cadd(s0, cmul(l[k], xs[kb + H + k]));
          s1 = cadd(s1, cmul(l[k + 1], xs[kb + H + k + 1]));
        }
        xs[r] = csub(xs[r], cadd(s0, s1));
      }
    }
    for (int r = r0 + (NT - 32) + tid; r < m; r += NT) {  // rows beyond the first pass
      double2 s0 = z, s1 = z;
#pragma unroll 8
      for (int k = 0; k < w; ++k) {
        const double2 lv = P[r + (int64_t)(kb + k) * m];
        if (k & 1) s1 = cadd(s1, cmul(lv, xs[kb + k]));
        else s0 = cadd(s0, cmul(lv, xs[kb + k]));
      }
      xs[r] = csub(xs[r], cadd(s0, s1));
    }
    __syncthreads();
  }
  for (int r = tid; r < m; r += NT) {
    if (r < p) yy[r] = xs[r];
    else ru[r - p] = xs[r];
  }
}

// ---- warp-per-front solves for fronts with m <= 32 R (R <= 4) -------------------
// Lane l owns front rows l + 32 h. No block barriers: pivots are broadcast
// with shuffles.
constexpr int SOLVE_CH = 8;   // columns per warp_sum8 reduction (bwd)

#ifndef KH_FWD_TMA_NW
#define KH_FWD_TMA_NW 1
#endif
// R rows per lane (rows lane + 32 h, h < R: m <= 32 R; one instantiation per
// front class, so no work on rows that cannot exist).
template <int NW, int R>
__global__ void __launch_bounds__(32 * NW) fwd_small_tma_kernel(KhTree T, const int32_t* __restrict__ level_fronts,
                                                                int32_t nlev, const double2* __restrict__ panels,
                                                                double2* y, double2* ru_cur, int64_t ru_stride_cur,
                                                                const double2* __restrict__ ru_child,
                                                                int64_t ru_stride_child, int32_t maxe) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int idx = blockIdx.x * NW + warp;
  if (idx >= nlev) return;
  const int b = blockIdx.y;
  const KhDevFront F = T.lf_fronts[(level_fronts - T.lf_base) + idx];
  const int p = F.p, q = F.q, m = p + q;
  const double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  double2* Ls = reinterpret_cast<double2*>(smem_raw) + (int64_t)warp * maxe;
  uint64_t* br = &bar[warp];
  auto cbase = [m](int c) { return c * m - (c * (c - 1)) / 2; };
  if (lane == 0) {
    mbar_init(br, 1);
    mbar_fence_init();
  }
  __syncwarp();
  KH_ASSERT(p * m - (p * (p - 1)) / 2 <= maxe && m <= 32 * R);
  if (lane == 0) mbar_arrive_expect_tx(br, 16u * (uint32_t)(p * m - (p * (p - 1)) / 2));
  __syncwarp();
  for (int c = lane; c < p; c += 32) bulk_g2s(Ls + cbase(c), P + c + (int64_t)c * m, 16u * (uint32_t)(m - c), br);
  double2* yy = y + (int64_t)b * T.n + F.first;
  double2* ru = ru_cur + (int64_t)b * ru_stride_cur + F.rupd_off;
  const double2 z = make_double2(0.0, 0.0);
  double2 x[R];  // lane l owns front rows l + 32 h
#pragma unroll
  for (int h = 0; h < R; ++h) x[h] = z;
  KH_ASSERT(m <= 32 * R);
  for (int c = F.child_begin; c < F.child_end; ++c) {
    const KhKid C = T.kids[c];
    const double2* rc = ru_child + (int64_t)b * ru_stride_child + C.rupd_off;
    const int32_t* cm = T.cmap + C.cmap_begin;
#pragma unroll
    for (int h = 0; h < R; ++h) {
      const int r = lane + 32 * h;
      const int ci = r < m ? cm[r] : -1;
      if (ci >= 0) x[h] = cadd(x[h], rc[ci]);
    }
  }
#pragma unroll
  for (int h = 0; h < R; ++h)
    if (lane + 32 * h < p) x[h] = cadd(x[h], yy[lane + 32 * h]);
  mbar_wait(br, 0);
  for (int k = 0; k < p; ++k) {
    const double2* col = Ls + cbase(k) - k;  // L[r, k] = col[r], r >= k
    double2 src = x[0];
#pragma unroll
    for (int h = 1; h < R; ++h)
      if (k >= 32 * h) src = x[h];
    const double2 yk = shfl2(src, k & 31);
#pragma unroll
    for (int h = 0; h < R; ++h) {
      const int r = lane + 32 * h;
      const double2 l = (r > k && r < m) ? col[r] : z;
      x[h] = cfms(x[h], l, yk);
    }
  }
#pragma unroll
  for (int h = 0; h < R; ++h) {
    const int r = lane + 32 * h;
    if (r < p) yy[r] = x[h];
    else if (r < m) ru[r - p] = x[h];
  }
}

// Backward solve of the fronts with m <= 64, one warp per (front, shift), the
// front's panel (lower part, column by column: column c = rows c..m-1) staged
// in shared memory by bulk async copies that lanes 0..p-1 issue at kernel
// start (one TMA-engine transfer per column, completion counted on the warp's
// mbarrier). The solution values of the update rows and the pivots' rhs are
// gathered while the copies are in flight, so the front costs one memory
// round trip for its panel instead of one per register chunk of columns.
//  t_k = y_k / d_k - sum_a L21[a, k] xu[a]   (column sums: warp_sum8 over 8 columns)
//  L11^T x = t                               (lane k owns t_k; pivots by shuffles)
#ifndef KH_BWD_TMA_NW
#define KH_BWD_TMA_NW 1
#endif
template <int NW, int R>
__global__ void __launch_bounds__(32 * NW) bwd_small_tma_kernel(KhTree T, const int32_t* __restrict__ level_fronts,
                                                                int32_t nlev, const double2* __restrict__ panels,
                                                                double2* y, int32_t maxe) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int idx = blockIdx.x * NW + warp;
  if (idx >= nlev) return;
  const int b = blockIdx.y;
  const KhDevFront F = T.lf_fronts[(level_fronts - T.lf_base) + idx];
  const int p = F.p, q = F.q, m = p + q;
  const double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  double2* Ls = reinterpret_cast<double2*>(smem_raw) + (int64_t)warp * maxe;
  uint64_t* br = &bar[warp];
  auto cbase = [m](int c) { return c * m - (c * (c - 1)) / 2; };
  if (lane == 0) {
    mbar_init(br, 1);
    mbar_fence_init();
  }
  __syncwarp();
  KH_ASSERT(p * m - (p * (p - 1)) / 2 <= maxe && m <= 32 * R);
  if (lane == 0) mbar_arrive_expect_tx(br, 16u * (uint32_t)(p * m - (p * (p - 1)) / 2));
  __syncwarp();
  for (int c = lane; c < p; c += 32) bulk_g2s(Ls + cbase(c), P + c + (int64_t)c * m, 16u * (uint32_t)(m - c), br);
  double2* yb = y + (int64_t)b * T.n;
  double2* yy = yb + F.first;
  const int64_t* urows = T.urows + F.rows_begin;
  const double2 z = make_double2(0.0, 0.0);
  double2 xu[R], yv[R], t[R];  // lane l: update rows / pivots l + 32 h
#pragma unroll
  for (int h = 0; h < R; ++h) {
    xu[h] = lane + 32 * h < q ? yb[urows[lane + 32 * h]] : z;
    yv[h] = lane + 32 * h < p ? yy[lane + 32 * h] : z;
    t[h] = z;
  }
  KH_ASSERT(m <= 32 * R);
  mbar_wait(br, 0);
  for (int kc = 0; kc < p; kc += SOLVE_CH) {
    double2 sv[SOLVE_CH];
#pragma unroll
    for (int u = 0; u < SOLVE_CH; ++u) {
      const int k = kc + u;
      const double2* col = Ls + cbase(k) + (p - k);  // L21[:, k]
      double2 acc = z;
#pragma unroll
      for (int h = 0; h < R; ++h) {
        const double2 l = (k < p && lane + 32 * h < q) ? col[lane + 32 * h] : z;
        acc = h == 0 ? cmul(l, xu[0]) : cadd(acc, cmul(l, xu[h]));
      }
      sv[u] = acc;
    }
    const double2 v = warp_sum8(sv, lane);
#pragma unroll
    for (int h = 0; h < R; ++h) {
      const int kk = lane + 32 * h, u = kk - kc;
      const int src = ((u >> 2) & 1) << 4 | ((u >> 1) & 1) << 3 | (u & 1) << 2;
      const double2 got = shfl2(v, src & 31);
      if (u >= 0 && u < SOLVE_CH && kk < p) t[h] = got;
    }
  }
#pragma unroll
  for (int h = 0; h < R; ++h) {
    const int k = lane + 32 * h;
    if (k < p) t[h] = csub(cmul(yv[h], cinv(Ls[cbase(k)])), t[h]);
  }
  // L11^T x = t bottom-up (column form: x_i final -> t_k -= L[i, k] x_i, k < i)
  for (int i = p - 1; i > 0; --i) {
    double2 src = t[0];
#pragma unroll
    for (int h = 1; h < R; ++h)
      if (i >= 32 * h) src = t[h];
    const double2 xi = shfl2(src, i & 31);
#pragma unroll
    for (int h = 0; h < R; ++h) {
      const int k = lane + 32 * h;
      if (k < i) t[h] = cfms(t[h], Ls[cbase(k) + i - k], xi);
    }
  }
#pragma unroll
  for (int h = 0; h < R; ++h)
    if (lane + 32 * h < p) yy[lane + 32 * h] = t[h];
}

// Backward solve of the large fronts of a narrow level (top of the tree):
// one CTA per (front, shift), t and x[urows] in shared memory.
//  1. t_k = y_k / d_k - sum_a L21[a, k] x[urows[a]]: warps over chunks of 8
//     columns, lanes down the rows (coalesced), warp_sum8 reductions;
//  2. blocks of 32 pivots from the last: warp 0 stages the block (coalesced)
//     in shared memory and solves L_blk^T x = t with shuffles while warps 1..7
//     load their first chunk of L[blk, 0:kb] (independent of x); after one
//     barrier, t[0:kb] -= L[blk, 0:kb]^T x[blk] by warp reductions.
__global__ void __launch_bounds__(NT, 2) bwd_top_kernel(KhTree T, const int32_t* __restrict__ level_fronts,
                                                        const double2* __restrict__ panels, double2* y) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* ts = reinterpret_cast<double2*>(smem_raw);  // p entries, then xu: q entries
  __shared__ double2 blk[FWD_W][FWD_W + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t f = level_fronts[blockIdx.x];
  const int b = blockIdx.y;
  const KhDevFront F = T.fronts[f];
  const int p = F.p, q = F.q, m = p + q;
  const double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  double2* yb = y + (int64_t)b * T.n;
  double2* yy = yb + F.first;
  double2* xu = ts + p;
  const int64_t* urows = T.urows + F.rows_begin;
  const double2 z = make_double2(0.0, 0.0);
  for (int a = tid; a < q; a += NT) xu[a] = yb[urows[a]];
  __syncthreads();
  // 1. t = D^-1 y - L21^T xu
  for (int k0 = 8 * warp; k0 < p; k0 += 8 * (NT / 32)) {
    double2 sacc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) sacc[u] = z;
#pragma unroll 2
    for (int a = lane; a < q; a += 32) {
      const double2 xa = xu[a];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (k0 + u < p) sacc[u] = cadd(sacc[u], cmul(P[p + a + (int64_t)(k0 + u) * m], xa));
    }
    const double2 v = warp_sum8(sacc, lane);
    const int u = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    const int k = k0 + u;
    if ((lane & 3) == 0 && k < p) ts[k] = csub(cmul(yy[k], cinv(P[k + (int64_t)k * m])), v);
  }
  __syncthreads();
  // 2. L11^T x = t, blocks of 32 from the last
  const int nblk = (p + FWD_W - 1) / FWD_W;
  for (int bi = nblk - 1; bi >= 0; --bi) {
    const int kb = bi * FWD_W, w = min(FWD_W, p - kb);
    const int nch = kb / 8;  // chunks of 8 columns left of the block
    double2 l[8];
    // stage the block with all warps (warp c&7 loads columns c = warp, warp+8, ..)
    for (int c = warp; c < w; c += NT / 32) blk[lane][c] = lane < w ? P[(kb + lane) + (int64_t)(kb + c) * m] : z;
    __syncthreads();
    if (warp == 0) {
      double2 t = lane < w ? ts[kb + lane] : z;
      for (int i = w - 1; i > 0; --i) {
        const double2 xi = shfl2(t, i);
        if (lane < i) t = cfms(t, blk[i][lane], xi);
      }
      if (lane < w) ts[kb + lane] = t;
    } else if (warp < nch) {  // chunk c = warp: prefetch L[kb+lane, 8c : 8c+8]
#pragma unroll
      for (int u = 0; u < 8; ++u) l[u] = lane < w ? P[(kb + lane) + (int64_t)(8 * warp + u) * m] : z;
    }
    __syncthreads();
    if (nch > 0) {
      const double2 xl = lane < w ? ts[kb + lane] : z;
      for (int c = warp; c < nch; c += NT / 32) {
        if (c != warp || warp == 0) {
#pragma unroll
          for (int u = 0; u < 8; ++u) l[u] = lane < w ? P[(kb + lane) + (int64_t)(8 * c + u) * m] : z;
        }
        double2 sacc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) sacc[u] = cmul(l[u], xl);
        const double2 v = warp_sum8(sacc, lane);
        const int u = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
        if ((lane & 3) == 0) ts[8 * c + u] = csub(ts[8 * c + u], v);
      }
    }
    __syncthreads();
  }
  for (int k = tid; k < p; k += NT) yy[k] = ts[k];
}

// ---- solves of the fronts with m > 64 on wide levels, panel staged by bulk copies
// One CTA per (front, shift) whose whole lower panel fits in shared memory
// (the host picks these kernels per level): warp 0 issues one bulk async copy
// per panel column at kernel start, the right-hand side / update-row values
// are gathered meanwhile, and after one mbarrier wait every operand of the
// sweep is on chip (the level kernels above take a global round trip per
// 32-pivot block for the block and another for the rows below it).
// Shared memory: the packed panel (column c = rows c..m-1 at c m - c(c-1)/2,
// `maxe` entries reserved) followed by the front's vector (m entries).
#ifndef KH_MID_TMA
#define KH_MID_TMA 1
#endif
constexpr int MID_NW = 4, MID_NT = 32 * MID_NW;
KH_DEV void mid_stage_panel(const double2* P, int p, int m, double2* Ls, uint64_t* bar) {
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid < 32) {
    if (lane == 0) mbar_arrive_expect_tx(bar, 16u * (uint32_t)(p * m - (p * (p - 1)) / 2));
    __syncwarp();
    for (int c = lane; c < p; c += 32)
      bulk_g2s(Ls + (c * m - (c * (c - 1)) / 2), P + c + (int64_t)c * m, 16u * (uint32_t)(m - c), bar);
  }
}

__global__ void __launch_bounds__(MID_NT) fwd_mid_tma_kernel(KhTree T, const int32_t* __restrict__ level_fronts,
                                                            const double2* __restrict__ panels, double2* y,
                                                            double2* ru_cur, int64_t ru_stride_cur,
                                                            const double2* __restrict__ ru_child,
                                                            int64_t ru_stride_child, int32_t maxe) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  double2* Ls = reinterpret_cast<double2*>(smem_raw);
  double2* xs = Ls + maxe;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const KhDevFront F = T.lf_fronts[(level_fronts - T.lf_base) + blockIdx.x];
  const int b = blockIdx.y;
  const int p = F.p, q = F.q, m = p + q;
  KH_ASSERT(p * m - (p * (p - 1)) / 2 <= maxe);
  const double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  double2* yy = y + (int64_t)b * T.n + F.first;
  double2* ru = ru_cur + (int64_t)b * ru_stride_cur + F.rupd_off;
  mid_stage_panel(P, p, m, Ls, &bar);
  // the front's rhs: pivot rows of y plus the children's updates (fixed child order)
  const int nk = F.child_end - F.child_begin;
  for (int r = tid; r < m; r += MID_NT) {
    double2 v = r < p ? yy[r] : make_double2(0.0, 0.0);
    for (int k = 0; k < nk; ++k) {
      const KhKid C = T.kids[F.child_begin + k];
      const int ci = T.cmap[C.cmap_begin + r];
      if (ci >= 0) v = cadd(v, ru_child[(int64_t)b * ru_stride_child + C.rupd_off + ci]);
    }
    xs[r] = v;
  }
  mbar_wait(&bar, 0);
  __syncthreads();
  auto L = [&](int r, int c) { return Ls[c * m - (c * (c - 1)) / 2 + r - c]; };  // r >= c
  for (int kb = 0; kb < p; kb += NB) {
    const int w = min(NB, p - kb);
    if (warp == 0) {
      const int i = lane;
      double2 xi = i < w ? xs[kb + i] : make_double2(0.0, 0.0);
#pragma unroll 8
      for (int k = 0; k < w; ++k) {
        const double2 l = (i > k && i < w) ? L(kb + i, kb + k) : make_double2(0.0, 0.0);
        const double2 xk = shfl2(xi, k);
        xi = cfms(xi, l, xk);
      }
      if (i < w) xs[kb + i] = xi;
    }
    __syncthreads();
    for (int r = kb + w + tid; r < m; r += MID_NT) {
      double2 s0 = make_double2(0.0, 0.0), s1 = s0;
#pragma unroll 4
      for (int k = 0; k < w; k += 2) {
        s0 = cadd(s0, cmul(L(r, kb + k), xs[kb + k]));
        if (k + 1 < w) s1 = cadd(s1, cmul(L(r, kb + k + 1), xs[kb + k + 1]));
      }
      xs[r] = csub(xs[r], cadd(s0, s1));
    }
    __syncthreads();
  }
  for (int r = tid; r < m; r += MID_NT) {
    if (r < p) yy[r] = xs[r];
    else ru[r - p] = xs[r];
  }
}

__global__ void __launch_bounds__(MID_NT) bwd_mid_tma_kernel(KhTree T, const int32_t* __restrict__ level_fronts,
                                                            const double2* __restrict__ panels, double2* y,
                                                            int32_t maxe) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  double2* Ls = reinterpret_cast<double2*>(smem_raw);
  double2* ts = Ls + maxe;  // p entries, then xu: q entries
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const KhDevFront F = T.lf_fronts[(level_fronts - T.lf_base) + blockIdx.x];
  const int b = blockIdx.y;
  const int p = F.p, q = F.q, m = p + q;
  KH_ASSERT(p * m - (p * (p - 1)) / 2 <= maxe);
  const double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  double2* yb = y + (int64_t)b * T.n;
  double2* yy = yb + F.first;
  double2* xu = ts + p;
  const int64_t* urows = T.urows + F.rows_begin;
  mid_stage_panel(P, p, m, Ls, &bar);
  for (int a = tid; a < q; a += MID_NT) xu[a] = yb[urows[a]];
  for (int k = tid; k < p; k += MID_NT) ts[k] = yy[k];
  mbar_wait(&bar, 0);
  __syncthreads();
  auto L = [&](int r, int c) { return Ls[c * m - (c * (c - 1)) / 2 + r - c]; };  // r >= c
  // t_k = y_k / d_k - sum_a L21[a, k] xu[a]   (warp per column k)
  for (int k = warp; k < p; k += MID_NW) {
    double2 s = make_double2(0.0, 0.0);
    for (int a = lane; a < q; a += 32) s = cadd(s, cmul(L(p + a, k), xu[a]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
    }
    if (lane == 0) ts[k] = csub(cmul(ts[k], cinv(L(k, k))), s);
  }
  __syncthreads();
  const int nblk = (p + NB - 1) / NB;
  for (int bi = nblk - 1; bi >= 0; --bi) {
    const int kb = bi * NB, w = min(NB, p - kb);
    if (warp == 0) {  // L_blk^T x = t_blk: lane i owns t_{kb+i}
      double2 t = lane < w ? ts[kb + lane] : make_double2(0.0, 0.0);
      for (int i = w - 1; i > 0; --i) {
        const double2 l = lane < i ? L(kb + i, kb + lane) : make_double2(0.0, 0.0);
        const double2 xi = shfl2(t, i);
        t = cfms(t, l, xi);
      }
      if (lane < w) ts[kb + lane] = t;
    }
    __syncthreads();
    // earlier pivots k < kb: t_k -= sum_i L[kb+i, k] x_{kb+i}   (warp per column)
    for (int k = warp; k < kb; k += MID_NW) {
      double2 s = lane < w ? cmul(L(kb + lane, k), ts[kb + lane]) : make_double2(0.0, 0.0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
      }
      if (lane == 0) ts[k] = csub(ts[k], s);
    }
    __syncthreads();
  }
  for (int k = tid; k < p; k += MID_NT) yy[k] = ts[k];
}

// ---- streamed solves of the fronts with m > 64 -----------------------------------
// One CTA per (front, shift). The panel is consumed in blocks of wf <= ST_W
// columns (as many as fit a stage of `stage` entries at the front's height),
// rows kb..m-1 of each (one contiguous segment per column, so one bulk async
// copy each), through a ring of `ns` shared-memory stages that the TMA engine
// fills ahead of the arithmetic: the loads do not depend on the sweep, so up
// to ns - 1 stages (tens of KB per SM) are in flight while a stage is
// consumed, which is what an HBM-bound sweep needs; the level kernels above
// take a dependent global round trip per 32-pivot block instead.
//   forward, blocks ascending: warp 0 solves the block's w x w unit-lower
//     system with shuffles, then thread-per-row x[r] -= sum_c L[r, c] x_c for
//     all r below (a per-warp redundant block solve saves the barrier but
//     saturates the shuffle pipe: 1800 cycles per stage, clock64 probe);
//   backward, blocks descending: s_c = sum_{r > block} L[r, c] x[r] over ALL
//     rows below the block (L11 and L21 alike: the column segments are
//     contiguous), thread-per-row partial sums, warp transpose-reduction,
//     fixed-order sum over the warps; then warp 0 finishes
//     x_blk = L_blk^-T (y_blk / d - s).
// Two CTA barriers per stage; results are deterministic (fixed row -> thread
// map and reduction order).
constexpr int ST_W = 8, ST_NT = 256, ST_NW = ST_NT / 32, ST_MAXS = 8;
#ifdef KH_STREAM_TIMING
// debug builds (profiles/probes/stream_timing.py): clock64 cycles of thread 0 of
// fwd_stream_kernel summed over CTAs: [prologue, mbarrier waits, block solve, rows, barrier+issue, stages, CTAs]
__device__ unsigned long long g_stphase[8];
#define ST_LAP(i)                                                          \
  if (tid == 0) {                                                          \
    const long long t1_ = clock64();                                       \
    atomicAdd(&g_stphase[i], (unsigned long long)(t1_ - tph_));            \
    tph_ = t1_;                                                            \
  }
#else
#define ST_LAP(i)
#endif

// columns per stage for a front of m rows
KH_DEV int stream_width(int m, int stage) { return max(1, min(ST_W, stage / m)); }

// stage `bi` (block of columns kb = wf bi ..) -> buf, by warp 0
KH_DEV void stream_issue(const double2* P, int m, int p, int wf, int bi, double2* buf, uint64_t* bar, int lane) {
  const int kb = wf * bi, w = min(wf, p - kb), rows = m - kb;
  // the buffer was read through the generic proxy: order those reads before the async-proxy writes
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (lane == 0) mbar_arrive_expect_tx(bar, 16u * (uint32_t)(w * rows));
  __syncwarp();
  if (lane < w) bulk_g2s(buf + lane * rows, P + kb + (int64_t)(kb + lane) * m, 16u * (uint32_t)rows, bar);
}

__global__ void __launch_bounds__(ST_NT) fwd_stream_kernel(KhTree T, const int32_t* __restrict__ level_fronts,
                                                           const double2* __restrict__ panels, double2* y,
                                                           double2* ru_cur, int64_t ru_stride_cur,
                                                           const double2* __restrict__ ru_child,
                                                           int64_t ru_stride_child, int32_t lvl_m, int32_t stage, int32_t ns) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[ST_MAXS];
  __shared__ double2 xb[ST_W];                           // the current block's solution
  double2* xs = reinterpret_cast<double2*>(smem_raw);  // lvl_m entries
  double2* ring = xs + lvl_m;                            // ns stages of `stage` entries
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const KhDevFront F = T.lf_fronts[(level_fronts - T.lf_base) + blockIdx.x];
  const int b = blockIdx.y;
  const int p = F.p, q = F.q, m = p + q;
  KH_ASSERT(m <= lvl_m && ns <= ST_MAXS);
  const double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  double2* yy = y + (int64_t)b * T.n + F.first;
  double2* ru = ru_cur + (int64_t)b * ru_stride_cur + F.rupd_off;
  const int wf = stream_width(m, stage), nblk = (p + wf - 1) / wf;
#ifdef KH_STREAM_TIMING
  long long tph_ = clock64();
  if (tid == 0) {
    atomicAdd(&g_stphase[5], (unsigned long long)nblk);
    atomicAdd(&g_stphase[6], 1ull);
  }
#endif
  if (tid == 0) {
    for (int i = 0; i < ns; ++i) mbar_init(&full[i], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == 0)
    for (int s = 0; s < ns && s < nblk; ++s) stream_issue(P, m, p, wf, s, ring + s * stage, &full[s], lane);
  // the front's rhs: pivot rows of y plus the children's updates (fixed child order)
  const int nk = F.child_end - F.child_begin;
  for (int r = tid; r < m; r += ST_NT) {
    double2 v = r < p ? yy[r] : make_double2(0.0, 0.0);
    for (int k = 0; k < nk; ++k) {
      const KhKid C = T.kids[F.child_begin + k];
      const int ci = T.cmap[C.cmap_begin + r];
      if (ci >= 0) v = cadd(v, ru_child[(int64_t)b * ru_stride_child + C.rupd_off + ci]);
    }
    xs[r] = v;
  }
  __syncthreads();
  ST_LAP(0)
  const double2 z = make_double2(0.0, 0.0);
  for (int s = 0; s < nblk; ++s) {
    const int slot = s % ns;
    const double2* buf = ring + slot * stage;
    const int kb = wf * s, w = min(wf, p - kb), rows = m - kb;
    mbar_wait(&full[slot], (uint32_t)((s / ns) & 1));
    ST_LAP(1)
    // the block's unit-lower solve by warp 0 (lane i owns row kb + i), published in xb
    if (warp == 0) {
      double2 xi = lane < w ? xs[kb + lane] : z;
      double2 lk[ST_W];
#pragma unroll
      for (int k = 0; k < ST_W; ++k) lk[k] = (k < w && lane > k && lane < w) ? buf[k * rows + lane] : z;
#pragma unroll
      for (int k = 0; k < ST_W; ++k) xi = cfms(xi, lk[k], shfl2(xi, k));
      if (lane < w) {
        xb[lane] = xi;
        yy[kb + lane] = xi;
      }
    }
    __syncthreads();
    double2 xc[ST_W];
#pragma unroll
    for (int c = 0; c < ST_W; ++c) xc[c] = c < w ? xb[c] : z;
    ST_LAP(2)
    for (int r = kb + w + tid; r < m; r += ST_NT) {
      const double2* l = buf + (r - kb);
      double2 a0 = z, a1 = z;
#pragma unroll
      for (int c = 0; c < ST_W; c += 2) {
        if (c < w) a0 = cadd(a0, cmul(l[c * rows], xc[c]));
        if (c + 1 < w) a1 = cadd(a1, cmul(l[(c + 1) * rows], xc[c + 1]));
      }
      xs[r] = csub(xs[r], cadd(a0, a1));
    }
    ST_LAP(3)
    __syncthreads();  // stage consumed, xs updated
    if (warp == 0 && s + ns < nblk) stream_issue(P, m, p, wf, s + ns, ring + slot * stage, &full[slot], lane);
    ST_LAP(4)
  }
  for (int r = p + tid; r < m; r += ST_NT) ru[r - p] = xs[r];
}

__global__ void __launch_bounds__(ST_NT) bwd_stream_kernel(KhTree T, const int32_t* __restrict__ level_fronts,
                                                           const double2* __restrict__ panels, double2* y,
                                                           int32_t lvl_m, int32_t stage, int32_t ns) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[ST_MAXS];
  __shared__ double2 red[2][ST_NW][ST_W];
  double2* xs = reinterpret_cast<double2*>(smem_raw);  // x: lvl_m entries (solution; update rows gathered)
  double2* ys = xs + lvl_m;                              // y of the pivot rows (read-only): lvl_m entries
  double2* ring = ys + lvl_m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const KhDevFront F = T.lf_fronts[(level_fronts - T.lf_base) + blockIdx.x];
  const int b = blockIdx.y;
  const int p = F.p, q = F.q, m = p + q;
  KH_ASSERT(m <= lvl_m && ns <= ST_MAXS);
  const double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  double2* yb = y + (int64_t)b * T.n;
  double2* yy = yb + F.first;
  const int64_t* urows = T.urows + F.rows_begin;
  const int wf = stream_width(m, stage), nblk = (p + wf - 1) / wf;
  if (tid == 0) {
    for (int i = 0; i < ns; ++i) mbar_init(&full[i], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == 0)
    for (int s = 0; s < ns && s < nblk; ++s)
      stream_issue(P, m, p, wf, nblk - 1 - s, ring + s * stage, &full[s], lane);
  for (int a = tid; a < q; a += ST_NT) xs[p + a] = yb[urows[a]];  // final: the ancestors are done
  for (int k = tid; k < p; k += ST_NT) ys[k] = yy[k];
  __syncthreads();
  const double2 z = make_double2(0.0, 0.0);
  for (int s = 0; s < nblk; ++s) {
    const int slot = s % ns;
    const double2* buf = ring + slot * stage;
    const int kb = wf * (nblk - 1 - s), w = min(wf, p - kb), rows = m - kb;
    mbar_wait(&full[slot], (uint32_t)((s / ns) & 1));
    // s_c = sum over the rows below the block of L[r, c] x[r]
    double2 acc[ST_W];
#pragma unroll
    for (int c = 0; c < ST_W; ++c) acc[c] = z;
    for (int r = kb + w + tid; r < m; r += ST_NT) {
      const double2 xr = xs[r];
      const double2* l = buf + (r - kb);
#pragma unroll
      for (int c = 0; c < ST_W; ++c)
        if (c < w) acc[c] = cadd(acc[c], cmul(l[c * rows], xr));
    }
    const double2 v = warp_sum8(acc, lane);
    if ((lane & 3) == 0) red[s & 1][warp][((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1)] = v;
    __syncthreads();
    // x_blk = L_blk^-T (y_blk / d - s) by warp 0: lane c owns column kb + c
    if (warp == 0) {
      double2 t = z;
      double2 li[ST_W];
#pragma unroll
      for (int i = 1; i < ST_W; ++i) li[i] = (i < w && lane < i) ? buf[lane * rows + i] : z;  // L[kb + i, kb + lane]
      if (lane < w) {
        double2 sum = red[s & 1][0][lane];
#pragma unroll
        for (int wp = 1; wp < ST_NW; ++wp) sum = cadd(sum, red[s & 1][wp][lane]);
        t = csub(cmul(ys[kb + lane], cinv(buf[lane * rows + lane])), sum);
      }
#pragma unroll
      for (int i = ST_W - 1; i > 0; --i) t = cfms(t, li[i], shfl2(t, i));
      if (lane < w) xs[kb + lane] = t;
    }
    __syncthreads();  // stage consumed, x_blk visible
    if (warp == 0 && s + ns < nblk)
      stream_issue(P, m, p, wf, nblk - 1 - (s + ns), ring + slot * stage, &full[slot], lane);
  }
  for (int k = tid; k < p; k += ST_NT) yy[k] = xs[k];
}

// ---- backward solve: x <- L^{-T} D^{-1} y, fronts top-down -------------------
__global__ void __launch_bounds__(NT) bwd_level_kernel(KhTree T, const int32_t* __restrict__ level_fronts,
                                                       const double2* __restrict__ panels, double2* y) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* st = reinterpret_cast<double2*>(smem_raw);  // p entries
  __shared__ double2 sL[NB * (NB + 1)];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t f = level_fronts[blockIdx.x];
  const int b = blockIdx.y;
  const KhDevFront F = T.fronts[f];
  const int p = F.p, q = F.q, m = p + q;
  const double2* P = panels + (int64_t)b * T.panel_total + F.panel_off;
  double2* yb = y + (int64_t)b * T.n;
  double2* yy = yb + F.first;
  const int64_t* urows = T.urows + F.rows_begin;
  // x of the update rows (final: ancestors are done), gathered once
  double2* xu = st + p;
  for (int a = tid; a < q; a += NT) xu[a] = yb[urows[a]];
  __syncthreads();
  // t_k = y_k / d_k - sum_a L21[a, k] x[urows[a]]   (warp per column k)
  for (int k = warp; k < p; k += NT / 32) {
    double2 s = make_double2(0.0, 0.0);
    const double2* col = P + p + (int64_t)k * m;
#pragma unroll 4
    for (int a = lane; a < q; a += 32) s = cadd(s, cmul(col[a], xu[a]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
    }
    if (lane == 0) st[k] = csub(cmul(yy[k], cinv(P[k + (int64_t)k * m])), s);
  }
  __syncthreads();
  // blocks from last to first: solve L_blk^T x_blk = t_blk, then push into earlier t
  const int nblk = (p + NB - 1) / NB;
  for (int bi = nblk - 1; bi >= 0; --bi) {
    const int kb = bi * NB, w = min(NB, p - kb);
    for (int idx = tid; idx < w * w; idx += NT) {
      int i = idx % w, j = idx / w;
      sL[i * (NB + 1) + j] = P[(kb + i) + (int64_t)(kb + j) * m];
    }
    __syncthreads();
    if (tid < 32) {
      for (int i = w - 1; i >= 0; --i) {
        double2 xi = st[kb + i];
        __syncwarp();
        if (tid < i) st[kb + tid] = cfms(st[kb + tid], sL[i * (NB + 1) + tid], xi);
        __syncwarp();
      }
    }
    __syncthreads();
    // earlier pivots k < kb: t_k -= sum_i L[kb+i, k] x_{kb+i}  (warp per column)
    for (int k = warp; k < kb; k += NT / 32) {
      double2 s = make_double2(0.0, 0.0);
      if (lane < w) s = cmul(P[(kb + lane) + (int64_t)k * m], st[kb + lane]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
      }
      if (lane == 0) st[k] = csub(st[k], s);
    }
    __syncthreads();
  }
  for (int k = tid; k < p; k += NT) yy[k] = st[k];
}

__global__ void gather_orig_kernel(int64_t n, const int64_t* __restrict__ src, const double* __restrict__ mv,
                                   const double* __restrict__ av, double* __restrict__ om, double* __restrict__ oa) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = src[e];
    om[e] = mv[s];
    oa[e] = av[s];
  }
}

__global__ void gather_rhs_kernel(int64_t n, const int64_t* __restrict__ perm, const double* __restrict__ g_re,
                                  const double* __restrict__ g_im, int64_t ldg, double2* y) {
  const int b = blockIdx.y;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    int64_t src = perm[k] + (int64_t)b * ldg;
    y[(int64_t)b * n + k] = make_double2(g_re[src], g_im ? g_im[src] : 0.0);
  }
}

__global__ void scatter_sol_kernel(int64_t n, const int64_t* __restrict__ perm, const double2* __restrict__ y,
                                   double* z_re, double* z_im, int64_t ldz) {
  const int b = blockIdx.y;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    int64_t dst = perm[k] + (int64_t)b * ldz;
    double2 v = y[(int64_t)b * n + k];
    z_re[dst] = v.x;
    if (z_im) z_im[dst] = v.y;
  }
}

__global__ void shift_absmax_kernel(const double* __restrict__ mv, const double* __restrict__ av, int64_t nnz,
                                    const double2* __restrict__ lam, double* part) {
  __shared__ double red[NT / 32];
  const int b = blockIdx.y;
  const double2 L = lam[b];
  double mx = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * NT) {
    double re = fma(L.x, av[e], mv[e]), im = L.y * av[e];
    mx = fmax(mx, sqrt(re * re + im * im));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < NT / 32; ++w) mx = fmax(mx, red[w]);
    part[(int64_t)b * gridDim.x + blockIdx.x] = mx;
  }
}

// op: 0 = sum, 1 = min, 2 = max over each row of a [rows][len] array
__global__ void rowreduce_kernel(const double* __restrict__ in, int64_t len, int op, double* out) {
  __shared__ double red[NT / 32];
  const int r = blockIdx.x;
  auto comb = [op](double a, double b) { return op == 0 ? a + b : (op == 1 ? fmin(a, b) : fmax(a, b)); };
  double v = op == 0 ? 0.0 : (op == 1 ? DBL_MAX : -DBL_MAX);
  for (int64_t i = threadIdx.x; i < len; i += NT) v = comb(v, in[(int64_t)r * len + i]);
  for (int o = 16; o > 0; o >>= 1) v = comb(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < NT / 32; ++w) v = comb(v, red[w]);
    out[r] = v;
  }
}

}  // namespace

cudaError_t kh_launch_big_assemble(const KhTree& T, const int32_t* tasks, int32_t ntasks, int32_t batch,
                                   const double2* lam, double2* panels, const double2* upd_child,
                                   int64_t upd_stride_child, cudaStream_t stream) {
  if (ntasks == 0 || batch == 0) return cudaSuccess;
  big_assemble_kernel<<<dim3(ntasks, batch), NT, 0, stream>>>(T, tasks, lam, panels, upd_child, upd_stride_child);
  kh_note_launch();
  return cudaGetLastError();
}


cudaError_t kh_launch_pivot_block(const KhTree& T, const int32_t* tasks, int32_t ntasks, int c0, int32_t batch,
                                 double2* panels, double* minpiv, double2* img, int64_t img_stride,
                                 cudaStream_t stream) {
  if (ntasks == 0 || batch == 0) return cudaSuccess;
  if (KH_PIVOT_WARP) return kh_launch_pivot_warp(T, tasks, ntasks, c0, batch, panels, minpiv, img, img_stride, stream);
  const int smem = piv_smem_bytes();
  cudaError_t e = kh_smem_optin((const void*)pivot_block_kernel, smem);
  if (e != cudaSuccess) return e;
  pivot_block_kernel<<<dim3(ntasks, batch), 32 * PIV_NW, smem, stream>>>(T, tasks, c0, panels, minpiv, img,
                                                                         img_stride);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_panel_solve(const KhTree& T, const int32_t* tasks, int32_t ntasks, int c0, int32_t batch,
                                  double2* panels, const double2* img, int64_t img_stride, cudaStream_t stream) {
  if (ntasks == 0 || batch == 0) return cudaSuccess;
  panel_trsm_kernel<<<dim3(ntasks, batch), 32 * PTR_NW, 0, stream>>>(T, tasks, c0, panels, img, img_stride);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_panel_update(const KhTree& T, const int32_t* tasks, int32_t ntasks, int c0, int32_t batch,
                                   double2* panels, cudaStream_t stream) {
  if (ntasks == 0 || batch == 0) return cudaSuccess;
  const int smem = (int)(CP_STAGES * sizeof(CpStage));
  cudaError_t e = kh_smem_optin((const void*)panel_update_kernel, smem);
  if (e != cudaSuccess) return e;
  panel_update_kernel<<<dim3(ntasks, batch), NT, smem, stream>>>(T, tasks, c0, panels);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_schur(const KhTree& T, const int32_t* tasks, int32_t ntasks, int32_t batch,
                            const double2* panels, double2* upd_cur, int64_t upd_stride_cur, const double2* upd_child,
                            int64_t upd_stride_child, cudaStream_t stream) {
  if (ntasks == 0 || batch == 0) return cudaSuccess;
  // the operand ring, reused by the epilogue's 64 x 65 product tile
  const int smem = (int)std::max(CP_STAGES * sizeof(CpStage), sizeof(double2) * TB * (TB + 1));
  cudaError_t e = kh_smem_optin((const void*)schur_update_kernel, smem);
  if (e != cudaSuccess) return e;
  schur_update_kernel<<<dim3(ntasks, batch), NT, smem, stream>>>(T, tasks, panels, upd_cur, upd_stride_cur,
                                                                 upd_child, upd_stride_child);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_fwd_small(const KhTree& T, const int32_t* level_fronts, int32_t nlev, int32_t batch,
                                const double2* panels, double2* y, double2* ru_cur, int64_t ru_stride_cur,
                                const double2* ru_child, int64_t ru_stride_child, int32_t max_panel,
                                cudaStream_t stream, int32_t max_m) {
  if (nlev == 0 || batch == 0) return cudaSuccess;
  constexpr int nw = KH_FWD_TMA_NW;
  const int smem = 16 * nw * max_panel;
  auto run = [&](auto kernel) -> cudaError_t {
    cudaError_t e = kh_smem_optin((const void*)kernel, smem);
    if (e != cudaSuccess) return e;
    kernel<<<dim3((nlev + nw - 1) / nw, batch), 32 * nw, smem, stream>>>(
        T, level_fronts, nlev, panels, y, ru_cur, ru_stride_cur, ru_child, ru_stride_child, max_panel);
    kh_note_launch();
    return cudaGetLastError();
  };
  if (max_m <= 32) return run(fwd_small_tma_kernel<nw, 1>);
  if (max_m <= 64) return run(fwd_small_tma_kernel<nw, 2>);
  if (max_m <= 96) return run(fwd_small_tma_kernel<nw, 3>);
  return max_m <= 128 ? run(fwd_small_tma_kernel<nw, 4>) : cudaErrorInvalidValue;
}

cudaError_t kh_launch_bwd_small(const KhTree& T, const int32_t* level_fronts, int32_t nlev, int32_t batch,
                                const double2* panels, double2* y, int32_t max_panel, cudaStream_t stream,
                                int32_t max_m) {
  if (nlev == 0 || batch == 0) return cudaSuccess;
  constexpr int nw = KH_BWD_TMA_NW;
  const int smem = 16 * nw * max_panel;
  auto run = [&](auto kernel) -> cudaError_t {
    cudaError_t e = kh_smem_optin((const void*)kernel, smem);
    if (e != cudaSuccess) return e;
    kernel<<<dim3((nlev + nw - 1) / nw, batch), 32 * nw, smem, stream>>>(T, level_fronts, nlev, panels, y,
                                                                         max_panel);
    kh_note_launch();
    return cudaGetLastError();
  };
  if (max_m <= 32) return run(bwd_small_tma_kernel<nw, 1>);
  if (max_m <= 64) return run(bwd_small_tma_kernel<nw, 2>);
  if (max_m <= 96) return run(bwd_small_tma_kernel<nw, 3>);
  return max_m <= 128 ? run(bwd_small_tma_kernel<nw, 4>) : cudaErrorInvalidValue;
}

#ifdef KH_STREAM_TIMING
extern "C" int kh_debug_stream_cycles(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, g_stphase, sizeof(unsigned long long) * 8) != cudaSuccess) return 4;
  static const unsigned long long zero[8] = {};
  return cudaMemcpyToSymbol(g_stphase, zero, sizeof zero) == cudaSuccess ? 0 : 4;
}
#endif

// stage size (entries) and ring depth of the streamed solves. A stage holds
// up to ST_W columns of the level's tallest front, at most 24 KB (taller
// fronts get fewer columns per stage). Wide levels (thousands of short
// panels: the rhs gather in front of the sweep dominates a CTA's life) take a
// ring of two, so that several CTAs per SM overlap each other; narrow levels
// (the top of the tree: few CTAs, long panels) a ring of four.
#ifndef KH_STREAM_STAGE_E
#define KH_STREAM_STAGE_E 1536
#endif
#ifndef KH_STREAM_STAGES
#define KH_STREAM_STAGES 4
#endif
#ifndef KH_STREAM_MIN_FRONTS
#define KH_STREAM_MIN_FRONTS 12
#endif
#ifndef KH_STREAM_MAX_FRONTS
#define KH_STREAM_MAX_FRONTS 64
#endif
#ifndef KH_STREAM_STAGES_WIDE
#define KH_STREAM_STAGES_WIDE 2
#endif
static int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}
static int stream_stage_entries(int lvl_m) {
  static const int e = env_int("KH_STREAM_STAGE_E", KH_STREAM_STAGE_E);
  return std::max(std::min(e, ST_W * lvl_m), lvl_m);
}
static int stream_stages(int stage, int64_t ctas) {
  static const int narrow = env_int("KH_STREAM_STAGES", KH_STREAM_STAGES);
  static const int wide = env_int("KH_STREAM_STAGES_WIDE", KH_STREAM_STAGES_WIDE);
  const int fit = (200 * 1024) / (16 * stage);
  return std::max(2, std::min(std::min(ctas >= 148 * 4 ? wide : narrow, fit), ST_MAXS));
}

// streamed solves of the large fronts (KH_STREAM_SOLVE=0: the level / top / mid kernels)
static bool stream_solves(int32_t nlev) {
  static const bool on = [] {
    const char* v = std::getenv("KH_STREAM_SOLVE");
    return !v || std::atoi(v) != 0;
  }();
  static const int lo = [] { const char* v = std::getenv("KH_STREAM_MIN_FRONTS"); return v ? std::atoi(v) : KH_STREAM_MIN_FRONTS; }();
  static const int hi = [] { const char* v = std::getenv("KH_STREAM_MAX_FRONTS"); return v ? std::atoi(v) : KH_STREAM_MAX_FRONTS; }();
  return on && nlev >= lo && nlev <= hi;
}
cudaError_t kh_launch_fwd_level(const KhTree& T, const int32_t* level_fronts, int32_t nlev, int32_t batch,
                                int32_t max_m, const double2* panels, double2* y, double2* ru_cur,
                                int64_t ru_stride_cur, const double2* ru_child, int64_t ru_stride_child,
                                cudaStream_t stream, int32_t mid_panel, int32_t mid_m, int32_t lvl_m) {
  if (nlev == 0 || batch == 0) return cudaSuccess;
  if (stream_solves(nlev) && lvl_m > 0) {
    const int stage = stream_stage_entries(lvl_m), ns = stream_stages(stage, (int64_t)nlev * batch);
    const int smem = 16 * (lvl_m + ns * stage);
    cudaError_t e = kh_smem_optin((const void*)fwd_stream_kernel, smem);
    if (e != cudaSuccess) return e;
    fwd_stream_kernel<<<dim3(nlev, batch), ST_NT, smem, stream>>>(T, level_fronts, panels, y, ru_cur, ru_stride_cur,
                                                                  ru_child, ru_stride_child, lvl_m, stage, ns);
    kh_note_launch();
    return cudaGetLastError();
  }
  if (KH_MID_TMA && mid_panel > 0 && (int64_t)nlev * batch > kNarrowLevelCtas) {
    const int smem = 16 * (mid_panel + mid_m);
    cudaError_t e = kh_smem_optin((const void*)fwd_mid_tma_kernel, smem);
    if (e != cudaSuccess) return e;
    fwd_mid_tma_kernel<<<dim3(nlev, batch), MID_NT, smem, stream>>>(T, level_fronts, panels, y, ru_cur,
                                                                    ru_stride_cur, ru_child, ru_stride_child,
                                                                    mid_panel);
    kh_note_launch();
    return cudaGetLastError();
  }
  if ((int64_t)nlev * batch > kNarrowLevelCtas) {
    fwd_level_kernel<<<dim3(nlev, batch), NT, 0, stream>>>(T, level_fronts, panels, y, ru_cur, ru_stride_cur,
                                                           ru_child, ru_stride_child);
    kh_note_launch();
    return cudaGetLastError();
  }
  const size_t smem = sizeof(double2) * (size_t)(max_m + FWD_W);
  cudaError_t e = kh_smem_optin((const void*)fwd_top_kernel, (int)smem);
  if (e != cudaSuccess) return e;
  fwd_top_kernel<<<dim3(nlev, batch), NT, smem, stream>>>(T, level_fronts, panels, y, ru_cur, ru_stride_cur,
                                                          ru_child, ru_stride_child);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_bwd_level(const KhTree& T, const int32_t* level_fronts, int32_t nlev, int32_t batch,
                                int32_t max_p, int32_t max_m, const double2* panels, double2* y,
                                cudaStream_t stream, int32_t mid_panel, int32_t mid_m, int32_t lvl_m) {
  if (nlev == 0 || batch == 0) return cudaSuccess;
  if (stream_solves(nlev) && lvl_m > 0) {
    const int stage = stream_stage_entries(lvl_m), ns = stream_stages(stage, (int64_t)nlev * batch);
    const int smem = 16 * (2 * lvl_m + ns * stage);
    cudaError_t e = kh_smem_optin((const void*)bwd_stream_kernel, smem);
    if (e != cudaSuccess) return e;
    bwd_stream_kernel<<<dim3(nlev, batch), ST_NT, smem, stream>>>(T, level_fronts, panels, y, lvl_m, stage, ns);
    kh_note_launch();
    return cudaGetLastError();
  }
  const bool narrow = (int64_t)nlev * batch <= kNarrowLevelCtasBwd;
  if (KH_MID_TMA && mid_panel > 0 && !narrow) {
    const int smem = 16 * (mid_panel + mid_m);
    cudaError_t e = kh_smem_optin((const void*)bwd_mid_tma_kernel, smem);
    if (e != cudaSuccess) return e;
    bwd_mid_tma_kernel<<<dim3(nlev, batch), MID_NT, smem, stream>>>(T, level_fronts, panels, y, mid_panel);
    kh_note_launch();
    return cudaGetLastError();
  }
  const size_t smem = sizeof(double2) * (size_t)max_m;
  cudaError_t e = kh_smem_optin(narrow ? (const void*)bwd_top_kernel : (const void*)bwd_level_kernel, (int)smem);
  if (e != cudaSuccess) return e;
  if (narrow) bwd_top_kernel<<<dim3(nlev, batch), NT, smem, stream>>>(T, level_fronts, panels, y);
  else bwd_level_kernel<<<dim3(nlev, batch), NT, smem, stream>>>(T, level_fronts, panels, y);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_gather_orig(int64_t n_orig, const int64_t* src, const double* mv, const double* av, double* om,
                                  double* oa, cudaStream_t stream) {
  if (n_orig <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((n_orig + 255) / 256, 148 * 8);
  gather_orig_kernel<<<blocks, 256, 0, stream>>>(n_orig, src, mv, av, om, oa);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_gather_rhs(int64_t n, int32_t batch, const int64_t* perm, const double* g_re,
                                 const double* g_im, int64_t ldg, double2* y, cudaStream_t stream) {
  if (n == 0 || batch == 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 1024);
  gather_rhs_kernel<<<dim3(blocks, batch), 256, 0, stream>>>(n, perm, g_re, g_im, ldg, y);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_scatter_sol(int64_t n, int32_t batch, const int64_t* perm, const double2* y, double* z_re,
                                  double* z_im, int64_t ldz, cudaStream_t stream) {
  if (n == 0 || batch == 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 1024);
  scatter_sol_kernel<<<dim3(blocks, batch), 256, 0, stream>>>(n, perm, y, z_re, z_im, ldz);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_shift_absmax_nnz(const double* mv, const double* av, int64_t nnz, int32_t batch,
                                       const double2* lam, double* part, int32_t nblk, cudaStream_t stream) {
  if (batch == 0) return cudaSuccess;
  shift_absmax_kernel<<<dim3(nblk, batch), NT, 0, stream>>>(mv, av, nnz, lam, part);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_rowreduce(const double* in, int64_t len, int32_t rows, int op, double* out,
                                cudaStream_t stream) {
  if (rows == 0) return cudaSuccess;
  rowreduce_kernel<<<rows, NT, 0, stream>>>(in, len, op, out);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_factor_small(int ms, const KhTree& T, const int32_t* level_fronts, int32_t nlev, int32_t batch,
                                   const double2* lam, double2* panels, double2* upd_cur, int64_t upd_stride_cur,
                                   const double2* upd_child, int64_t upd_stride_child, double* minpiv,
                                   cudaStream_t stream, const KhFwd* fwd) {
  if (nlev == 0 || batch == 0) return cudaSuccess;
  const dim3 grid(nlev, batch);
  FwdArgs fw{};
  if (fwd) fw = {fwd->y, fwd->ru_cur, fwd->ru_stride_cur, fwd->ru_child, fwd->ru_stride_child};
  auto run = [&](auto kernel, int ms_, int threads, int) -> cudaError_t {
    const int smem = front_smem_bytes(ms_);
    cudaError_t e = kh_smem_optin((const void*)kernel, smem);
    if (e != cudaSuccess) return e;
    kernel<<<grid, threads, smem, stream>>>(T, level_fronts, lam, panels, upd_cur, upd_stride_cur, upd_child,
                                            upd_stride_child, minpiv, fw);
    kh_note_launch();
    return cudaGetLastError();
  };
  switch (ms) {
    case 32: return fwd ? run(factor_front_kernel<32, KH_NW32, true>, 32, 32 * KH_NW32, 0)
                        : run(factor_front_kernel<32, KH_NW32, false>, 32, 32 * KH_NW32, 0);
    case 40:  // the shared-memory kernel of the m <= 48 class serves m <= 40 too
    case 48: return fwd ? run(factor_front_kernel<48, KH_NW48, true>, 48, 32 * KH_NW48, 1)
                        : run(factor_front_kernel<48, KH_NW48, false>, 48, 32 * KH_NW48, 1);
    case 64: return fwd ? run(factor_front_kernel<64, KH_NW64, true>, 64, 32 * KH_NW64, 2)
                        : run(factor_front_kernel<64, KH_NW64, false>, 64, 32 * KH_NW64, 2);
    case KH_CLASS4: return fwd ? run(factor_front_kernel<KH_CLASS4, KH_NW96, true>, KH_CLASS4, 32 * KH_NW96, 3)
                        : run(factor_front_kernel<KH_CLASS4, KH_NW96, false>, KH_CLASS4, 32 * KH_NW96, 3);
    case 128: return fwd ? run(factor_front_kernel<128, KH_NW128, true>, 128, 32 * KH_NW128, 4)
                         : run(factor_front_kernel<128, KH_NW128, false>, 128, 32 * KH_NW128, 4);
    default: return cudaErrorInvalidValue;
  }
}

#ifdef KH_PHASE_TIMING
extern "C" int kh_debug_phase_cycles(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, g_phase, sizeof(unsigned long long) * 9 * 8) != cudaSuccess) return 4;
  static const unsigned long long zero[9 * 8] = {};
  return cudaMemcpyToSymbol(g_phase, zero, sizeof zero) == cudaSuccess ? 0 : 4;
}
#endif
