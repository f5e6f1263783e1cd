// Space-time residual R = F - (M_x Y1 + A_x Y2) with Y = [Y1 | Y2] = U [A_t^T | M_t^T].
//
// Replaces `residual` (solvers.py:428-440), which applies
// K u = vec(M_x U A_t^T + A_x U M_t^T) through two `kron_apply_right` calls
// (dense.py:264-286). The dense temporal products run on the DMMA GEMM; this
// kernel is the fused dual SpMM (M_x and A_x share one CSR pattern) plus the
// subtraction from F and the partial sums of ||R||^2 and ||F||^2 (a fixed
// grid and a fixed reduction order keep the result deterministic).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace {

// Work item = (256 consecutive rows, RES_TCH consecutive time columns): each
// thread keeps its row's CSR entries in registers (read once, not once per
// time column) and sweeps the time columns; consecutive threads touch
// consecutive rows, so the Y / F / R accesses are coalesced. Items are handed
// out by a fixed grid-stride loop, so the partial sums are deterministic.
#ifndef KH_RES_TCH
#define KH_RES_TCH 16
#endif
constexpr int RES_TCH = KH_RES_TCH, RES_ROWNZ = 8;
// ABS: instead of R, the magnitude |f| + sum |m y1| + sum |a y2| of the terms
// whose cancellation the fp64 residual evaluates (its rounding floor is
// ~eps times the norm of that); R is not written.
template <bool ABS = false>
__global__ void __launch_bounds__(256) pair_residual_kernel(int64_t n, int64_t nt, const int64_t* __restrict__ indptr,
                                                            const int64_t* __restrict__ indices,
                                                            const double* __restrict__ mv,
                                                            const double* __restrict__ av,
                                                            const double* __restrict__ Y, int64_t ldy,
                                                            const double* __restrict__ F, int64_t ldf, double* R,
                                                            int64_t ldr, double* part) {
  __shared__ double red[2][8];
  const int64_t nrb = (n + 255) / 256, ntc = (nt + RES_TCH - 1) / RES_TCH;
  double rr = 0.0, ff = 0.0;
  for (int64_t item = blockIdx.x; item < nrb * ntc; item += gridDim.x) {
    const int64_t rb = item % nrb, tc = item / nrb;
    const int64_t i = rb * 256 + threadIdx.x;
    if (i >= n) continue;
    const int64_t e0 = indptr[i], e1 = indptr[i + 1];
    const int nz = (int)(e1 - e0);
    int64_t col[RES_ROWNZ];
    double mm[RES_ROWNZ], aa[RES_ROWNZ];
#pragma unroll
    for (int k = 0; k < RES_ROWNZ; ++k) {
      const bool ok = k < nz;
      col[k] = ok ? indices[e0 + k] : i;
      mm[k] = ok ? mv[e0 + k] : 0.0;
      aa[k] = ok ? av[e0 + k] : 0.0;
    }
    const int64_t t1 = min(nt, (tc + 1) * RES_TCH);
    for (int64_t t = tc * RES_TCH; t < t1; ++t) {
      const double* y1 = Y + t * ldy;
      const double* y2 = Y + (t + nt) * ldy;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < RES_ROWNZ; ++k) {
        if (ABS) {
          s = fma(fabs(mm[k]), fabs(y1[col[k]]), s);
          s = fma(fabs(aa[k]), fabs(y2[col[k]]), s);
        } else {
          s = fma(mm[k], y1[col[k]], s);
          s = fma(aa[k], y2[col[k]], s);
        }
      }
      for (int64_t e = e0 + RES_ROWNZ; e < e1; ++e) {  // rows longer than RES_ROWNZ
        const int64_t j = indices[e];
        if (ABS) {
          s = fma(fabs(mv[e]), fabs(y1[j]), s);
          s = fma(fabs(av[e]), fabs(y2[j]), s);
        } else {
          s = fma(mv[e], y1[j], s);
          s = fma(av[e], y2[j], s);
        }
      }
      const double f = F[i + t * ldf];
      const double r = ABS ? fabs(f) + s : f - s;
      if (!ABS && R) R[i + t * ldr] = r;
      rr = fma(r, r, rr);
      ff = fma(f, f, ff);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    rr += __shfl_xor_sync(0xffffffffu, rr, o);
    ff += __shfl_xor_sync(0xffffffffu, ff, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = rr;
    red[1][threadIdx.x >> 5] = ff;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) {
      rr += red[0][w];
      ff += red[1][w];
    }
    part[blockIdx.x] = rr;
    part[gridDim.x + blockIdx.x] = ff;
  }
}

// ---- compensated (double-double) residual -------------------------------------
// At fine spatial meshes the fp64 evaluation of f - K u loses digits: the
// rounding of Y2 = U M_t^T (relative eps) is amplified by the stiffness A_x
// (|A_x| |Y2| / |A_x Y2| ~ 1 / h^2), which puts a floor of ~3e-11 under the
// refined residual at config c4. The compensated path
// keeps Y2 as an unevaluated sum hi + lo (Dot2 of Ogita, Rump and Oishi: every
// product split exactly by an FMA, every sum by TwoSum) and applies M_x, A_x
// and the subtraction from F in the same compensated arithmetic; Y1 = U A_t^T
// stays fp64 (M_x is a positive mass matrix: its rounding is not amplified).
KH_DEV void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
// (hi, lo) += a * b, products and sums compensated
KH_DEV void dd_fma(double& hi, double& lo, double a, double b) {
  const double p = a * b;
  const double pe = fma(a, b, -p);
  double s, e;
  two_sum(hi, p, s, e);
  hi = s;
  lo += e + pe;
}

// C (m x n) = A (m x k) B (k x n), column-major, result as hi + lo. Tile 64 x 32,
// 256 threads, each a 4 x 2 block of compensated accumulators; A and B chunks
// of DD_KC columns / rows staged in shared memory (coalesced loads).
constexpr int DD_BM = 64, DD_BN = 32, DD_KC = 32;
__global__ void __launch_bounds__(256) dgemm_dd_kernel(int64_t M, int64_t N, int64_t K, const double* __restrict__ A,
                                                       int64_t lda, const double* __restrict__ B, int64_t ldb,
                                                       double* __restrict__ Chi, double* __restrict__ Clo,
                                                       int64_t ldc) {
  __shared__ double As[DD_KC][DD_BM + 1];
  __shared__ double Bs[DD_KC][DD_BN + 1];
  const int tid = threadIdx.x;
  const int64_t i0 = (int64_t)blockIdx.y * DD_BM, j0 = (int64_t)blockIdx.x * DD_BN;
  const int tr = (tid & 15) * 4, tc = (tid >> 4) * 2;
  double hi[4][2] = {}, lo[4][2] = {};
  for (int64_t k0 = 0; k0 < K; k0 += DD_KC) {
    for (int e = tid; e < DD_KC * DD_BM; e += 256) {
      const int r = e % DD_BM, kk = e / DD_BM;
      const int64_t gi = i0 + r, gk = k0 + kk;
      As[kk][r] = (gi < M && gk < K) ? A[gi + gk * lda] : 0.0;
    }
    for (int e = tid; e < DD_KC * DD_BN; e += 256) {
      const int kk = e % DD_KC, c = e / DD_KC;
      const int64_t gj = j0 + c, gk = k0 + kk;
      Bs[kk][c] = (gj < N && gk < K) ? B[gk + gj * ldb] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < DD_KC; ++kk) {
      double a[4], b[2];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = As[kk][tr + u];
#pragma unroll
      for (int v = 0; v < 2; ++v) b[v] = Bs[kk][tc + v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) dd_fma(hi[u][v], lo[u][v], a[u], b[v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int64_t gi = i0 + tr + u, gj = j0 + tc + v;
      if (gi < M && gj < N) {
        double s, e;
        two_sum(hi[u][v], lo[u][v], s, e);  // normalized pair
        Chi[gi + gj * ldc] = s;
        Clo[gi + gj * ldc] = e;
      }
    }
}

// R = F - (M_x Y1 + A_x (Y2hi + Y2lo)) in compensated arithmetic (rounded to
// fp64 once at the end), with the ||R||^2, ||F||^2 partial sums; the work
// items and reduction order of pair_residual_kernel (deterministic).
__global__ void __launch_bounds__(256) pair_residual_dd_kernel(
    int64_t n, int64_t nt, const int64_t* __restrict__ indptr, const int64_t* __restrict__ indices,
    const double* __restrict__ mv, const double* __restrict__ av, const double* __restrict__ Y1, int64_t ldy1,
    const double* __restrict__ Y2h, const double* __restrict__ Y2l, int64_t ldy2, const double* __restrict__ F,
    int64_t ldf, double* R, int64_t ldr, double* part) {
  __shared__ double red[2][8];
  const int64_t nrb = (n + 255) / 256, ntc = (nt + RES_TCH - 1) / RES_TCH;
  double rr = 0.0, ff = 0.0;
  for (int64_t item = blockIdx.x; item < nrb * ntc; item += gridDim.x) {
    const int64_t rb = item % nrb, tc = item / nrb;
    const int64_t i = rb * 256 + threadIdx.x;
    if (i >= n) continue;
    const int64_t e0 = indptr[i], e1 = indptr[i + 1];
    const int64_t t1 = min(nt, (tc + 1) * RES_TCH);
    for (int64_t t = tc * RES_TCH; t < t1; ++t) {
      const double f = F[i + t * ldf];
      double hi = f, lo = 0.0;
      for (int64_t e = e0; e < e1; ++e) {
        const int64_t j = indices[e];
        dd_fma(hi, lo, -mv[e], Y1[j + t * ldy1]);
        dd_fma(hi, lo, -av[e], Y2h[j + t * ldy2]);
        lo = fma(-av[e], Y2l[j + t * ldy2], lo);
      }
      const double r = hi + lo;
      if (R) R[i + t * ldr] = r;
      rr = fma(r, r, rr);
      ff = fma(f, f, ff);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    rr += __shfl_xor_sync(0xffffffffu, rr, o);
    ff += __shfl_xor_sync(0xffffffffu, ff, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = rr;
    red[1][threadIdx.x >> 5] = ff;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) {
      rr += red[0][w];
      ff += red[1][w];
    }
    part[blockIdx.x] = rr;
    part[gridDim.x + blockIdx.x] = ff;
  }
}

__global__ void __launch_bounds__(256) sumsq_kernel(const double* __restrict__ x, int64_t n, double* part) {
  __shared__ double red[8];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = fma(x[i], x[i], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(256) daxpy_kernel(int64_t n, double alpha, const double* __restrict__ x,
                                                    double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(alpha, x[i], y[i]);
}

}  // namespace

cudaError_t kh_launch_daxpy(int64_t n, double alpha, const double* x, double* y, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  daxpy_kernel<<<blocks, 256, 0, stream>>>(n, alpha, x, y);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_dgemm_dd(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                               int64_t ldb, double* Chi, double* Clo, int64_t ldc, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((N + DD_BN - 1) / DD_BN), (unsigned)((M + DD_BM - 1) / DD_BM));
  dgemm_dd_kernel<<<grid, 256, 0, stream>>>(M, N, K, A, lda, B, ldb, Chi, Clo, ldc);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_pair_residual_dd(int64_t n, int64_t nt, const int64_t* indptr, const int64_t* indices,
                                       const double* mv, const double* av, const double* Y1, int64_t ldy1,
                                       const double* Y2h, const double* Y2l, int64_t ldy2, const double* F,
                                       int64_t ldf, double* R, int64_t ldr, double* part, int32_t nblk,
                                       cudaStream_t stream) {
  pair_residual_dd_kernel<<<nblk, 256, 0, stream>>>(n, nt, indptr, indices, mv, av, Y1, ldy1, Y2h, Y2l, ldy2, F,
                                                    ldf, R, ldr, part);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_sumsq(const double* x, int64_t n, double* part, int32_t nblk, cudaStream_t stream) {
  sumsq_kernel<<<nblk, 256, 0, stream>>>(x, n, part);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_pair_residual(int64_t n, int64_t nt, const int64_t* indptr, const int64_t* indices,
                                    const double* mv, const double* av, const double* Y, int64_t ldy,
                                    const double* F, int64_t ldf, double* R, int64_t ldr, double* part,
                                    int32_t nblk, cudaStream_t stream) {
  pair_residual_kernel<false><<<nblk, 256, 0, stream>>>(n, nt, indptr, indices, mv, av, Y, ldy, F, ldf, R, ldr, part);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_residual_scale(int64_t n, int64_t nt, const int64_t* indptr, const int64_t* indices,
                                     const double* mv, const double* av, const double* Y, int64_t ldy,
                                     const double* F, int64_t ldf, double* part, int32_t nblk, cudaStream_t stream) {
  pair_residual_kernel<true><<<nblk, 256, 0, stream>>>(n, nt, indptr, indices, mv, av, Y, ldy, F, ldf, nullptr, 0,
                                                       part);
  kh_note_launch();
  return cudaGetLastError();
}
