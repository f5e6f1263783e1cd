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
        s = fma(mm[k], y1[col[k]], s);
        s = fma(aa[k], y2[col[k]], s);
      }
      for (int64_t e = e0 + RES_ROWNZ; e < e1; ++e) {  // rows longer than RES_ROWNZ
        const int64_t j = indices[e];
        s = fma(mv[e], y1[j], s);
        s = fma(av[e], y2[j], s);
      }
      const double f = F[i + t * ldf];
      const double r = f - s;
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

__global__ void __launch_bounds__(256) dot_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                  int64_t n, double* part) {
  __shared__ double red[8];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = fma(x[i], y[i], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(256) dscal_kernel(int64_t n, double alpha, double* __restrict__ x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= alpha;
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

cudaError_t kh_launch_dot(const double* x, const double* y, int64_t n, double* part, int32_t nblk,
                          cudaStream_t stream) {
  dot_kernel<<<nblk, 256, 0, stream>>>(x, y, n, part);
  kh_note_launch();
  return cudaGetLastError();
}

cudaError_t kh_launch_dscal(int64_t n, double alpha, double* x, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  dscal_kernel<<<blocks, 256, 0, stream>>>(n, alpha, x);
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
  pair_residual_kernel<<<nblk, 256, 0, stream>>>(n, nt, indptr, indices, mv, av, Y, ldy, F, ldf, R, ldr, part);
  kh_note_launch();
  return cudaGetLastError();
}
