// fp64 DMMA GEMM for the modal transforms (C = alpha*A*B + beta*C, column-
// major). Replaces the reference's zgemm chains at solvers.py:368-372
// (G = F A^-1 conj(U) S^-1 conj(Vh)) and :397-400 (U = Z Vh^T S U^T); the host
// folds those N_t x N_t factors into one real matrix per direction, so each
// transform is a single real GEMM (M_x x N_t) * (N_t x N_t).
//
// Tiling: 128x64 CTA tile, K chunks of 16 staged by cp.async in a 3-stage
// ring, 8 warps of 32x32 each issuing mma.sync.m8n8k4.f64 (DMMA). Shared
// layouts are padded so both fragment loads are bank-conflict free:
// A chunk [k][m] with ld 132, B chunk [n][k] with ld 20.
#include "common.cuh"
#include "kernels.h"

namespace {

#ifndef KH_GEMM_BK
#define KH_GEMM_BK 16
#endif
#ifndef KH_GEMM_NST
#define KH_GEMM_NST 3
#endif
constexpr int BM = 128, BN = 64, BK = KH_GEMM_BK, NST = KH_GEMM_NST;
constexpr int LDA_S = BM + 4, LDB_S = BK + 4;
constexpr int A_STAGE = BK * LDA_S, B_STAGE = BN * LDB_S;
constexpr size_t SMEM_BYTES = sizeof(double) * NST * (A_STAGE + B_STAGE);

// SCATTER: row r of the result goes to part c = r / rp at dst[c] (row r - c rp,
// leading dimension ldd): the back transform's partial sums are written
// straight into each destination rank's receive slot over NVLink peer memory,
// tile by tile as the tiles finish (fused GEMM + scatter of the reduce-scatter).
template <bool SCATTER>
__global__ void __launch_bounds__(256) dgemm_kernel(int64_t M, int64_t N, int64_t K, double alpha,
                                                    const double* __restrict__ A, int64_t lda,
                                                    const double* __restrict__ B, int64_t ldb,
                                                    double beta, double* __restrict__ C, int64_t ldc,
                                                    double* const* __restrict__ dst, int64_t rp, int64_t ldd,
                                                    int64_t sA, int64_t sB, int64_t sC) {
  extern __shared__ __align__(16) double smem[];
  // batched (strided) GEMMs: blockIdx.z selects the problem
  A += blockIdx.z * sA;
  B += blockIdx.z * sB;
  if (!SCATTER) C += blockIdx.z * sC;
  double* As = smem;
  double* Bs = smem + NST * A_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 3, wn = warp >> 2;
  const int64_t n0 = (int64_t)blockIdx.x * BN, m0 = (int64_t)blockIdx.y * BM;
  const int nk = (int)((K + BK - 1) / BK);

  auto load_stage = [&](int st, int kc) {
    const int64_t k0 = (int64_t)kc * BK;
    double* as = As + st * A_STAGE;
    double* bs = Bs + st * B_STAGE;
#pragma unroll
    for (int r = 0; r < (BK * BM) / 256; ++r) {
      int idx = tid + r * 256;
      int k = idx / BM, i = idx % BM;
      int64_t gi = m0 + i, gk = k0 + k;
      bool ok = gi < M && gk < K;
      cp_async8(as + k * LDA_S + i, ok ? A + gi + gk * lda : A, ok);
    }
#pragma unroll
    for (int r = 0; r < (BK * BN) / 256; ++r) {
      int idx = tid + r * 256;
      int k = idx % BK, j = idx / BK;
      int64_t gj = n0 + j, gk = k0 + k;
      bool ok = gj < N && gk < K;
      cp_async8(bs + j * LDB_S + k, ok ? B + gk + gj * ldb : B, ok);
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < NST - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<NST - 2>();
    __syncthreads();
    {
      int nxt = kc + NST - 1;
      if (nxt < nk) load_stage(nxt % NST, nxt);
      cp_async_commit();
    }
    const double* as = As + (kc % NST) * A_STAGE;
    const double* bs = Bs + (kc % NST) * B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) af[mt] = as[(kk + t) * LDA_S + wm * 32 + mt * 8 + g];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = bs[(wn * 32 + nt * 8 + g) * LDB_S + kk + t];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    int64_t row = m0 + wm * 32 + mt * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int64_t col = n0 + wn * 32 + nt * 8 + 2 * t + h;
        if (col >= N) continue;
        double v = alpha * acc[mt][nt][h];
        if (SCATTER) {
          const int64_t part = row / rp;
          dst[part][(row - part * rp) + col * ldd] = v;
        } else {
          double* c = C + row + col * ldc;
          if (beta != 0.0) v = fma(beta, *c, v);
          *c = v;
        }
      }
  }
}

}  // namespace

namespace {

template <bool SCATTER>
cudaError_t launch(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda, const double* B,
                   int64_t ldb, double beta, double* C, int64_t ldc, double* const* dst, int64_t rp, int64_t ldd,
                   cudaStream_t stream, int32_t batch = 1, int64_t sA = 0, int64_t sB = 0, int64_t sC = 0) {
  if (M <= 0 || N <= 0 || batch <= 0) return cudaSuccess;
  const cudaError_t e = kh_smem_optin((const void*)dgemm_kernel<SCATTER>, (int)SMEM_BYTES);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)batch);
  dgemm_kernel<SCATTER><<<grid, 256, SMEM_BYTES, stream>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, dst, rp,
                                                           ldd, sA, sB, sC);
  kh_note_launch();
  return cudaGetLastError();
}

// out[e] = sum_{c < g} parts[c * len + e], in slot order (deterministic)
__global__ void sum_parts_kernel(int32_t g, const double* __restrict__ parts, int64_t len, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x) {
    double s = parts[e];
    for (int32_t c = 1; c < g; ++c) s += parts[c * len + e];
    out[e] = s;
  }
}

}  // namespace

cudaError_t kh_launch_dgemm(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                            const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                            cudaStream_t stream) {
  return launch<false>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, nullptr, 1, 0, stream);
}

cudaError_t kh_launch_dgemm_batched(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                                    int64_t sA, const double* B, int64_t ldb, int64_t sB, double beta, double* C,
                                    int64_t ldc, int64_t sC, int32_t batch, cudaStream_t stream) {
  return launch<false>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, nullptr, 1, 0, stream, batch, sA, sB, sC);
}

cudaError_t kh_launch_dgemm_rowscatter(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                                       const double* B, int64_t ldb, double* const* dst, int64_t rp, int64_t ldd,
                                       cudaStream_t stream) {
  return launch<true>(M, N, K, 1.0, A, lda, B, ldb, 0.0, nullptr, 0, dst, rp, ldd, stream);
}

cudaError_t kh_launch_sum_parts(int32_t g, const double* parts, int64_t len, double* out, cudaStream_t stream) {
  if (len <= 0) return cudaSuccess;
  const int blocks = (int)((len + 255) / 256 < 148 * 8 ? (len + 255) / 256 : 148 * 8);
  sum_parts_kernel<<<blocks, 256, 0, stream>>>(g, parts, len, out);
  kh_note_launch();
  return cudaGetLastError();
}
