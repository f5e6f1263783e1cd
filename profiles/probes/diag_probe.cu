// Latency probe of the 8 x 8 diagonal-block LDL^T (diag_block_ldlt) and one
// rank-8 DMMA tile update, in isolation: cycles per call for 1..16 warps per SM.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_2008_01996_b200/csrc diag_probe.cu
#include "../../paper_2008_01996_b200/csrc/frontal.cu"

#include <cstdio>

namespace {
// variant measured against diag_block_ldlt (slower: ~3600 vs ~3000 cycles)
// Same contract as diag_block_ldlt, without shuffles: every lane of warp 0
// loads the whole w x w lower block (shared-memory broadcasts) and factors it
// redundantly in registers, so a pivot's dependency chain is only the
// reciprocal and two complex multiply-adds; lane i < w then stores row i.
KH_DEV void diag_block_ldlt_regs(double2* S, const int32_t* cb, double2* dinv, double2* dg, int kb, int w, int m,
                                 double& minp) {
  constexpr int BK = 8;
  const int lane = threadIdx.x & 31;
  double2 a[BK][BK];  // a[i][j], j <= i
#pragma unroll
  for (int j = 0; j < BK; ++j) {
    const int cj = cb[min(kb + j, m - 1)] + kb;
#pragma unroll
    for (int i = j; i < BK; ++i) a[i][j] = (i < w) ? S[cj + i] : make_double2(1.0, 0.0);
  }
  double2 di[BK];
#pragma unroll
  for (int k = 0; k < BK; ++k) {
    di[k] = cinv(a[k][k]);
#pragma unroll
    for (int i = k + 1; i < BK; ++i) {
      const double2 lik = cmul(a[i][k], di[k]);
#pragma unroll
      for (int j = k + 1; j <= i; ++j) a[i][j] = cfms(a[i][j], lik, a[j][k]);
      a[i][k] = lik;
    }
  }
#pragma unroll
  for (int i = 0; i < BK; ++i)
    if (lane == i && i < w) {
#pragma unroll
      for (int j = 0; j <= i; ++j) S[cb[min(kb + j, m - 1)] + kb + i] = a[i][j];
      dinv[i] = di[i];
      dg[kb + i] = a[i][i];
    }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < BK; ++k)
      if (k < w) {
        const double ad = sqrt(cabs2(a[k][k]));
        minp = (ad != ad) ? -1.0 : fmin(minp, ad);
      }
  }
}

}  // namespace

void kh_note_launch() {}

__global__ void probe_diag(double* out, int reps) {
  __shared__ double2 S[4][8 * 10];
  __shared__ double2 dinv[4][8], dg[4][8];
  __shared__ int32_t cb[8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 8) cb[threadIdx.x] = threadIdx.x * 10;
  for (int i = lane; i < 80; i += 32) S[w][i] = make_double2(1.0 + (i % 10 == i / 10 ? 8.0 : 0.01 * i), 0.1);
  __syncthreads();
  double minp = 1e300;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    diag_block_ldlt(S[w], cb, dinv[w], dg[w], 0, 8, 8, minp);
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * 4 + w] = (double)(t1 - t0) / reps + minp * 1e-300;
}

__global__ void probe_diag_regs(double* out, int reps) {
  __shared__ double2 S[4][8 * 10];
  __shared__ double2 dinv[4][8], dg[4][8];
  __shared__ int32_t cb[8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 8) cb[threadIdx.x] = threadIdx.x * 10;
  for (int i = lane; i < 80; i += 32) S[w][i] = make_double2(1.0 + (i % 10 == i / 10 ? 8.0 : 0.01 * i), 0.1);
  __syncthreads();
  double minp = 1e300;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    diag_block_ldlt_regs(S[w], cb, dinv[w], dg[w], 0, 8, 8, minp);
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * 4 + w] = (double)(t1 - t0) / reps + minp * 1e-300;
}

__global__ void probe_tile(double* out, int reps) {
  __shared__ double2 S[2][24 * 34];
  __shared__ double2 W[2][8 * 34];
  __shared__ int32_t cb[24];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 24) cb[threadIdx.x] = threadIdx.x * 34;
  for (int i = lane; i < 24 * 34; i += 32) S[w][i] = make_double2(0.001 * i, 0.0);
  for (int i = lane; i < 8 * 34; i += 32) W[w][i] = make_double2(0.002 * i, 0.1);
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    rank8_tile(S[w], cb, W[w], 34, nullptr, 0, 8, 8 + 8 * (r & 1), 8, 24, 24);
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * 4 + w] = (double)(t1 - t0) / reps;
}

int main() {
  double* d;
  cudaMalloc(&d, 148 * 16 * 4 * 8);
  double h[148 * 16 * 4];
  for (int warps = 1; warps <= 4; warps *= 2)
    for (int ctas = 1; ctas <= 4; ctas *= 2) {
      probe_diag<<<148 * ctas, 32 * warps>>>(d, 200);
      cudaMemcpy(h, d, 8 * 148 * ctas * 4, cudaMemcpyDeviceToHost);
      double s = 0;
      int n = 0;
      for (int b = 0; b < 148 * ctas; ++b)
        for (int w = 0; w < warps; ++w) s += h[b * 4 + w], ++n;
      printf("diag_block_ldlt: %2d warps/SM: %.0f cycles/call\n", warps * ctas, s / n);
    }
  for (int warps = 1; warps <= 4; warps *= 2)
    for (int ctas = 1; ctas <= 4; ctas *= 2) {
      probe_diag_regs<<<148 * ctas, 32 * warps>>>(d, 200);
      cudaMemcpy(h, d, 8 * 148 * ctas * 4, cudaMemcpyDeviceToHost);
      double s = 0;
      int n = 0;
      for (int b = 0; b < 148 * ctas; ++b)
        for (int w = 0; w < warps; ++w) s += h[b * 4 + w], ++n;
      printf("diag_block_ldlt_regs: %2d warps/SM: %.0f cycles/call\n", warps * ctas, s / n);
    }
  for (int warps = 1; warps <= 2; warps *= 2) {
    probe_tile<<<148, 32 * warps, 0>>>(d, 200);
    cudaMemcpy(h, d, 8 * 148 * 4, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int b = 0; b < 148; ++b)
      for (int w = 0; w < warps; ++w) s += h[b * 4 + w];
    printf("rank8_tile: %d warps/SM: %.0f cycles/call\n", warps, s / (148 * warps));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
