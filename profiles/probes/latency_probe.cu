// Dependent-chain latencies on sm_100a (cycles per op, one warp per SM):
// DFMA, DMUL, DMMA.8x8x4, SHFL, LDS.128, MUFU.RCP64H-based reciprocal.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, int n) {
  __shared__ double2 buf[64];
  const int lane = threadIdx.x;
  buf[lane] = make_double2(lane, 0);
  buf[lane + 32] = make_double2(lane + 32, 0);
  __syncwarp();
  double x = 1.0 + lane * 1e-3, y = 0.999;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
  t1 = clock64();
  if (lane == 0) out[0] = (double)(t1 - t0) / n;
  // DMMA chain
  double c0 = x, c1 = x;
  t0 = clock64();
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(y), "d"(y));
  t1 = clock64();
  if (lane == 0) out[1] = (double)(t1 - t0) / n;
  // SHFL chain (double = 2 SHFL, the 2nd independent)
  int v = lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
  t1 = clock64();
  if (lane == 0) out[2] = (double)(t1 - t0) / n;
  // LDS.128 chain
  int idx = lane;
  double acc = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const double2 q = buf[idx];
    idx = ((int)q.x + 1) & 63;
  }
  t1 = clock64();
  if (lane == 0) out[3] = (double)(t1 - t0) / n;
  // reciprocal chain
  double r = 1.5 + lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) r = __drcp_rn(r) + 1.0;
  t1 = clock64();
  if (lane == 0) out[4] = (double)(t1 - t0) / n;
  // DMUL chain
  double m = 1.0000001;
  t0 = clock64();
  for (int i = 0; i < n; ++i) m = m * y;
  t1 = clock64();
  if (lane == 0) out[5] = (double)(t1 - t0) / n;
  out[8 + lane] = x + c0 + c1 + v + idx + acc + r + m;
}

int main() {
  double* d;
  cudaMalloc(&d, 64 * 8);
  lat<<<1, 32>>>(d, 1000);
  lat<<<1, 32>>>(d, 1000);
  double h[6];
  cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
  const char* nm[6] = {"DFMA", "DMMA.8x8x4", "SHFL(int)", "LDS.128", "drcp_rn+DADD", "DMUL"};
  for (int i = 0; i < 6; ++i) printf("%-14s %6.1f cycles\n", nm[i], h[i]);
  return 0;
}
