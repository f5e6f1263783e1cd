// FP64 vector (DFMA) throughput on sm_100a: 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tput(double* out, int n) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double y = 0.999999, c = 1e-9;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], y, c);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* d;
  cudaMalloc(&d, 148 * 8 * 1024 * 8);
  for (int warps = 1; warps <= 32; warps *= 2) {
    const int n = 20000;
    tput<<<148, 32 * warps>>>(d, n);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    tput<<<148, 32 * warps>>>(d, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 8 * n * 148.0 * 32 * warps;
    printf("warps/SM %2d: %.2f TFLOP/s (DFMA), %.2f cycles per warp-DFMA per SM\n", warps, fl / ms / 1e9,
           (ms * 1e-3 * 1.965e9) / (8.0 * n * warps));
  }
  return 0;
}
