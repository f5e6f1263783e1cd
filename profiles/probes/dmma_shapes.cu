// Throughput probe of the fp64 mma.sync shapes on sm_100a (design evidence for
// the DMMA kernels): each warp issues independent MMAs into 4 accumulators.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a dmma_shapes.cu -o dmma_shapes
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void probe(double* out, int iters) {
  double a[8], b[4], c[4][4];
  for (int i = 0; i < 8; ++i) a[i] = 1e-9 * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = 1e-9 * (threadIdx.x - i);
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) c[j][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (SHAPE == 0) {  // m8n8k4: 256 FMA
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a[0]), "d"(b[0]));
      } else if (SHAPE == 1) {  // m16n8k4: 512 FMA
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else if (SHAPE == 2) {  // m16n8k8: 1024 FMA
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      } else {  // m16n8k16: 2048 FMA
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) s += c[j][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 1024 * 8);
  const int fma_per[4] = {256, 512, 1024, 2048};
  const char* name[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int s = 0; s < 4; ++s) {
      const int iters = 4096;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto launch = [&]() {
        if (s == 0) probe<0><<<148 * 2, 32 * warps>>>(out, iters);
        if (s == 1) probe<1><<<148 * 2, 32 * warps>>>(out, iters);
        if (s == 2) probe<2><<<148 * 2, 32 * warps>>>(out, iters);
        if (s == 3) probe<3><<<148 * 2, 32 * warps>>>(out, iters);
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * fma_per[s] * 4.0 * iters * 148 * 2 * warps;
      printf("%-9s warps/CTA=%2d (2 CTA/SM): %.2f TFLOP/s\n", name[s], warps, flops / ms / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
