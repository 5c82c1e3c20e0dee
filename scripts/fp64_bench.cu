// fp64 throughput microbenchmark (developer tool): DMMA.8x8x4 (mma.sync f64) vs DFMA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/fp64_bench scripts/fp64_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
  double d[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double d[16];
  for (int j = 0; j < 16; ++j) d[j] = threadIdx.x + j;
  const double a = 1.0000001, b = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) d[j] = fma(d[j], a, b);
  }
  double s = 0;
  for (int j = 0; j < 16; ++j) s += d[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out;
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int w : {4, 8, 16}) {
    dmma_loop<<<148, 32 * w>>>(out, 10);
    cudaEventRecord(e0);
    dmma_loop<<<148, 32 * w>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 148.0 * w * iters * 8 * 256 * 2;
    printf("DMMA warps/SM %2d: %.2f TFLOP/s fp64\n", w, flops / (ms * 1e-3) / 1e12);
    dfma_loop<<<148, 32 * w>>>(out, 10);
    cudaEventRecord(e0);
    dfma_loop<<<148, 32 * w>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double f2 = 148.0 * 32 * w * iters * 16 * 2;
    printf("DFMA warps/SM %2d: %.2f TFLOP/s fp64\n", w, f2 / (ms * 1e-3) / 1e12);
  }
  return 0;
}
