// Throughput of fp64 mma.sync (DMMA m8n8k4) vs DFMA on one B200: register-only loops, all SMs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/dmma_bench scripts/dmma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.0) out[0] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t] = fma(a, b, c[t]);
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int threads : {128, 256, 512, 1024}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      dmma_loop<<<sms, threads>>>(o, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 256 * 8 * (double)iters * (threads / 32) * sms;
      if (rep) printf("DMMA threads %4d: %.2f TF/s\n", threads, fl / ms / 1e9);
      cudaEventRecord(e0);
      dfma_loop<<<sms, threads>>>(o, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 8 * (double)iters * threads * sms;
      if (rep) printf("DFMA threads %4d: %.2f TF/s\n", threads, fl / ms / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
