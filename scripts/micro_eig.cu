// Developer microbenchmarks for the persistent eigensolver design (B200):
//   grid barrier latency (148 co-resident CTAs, one atomic counter + generation flag),
//   fp64 DFMA throughput, dependent fp64 division / sqrt chain latency, __syncthreads latency.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/micro_eig scripts/micro_eig.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void grid_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd((unsigned*)gen, 1u);
    } else {
      while (*gen == g) { __nanosleep(20); }
    }
    __threadfence();
  }
  __syncthreads();
}
__device__ __forceinline__ void grid_barrier_spin(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g) : "l"(gen));
    unsigned old;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(count));
    if (old == nblocks - 1) {
      *count = 0;
      asm volatile("st.release.gpu.u32 [%0], %1;" :: "l"(gen), "r"(g + 1));
    } else {
      unsigned cur;
      do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(gen)); } while (cur == g);
    }
  }
  __syncthreads();
}
__global__ void barrier_loop(unsigned* cnt, unsigned* gen, int iters, int spin) {
  for (int i = 0; i < iters; ++i) {
    if (spin) grid_barrier_spin(cnt, gen, gridDim.x);
    else grid_barrier(cnt, gen, gridDim.x);
  }
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
__global__ void div_chain(double* out, int iters, int mode) {
  double x = 1.0 + threadIdx.x * 1e-6, y = 3.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) x = y / x + 1.0;
    else if (mode == 1) x = sqrt(x) + 1.0;
    else x = fma(x, 1.0000001, 1e-9);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (double)(t1 - t0) / iters;
  out[0] = x;
}
__global__ void sync_loop(double* out, int iters) {
  __shared__ double s[1024];
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    s[threadIdx.x] = x;
    __syncthreads();
    x += s[(threadIdx.x + 1) % blockDim.x];
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[1] = (double)(t1 - t0) / iters / 2;
  out[2 + threadIdx.x] = x;
}
int main() {
  unsigned *cnt, *gen;
  double* out;
  cudaMalloc(&cnt, 8);
  cudaMalloc(&gen, 8);
  cudaMemset(cnt, 0, 8);
  cudaMemset(gen, 0, 8);
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int spin = 0; spin < 2; ++spin)
    for (int nb : {16, 74, 148}) {
      barrier_loop<<<nb, 256>>>(cnt, gen, 10, spin);
      cudaEventRecord(e0);
      barrier_loop<<<nb, 256>>>(cnt, gen, 2000, spin);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("grid barrier (%s) %3d CTAs: %.3f us\n", spin ? "acq/rel spin" : "fence+nanosleep", nb, ms * 1e3 / 2000);
    }
  for (int w : {8, 16}) {
    dfma_loop<<<148, 32 * w>>>(out, 10);
    cudaEventRecord(e0);
    dfma_loop<<<148, 32 * w>>>(out, 20000);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA warps/SM %2d: %.2f TFLOP/s fp64\n", w, 148.0 * 32 * w * 20000 * 16 * 2 / (ms * 1e-3) / 1e12);
  }
  double h[2];
  const char* nm[3] = {"fp64 div", "fp64 sqrt", "fp64 fma"};
  for (int mode = 0; mode < 3; ++mode) {
    div_chain<<<1, 32>>>(out, 1000, mode);
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("%s dependent chain: %.1f cycles/op\n", nm[mode], h[1]);
  }
  for (int t : {128, 256, 512, 1024}) {
    sync_loop<<<1, t>>>(out, 1000);
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("__syncthreads + smem round, %4d threads: %.1f cycles\n", t, h[1]);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
