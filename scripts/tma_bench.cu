// TMA throughput microbenchmark (developer tool, not part of the library):
// every CTA streams boxes of a [D][rows][n] fp32 tensor through a ring of stages and only
// waits/re-arms the barriers.  Reports bytes per clock per SM for several box shapes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_bench scripts/tma_bench.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128) tma_stream(const __grid_constant__ CUtensorMap map, int box_inner,
                                                     int box_rows, int rows, int n, int D, int iters, int stages, int nbx,
                                                     long long* clk, int lanes_issuers, int shared_mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int box_bytes = box_inner * box_rows * 4 * nbx;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + stages * box_bytes);
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages * max((int)(blockDim.x / 32), lanes_issuers); ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int lanes_mode = blockDim.x <= 32 && lanes_issuers > 1;
  const int nw = lanes_mode ? lanes_issuers : blockDim.x / 32;
  const int w = lanes_mode ? threadIdx.x : threadIdx.x / 32;
  if (lanes_mode ? (threadIdx.x >= lanes_issuers) : ((threadIdx.x & 31) != 0)) return;
  bars += w * stages;
  smem += w * stages * box_bytes;
  const int nrb = rows / box_rows, ncb = n / box_inner;
  long long t0 = clock64();
  uint32_t phase = 0;
  for (int it = 0; it < iters; ++it) {
    const int st = it % stages;
    if (it >= stages) {
      // wait for the load issued `stages` iterations ago
      uint32_t ok = 0;
      const uint32_t par = ((it / stages) - 1) & 1;
      while (!ok)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0,1,0,P;\n\t}"
                     : "=r"(ok) : "r"(su32(&bars[st])), "r"(par));
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[st])), "r"(box_bytes));
    for (int b = 0; b < nbx; ++b) {
      const long long g = shared_mode ? (((long long)(blockIdx.x % shared_mode) * nw + w) * iters + it) * nbx + b : (((long long)blockIdx.x * nw + w) * iters + it) * nbx + b;
      const int cb = (int)(g % ncb), rb = (int)((g / ncb) % nrb), z = (int)((g / ((long long)ncb * nrb)) % D);
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
          ::"r"(su32(smem + st * box_bytes + b * (box_bytes / nbx))), "l"(&map), "r"(su32(&bars[st])), "r"(cb * box_inner), "r"(rb * box_rows), "r"(z)
          : "memory");
    }
  }
  for (int k = 0; k < stages; ++k) {
    const int it = iters + k;
    const int st = it % stages;
    uint32_t ok = 0;
    const uint32_t par = ((it / stages) - 1) & 1;
    while (!ok)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0,1,0,P;\n\t}"
                   : "=r"(ok) : "r"(su32(&bars[st])), "r"(par));
  }
  if (w == 0) clk[blockIdx.x] = clock64() - t0;
}

int main() {
  const int rows = 1080 / 8 * 8, n = 1920, D = 64;
  float* X;
  cudaMalloc(&X, (size_t)D * 1080 * n * 4);
  cudaMemset(X, 0, (size_t)D * 1080 * n * 4);
  long long* clk;
  cudaMalloc(&clk, 4 * 148 * 8);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  struct Cfg { int inner, brows; CUtensorMapSwizzle sw; int stages; int nbx; int warps; int cps; };
  std::vector<Cfg> cfgs = {{32, 128, CU_TENSOR_MAP_SWIZZLE_128B, 2, 1, -4, 1}, {32, 128, CU_TENSOR_MAP_SWIZZLE_128B, 1, 1, -8, 1}};
  for (int Dv : {64})
  for (int shm : {0, 1, 9, 37})
  for (int grid : {148}) {
    for (auto c : cfgs) {
      CUtensorMap map;
      cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)1080, (cuuint64_t)Dv};
      cuuint64_t str[2] = {(cuuint64_t)n * 4, (cuuint64_t)1080 * n * 4};
      cuuint32_t box[3] = {(cuuint32_t)c.inner, (cuuint32_t)c.brows, 1};
      cuuint32_t es[3] = {1, 1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       c.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
      const int box_bytes = c.inner * c.brows * 4 * c.nbx;
      const int nis = c.warps < 0 ? -c.warps : c.warps;
      const int smem = nis * c.stages * box_bytes + 1024 + 256 * nis;
      cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const int iters = (int)((64LL << 20) / box_bytes);  // 64 MB per CTA
      tma_stream<<<grid * c.cps, c.warps < 0 ? 32 : 32 * c.warps, smem>>>(map, c.inner, c.brows, rows, n, Dv, iters / 8, c.stages, c.nbx, clk, c.warps < 0 ? -c.warps : 1, shm);  // warm
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      tma_stream<<<grid * c.cps, c.warps < 0 ? 32 : 32 * c.warps, smem>>>(map, c.inner, c.brows, rows, n, Dv, iters, c.stages, c.nbx, clk, c.warps < 0 ? -c.warps : 1, shm);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<long long> h(grid * c.cps);
      cudaMemcpy(h.data(), clk, grid * c.cps * 8, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (auto v : h) mx = v > mx ? v : mx;
      const double bytes = (double)iters * box_bytes * nis * c.cps;
      printf("shared %2d D %2d grid %3d warps %d ctas/sm %d box {%3d x %3d} x%d sw=%d stages %2d: %.1f B/clk/SM, total %.2f TB/s  (%s)\n", shm, Dv, grid, c.warps, c.cps, c.inner,
             c.brows, c.nbx, (int)c.sw, c.stages, bytes / mx, bytes * grid / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
    }
  }
  return 0;
}
