// Microbenchmark (B200): cost of one grid-wide barrier in a persistent cooperative kernel
// (the evaluate kernel's per-sweep synchronisation) vs a thread-block-cluster barrier, and
// of the residual exchange that follows it. nvcc -arch=sm_100a -O3 barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vg = gen;
    const unsigned g = *vg;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*vg == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// same, with acquire/release PTX instead of full fences
__device__ __forceinline__ void grid_barrier2(unsigned* count, unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(count), "r"(1u) : "memory");
    if (old == nblocks - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(count) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gen) : "memory");
    } else {
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(gen) : "memory");
      } while (cur == g);
    }
  }
  __syncthreads();
}

__global__ void k_grid(unsigned* bar, int iters, int mode, unsigned long long* slots, long long* out) {
  long long t0 = clock64();
  unsigned long long acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (mode >= 2 && threadIdx.x < 20) atomicMax(&slots[(i % 3) * 32 + threadIdx.x], (unsigned long long)(blockIdx.x + i));
    if (mode == 0 || mode == 2) grid_barrier(bar, bar + 1, gridDim.x);
    else grid_barrier2(bar, bar + 1, gridDim.x);
    if (mode >= 2 && threadIdx.x < 20) acc += __ldcg(&slots[(i % 3) * 32 + threadIdx.x]);
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
  if (acc == 42) out[1] = acc;
}

__global__ void __cluster_dims__(16, 1, 1) k_cluster16(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
}
__global__ void __cluster_dims__(8, 1, 1) k_cluster8(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
  unsigned* bar;
  unsigned long long* slots;
  long long* out;
  cudaMalloc(&bar, 64);
  cudaMalloc(&slots, 4096);
  cudaMalloc(&out, 64);
  cudaMemset(bar, 0, 64);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 2000;
  for (int cfg = 0; cfg < 3; ++cfg)
    for (int mode = 0; mode < 4; ++mode) {
      const int threads = cfg == 0 ? 256 : cfg == 1 ? 1024 : 288;
      int nb = cfg == 2 ? 592 : 148;
      void* args[] = {&bar, (void*)&iters, &mode, &slots, &out};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaLaunchCooperativeKernel((void*)k_grid, nb, threads, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_grid, nb, threads, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("grid barrier %dx%d mode %d (%s%s): %.3f us per iteration (%s)\n", nb, threads, mode,
             mode & 1 ? "acq/rel PTX" : "threadfence", mode >= 2 ? " + residual atomics/reads" : "",
             ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  for (int cs : {8, 16}) {
    cudaFuncSetAttribute((void*)k_cluster16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    if (cs == 16) k_cluster16<<<144, 1024>>>(iters, out);
    else k_cluster8<<<144, 1024>>>(iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("cluster barrier size %d x1024: %.3f us per iteration (%s)\n", cs, ms * 1e3 / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  int ncl = 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = 144;
  cfg.blockDim = 1024;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = 16;
  at.val.clusterDim.y = at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  cudaOccupancyMaxActiveClusters(&ncl, (void*)k_cluster16, &cfg);
  printf("max active 16-CTA clusters (1024 threads): %d\n", ncl);
  at.val.clusterDim.x = 8;
  cudaOccupancyMaxActiveClusters(&ncl, (void*)k_cluster8, &cfg);
  printf("max active 8-CTA clusters (1024 threads): %d\n", ncl);
  return 0;
}
