// Microbenchmarks of the primitives S1/S3 are built from (sm_100a).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench.cu && ./mb
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__global__ void k_match(uint32_t* out, int iters, uint32_t seed) {
  uint32_t x = seed ^ threadIdx.x, acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    unsigned m = __match_any_sync(0xffffffffu, (x >> 28) & 7u);
    acc += __popc(m);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (uint32_t)(t1 - t0);
  if (acc == 12345) out[1000] = acc;
}

__global__ void k_rankloop(uint32_t* out, int iters) {
  __shared__ uint32_t cnt[16][512];
  for (int i = threadIdx.x; i < 16 * 512; i += blockDim.x) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = threadIdx.x * 2654435761u, acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    uint32_t d = (x >> 23) & 511u;
    unsigned m = __match_any_sync(0xffffffffu, d);
    uint32_t before = cnt[warp][d];
    acc += before + __popc(m & ((1u << lane) - 1));
    __syncwarp();
    if (lane == __ffs(m) - 1) cnt[warp][d] = before + __popc(m);
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (uint32_t)(t1 - t0);
  if (acc == 12345) out[1000] = acc;
}

__global__ void k_rankloop_atom(uint32_t* out, int iters) {
  __shared__ uint32_t cnt[16][512];
  for (int i = threadIdx.x; i < 16 * 512; i += blockDim.x) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = threadIdx.x * 2654435761u, acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    uint32_t d = (x >> 23) & 511u;
    unsigned m = __match_any_sync(0xffffffffu, d);
    const int leader = __ffs(m) - 1;
    uint32_t old = 0;
    if (lane == leader) old = atomicAdd(&cnt[warp][d], (uint32_t)__popc(m));
    old = __shfl_sync(0xffffffffu, old, leader);
    acc += old + __popc(m & ((1u << lane) - 1));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (uint32_t)(t1 - t0);
  if (acc == 12345) out[1000] = acc;
}

// 8 items per thread: all matches first, then the counter updates
__global__ void k_rankloop_batch(uint32_t* out, int iters) {
  __shared__ uint32_t cnt[16][512];
  for (int i = threadIdx.x; i < 16 * 512; i += blockDim.x) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = threadIdx.x * 2654435761u, acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; i += 8) {
    uint32_t d[8];
    unsigned m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x = x * 1664525u + 1013904223u;
      d[j] = (x >> 23) & 511u;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = __match_any_sync(0xffffffffu, d[j]);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int leader = __ffs(m[j]) - 1;
      uint32_t old = 0;
      if (lane == leader) old = atomicAdd(&cnt[warp][d[j]], (uint32_t)__popc(m[j]));
      old = __shfl_sync(0xffffffffu, old, leader);
      acc += old + __popc(m[j] & ((1u << lane) - 1));
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (uint32_t)(t1 - t0);
  if (acc == 12345) out[1000] = acc;
}

__global__ void k_cluster_sync(uint32_t* out, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (uint32_t)(t1 - t0);
}

__global__ void k_dsmem_store(uint32_t* out, int iters, int width) {
  extern __shared__ uint2 buf[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), r = cl.block_rank();
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t pos = (threadIdx.x * 2654435761u + i * 40503u) & 4095u;  // scattered
    int dst = (r + 1 + (threadIdx.x & 7)) % C;
    uint2* p = cl.map_shared_rank(buf, dst);
    p[pos] = make_uint2(i, threadIdx.x);
  }
  cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && r == 0) out[0] = (uint32_t)(t1 - t0);
}

__global__ void k_grid_sync(uint32_t* out, int iters) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (uint32_t)(t1 - t0);
}

__global__ void k_empty() {}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 8192);
  uint32_t h[4];
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  const int it = 1000;
  // match_any alone (16 warps/CTA, 8 CTAs)
  k_match<<<8, 512>>>(d, it, 1);
  cudaMemcpy(h, d, 4, cudaMemcpyDeviceToHost);
  printf("match_any: %.1f cyc/iter (16 warps/SM)\n", h[0] / (double)it);
  k_match<<<8, 32>>>(d, it, 1);
  cudaMemcpy(h, d, 4, cudaMemcpyDeviceToHost);
  printf("match_any: %.1f cyc/iter (1 warp/SM)\n", h[0] / (double)it);
  k_rankloop<<<8, 512>>>(d, it);
  cudaMemcpy(h, d, 4, cudaMemcpyDeviceToHost);
  printf("rank loop (match+lds+2 syncwarp+sts): %.1f cyc/iter (16 warps/SM)\n", h[0] / (double)it);
  k_rankloop_atom<<<8, 512>>>(d, it);
  cudaMemcpy(h, d, 4, cudaMemcpyDeviceToHost);
  printf("rank loop atomic+shfl: %.1f cyc/iter (16 warps/SM)\n", h[0] / (double)it);
  k_rankloop_batch<<<8, 512>>>(d, it);
  cudaMemcpy(h, d, 4, cudaMemcpyDeviceToHost);
  printf("rank loop batched matches + atomic+shfl: %.1f cyc/iter (16 warps/SM)\n", h[0] / (double)it);
  k_rankloop<<<8, 256>>>(d, it);
  cudaMemcpy(h, d, 4, cudaMemcpyDeviceToHost);
  printf("rank loop orig: %.1f cyc/iter (8 warps/SM)\n", h[0] / (double)it);
  for (int C : {2, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaFuncSetAttribute(k_cluster_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchKernelEx(&cfg, k_cluster_sync, d, it);
    cudaError_t e = cudaMemcpy(h, d, 4, cudaMemcpyDeviceToHost);
    printf("cluster.sync C=%d: %.1f cyc (%s)\n", C, h[0] / (double)it, cudaGetErrorString(e));
    cfg.dynamicSmemBytes = 4096 * 8;
    cudaFuncSetAttribute(k_dsmem_store, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchKernelEx(&cfg, k_dsmem_store, d, 64, 8);
    e = cudaMemcpy(h, d, 4, cudaMemcpyDeviceToHost);
    printf("DSMEM 8B scattered stores C=%d: %.1f cyc per 512-thread round (%s)\n", C, h[0] / 64.0,
           cudaGetErrorString(e));
  }
  for (int nb : {8, 64, 148}) {

    int it2 = 100;
    void* args2[] = {&d, &it2};
    cudaLaunchCooperativeKernel((void*)k_grid_sync, nb, 512, args2, 0, 0);
    cudaError_t e = cudaMemcpy(h, d, 4, cudaMemcpyDeviceToHost);
    printf("grid.sync %d CTAs: %.1f cyc (%s)\n", nb, h[0] / 100.0, cudaGetErrorString(e));

  }
  // launch latency: back-to-back empty kernels
  for (int i = 0; i < 10; ++i) k_empty<<<1, 32>>>();
  cudaEventRecord(a);
  for (int i = 0; i < 100; ++i) k_empty<<<1, 32>>>();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("empty kernel back-to-back: %.2f us each\n", ms * 10);
  int dev;
  cudaGetDevice(&dev);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("SM clock attr %d kHz\n", clk);
  return 0;
}
