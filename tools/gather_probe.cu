// Row-gather bandwidth probe (sm_100a): how fast can one SM pull randomly
// permuted rows of 2-8 KB from HBM into shared memory?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gp tools/gather_probe.cu && /tmp/gp
// Modes: 0 = cp.async.bulk per row (mbarrier ring, 1 producer warp),
//        2 = plain 128-bit loads into registers (8 rows in flight per warp).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));          \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\nWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar) : "memory");
}

constexpr int MAXS = 32;

// mode 0: npw producer warps (the last ones) issue one bulk copy per row,
// group g by producer warp g % npw; consumers (nct threads) sum.  The
// range's row indices are staged in shared memory first.
constexpr int MAXL = 4096;
__global__ void k_bulk(const float4* __restrict__ src, const int* __restrict__ perm, int nrows,
                       int rowv, int GR, int NS, int npw, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[2 * MAXS];
  __shared__ int s_row[MAXL];
  const int nct = blockDim.x - 32 * npw;
  const int rb = rowv * 16;
  const int b = blockIdx.x, nb = gridDim.x;
  const int p0 = (int)((int64_t)b * nrows / nb), p1 = (int)((int64_t)(b + 1) * nrows / nb);
  const int L = min(p1 - p0, MAXL), ng = (L + GR - 1) / GR;
  const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * MAXS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, nct / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < L; i += blockDim.x) s_row[i] = perm[p0 + i];
  __syncthreads();
  if ((int)threadIdx.x >= nct) {
    const int lane = threadIdx.x & 31, pw = (threadIdx.x - nct) >> 5;
    for (int g = pw; g < ng; g += npw) {
      const int s = g % NS, it = g / NS;
      if (it > 0) mbar_wait(empty0 + 8 * s, (it - 1) & 1);
      const int n = min(GR, L - g * GR);
      if (lane == 0) mbar_arrive_tx(full0 + 8 * s, n * rb);
      __syncwarp();
      if (lane < n)
        bulk_g2s(smem_u32(smem + (size_t)s * GR * rb + (size_t)lane * rb),
                 src + (size_t)s_row[g * GR + lane] * rowv, rb, full0 + 8 * s);
    }
    return;
  }
  float4 acc = make_float4(0, 0, 0, 0);
  for (int g = 0; g < ng; ++g) {
    const int s = g % NS, it = g / NS;
    mbar_wait(full0 + 8 * s, it & 1);
    const int n = min(GR, L - g * GR);
    const float4* slot = reinterpret_cast<const float4*>(smem + (size_t)s * GR * rb);
    for (int j = 0; j < n; ++j)
      for (int c = threadIdx.x; c < rowv; c += nct) {
        float4 v = slot[j * rowv + c];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(empty0 + 8 * s);
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

// mode 2: warp per row, 8 rows in flight per warp, 16 B per lane per load
__global__ void k_ldg(const float4* __restrict__ src, const int* __restrict__ perm, int nrows,
                      int rowv, float* out) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r0 = warp * 8; r0 < nrows; r0 += nw * 8) {
    for (int c = lane; c < rowv; c += 32) {
      float4 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        v[q] = r0 + q < nrows ? __ldcs(src + (size_t)perm[r0 + q] * rowv + c) : make_float4(0, 0, 0, 0);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        acc.x += v[q].x; acc.y += v[q].y; acc.z += v[q].z; acc.w += v[q].w;
      }
    }
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t total = 1ull << 30;  // 1 GiB of rows
  float4* src;
  CK(cudaMalloc(&src, total));
  CK(cudaMemset(src, 0, total));
  float* out;
  CK(cudaMalloc(&out, 64));
  int* perm;
  const int maxrows = (int)(total / 2048);
  CK(cudaMalloc(&perm, sizeof(int) * maxrows));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rb : {2048, 4096, 8192}) {
    const int rowv = rb / 16;
    const int nrows = (int)(total / rb) / 2;  // 512 MB moved
    std::vector<int> h(nrows);
    for (int i = 0; i < nrows; ++i) h[i] = i;
    srand(7);
    for (int i = nrows - 1; i > 0; --i) std::swap(h[i], h[rand() % (i + 1)]);
    CK(cudaMemcpy(perm, h.data(), sizeof(int) * nrows, cudaMemcpyHostToDevice));
    auto time = [&](auto launch) {
      launch();
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) launch();
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      return (double)nrows * rb * 5 / (ms * 1e-3) / 1e9;
    };
    // mode 0: bulk copies (rows per CTA capped at MAXL: use enough CTAs)
    for (int cps : {1, 2})
      for (int npw : {1, 2, 4, 8})
        for (int GR : {2, 4, 8}) {
          const int ringkb = 192 / cps;
          int NS = ringkb * 1024 / (GR * rb);
          if (NS < 2) continue;
          if (NS > MAXS) NS = MAXS;
          const size_t sm = (size_t)NS * GR * rb;
          CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
          const int nct = std::min(512, std::max(32, rowv));
          const int grid = std::max(sms * cps, (nrows + MAXL - 1) / MAXL);
          double gbs = time([&] {
            k_bulk<<<grid, nct + 32 * npw, sm>>>(src, perm, nrows, rowv, GR, NS, npw, out);
          });
          printf("row %5d B  bulk   ctas/SM %d producers %d GR %d NS %2d grid %d : %7.0f GB/s\n", rb,
                 cps, npw, GR, NS, grid, gbs);
        }
    // mode 2: plain loads
    for (int cps : {1, 2, 4, 8}) {
      double gbs = time([&] { k_ldg<<<sms * cps, 256, 0>>>(src, perm, nrows, rowv, out); });
      printf("row %5d B  ldg    ctas/SM %d (8 warps, 8 rows in flight/warp)        : %7.0f GB/s\n", rb,
             cps, gbs);
    }
  }
  return 0;
}
