// NVLink ceiling probe (2 GPUs, one process, peer access enabled): per
// direction GB/s of the traffic patterns of the fused S5+S6 kernel, both
// GPUs active at once (bidirectional, like the real exchange).
//   pull : cp.async.bulk (TMA) 2 KB rows from the peer into shared memory
//   push : SM 16-byte stores of 2 KB rows into the peer
//   mixed: every CTA pulls one row and pushes one row per item (k_p2p_bulk's
//          mix: peer M rows in, updated E rows out)
//   ce   : cudaMemcpyPeerAsync both ways (copy engines)
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/p2p tools/p2p_probe.cu
//   /tmp/p2p
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

constexpr int ROW = 2048;  // bytes
constexpr int NS = 8;      // ring slots per CTA

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// mode 0 pull, 1 push, 2 mixed.  rows are spread (stride) like scattered table rows.
__global__ void __launch_bounds__(160) k_probe(const char* __restrict__ src, char* __restrict__ dst,
                                               int64_t rows, int mode) {
  __shared__ __align__(128) char ring[NS][ROW];
  __shared__ __align__(8) uint64_t full[NS];
  const int tid = threadIdx.x;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  if (mode == 1) {  // push: 128 threads x 16 B = one row per iteration
    for (int64_t r = r0; r < r1; ++r) {
      if (tid < 128) {
        const int4 v = make_int4((int)r, tid, 1, 2);
        reinterpret_cast<int4*>(dst + r * ROW)[tid] = v;
      }
    }
    return;
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t n = r1 - r0;
  if (tid == 0) {  // producer: prefill the ring
    for (int64_t i = 0; i < n && i < NS; ++i) {
      const uint32_t b = smem_u32(&full[i % NS]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(ROW)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(ring[i % NS])),
          "l"(src + (r0 + i) * ROW), "r"(ROW), "r"(b)
          : "memory");
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    const int s = (int)(i % NS);
    const uint32_t b = smem_u32(&full[s]);
    const uint32_t ph = (uint32_t)((i / NS) & 1);
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(ok)
          : "r"(b), "r"(ph)
          : "memory");
    int4 v = make_int4(0, 0, 0, 0);
    if (tid < 128) v = reinterpret_cast<const int4*>(ring[s])[tid];
    if (mode == 2 && tid < 128) reinterpret_cast<int4*>(dst + (r0 + i) * ROW)[tid] = v;
    __syncthreads();
    if (tid == 0 && i + NS < n) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(ROW)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(ring[s])),
          "l"(src + (r0 + i + NS) * ROW), "r"(ROW), "r"(b)
          : "memory");
    }
    if (mode == 0 && tid < 128 && v.x == 0x7fffffff) dst[0] = 1;  // keep the loads alive
  }
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("needs 2 GPUs\n");
    return 0;
  }
  const int64_t bytes = 1ll << 30;  // 1 GiB per buffer
  const int64_t rows = bytes / ROW;
  char *a[2], *b[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&a[d], bytes));
    CK(cudaMalloc(&b[d], bytes));
    CK(cudaMemset(a[d], d + 1, bytes));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const char* names[] = {"pull (bulk copy from peer)", "push (SM stores to peer)",
                         "mixed (pull a row + push a row)"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int cps : {1, 2, 4, 8}) {
      float best = 0.f;
      for (int rep = 0; rep < 3; ++rep) {
        for (int d = 0; d < 2; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventRecord(e0[d], st[d]));
          // GPU d reads the peer's a and writes the peer's b (mixed) / its own b (pull)
          char* dst = mode == 0 ? b[d] : b[1 - d];
          k_probe<<<sms * cps, 160, 0, st[d]>>>(a[1 - d], dst, rows, mode);
          CK(cudaGetLastError());
          CK(cudaEventRecord(e1[d], st[d]));
        }
        float ms = 0.f;
        for (int d = 0; d < 2; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventSynchronize(e1[d]));
          float t = 0.f;
          CK(cudaEventElapsedTime(&t, e0[d], e1[d]));
          if (t > ms) ms = t;
        }
        // per direction: pull or push moves `bytes` each way; mixed moves
        // `bytes` in (pulls) and `bytes` out (pushes) per GPU, i.e. 2x bytes on
        // every direction of the link (the peer's pulls and pushes)
        const double dir = mode == 2 ? 2.0 * bytes : (double)bytes;
        const float gbs = (float)(dir / (ms * 1e-3) / 1e9);
        if (gbs > best) best = gbs;
      }
      printf("%-34s %d CTA/SM: %7.1f GB/s per direction\n", names[mode], cps, best);
    }
  }
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaSetDevice(0));
    CK(cudaEventRecord(e0[0], st[0]));
    CK(cudaMemcpyPeerAsync(b[1], 1, a[0], 0, bytes, st[0]));
    CK(cudaEventRecord(e1[0], st[0]));
    CK(cudaSetDevice(1));
    CK(cudaEventRecord(e0[1], st[1]));
    CK(cudaMemcpyPeerAsync(b[0], 0, a[1], 1, bytes, st[1]));
    CK(cudaEventRecord(e1[1], st[1]));
    float ms = 0.f;
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventSynchronize(e1[d]));
      float t;
      CK(cudaEventElapsedTime(&t, e0[d], e1[d]));
      if (t > ms) ms = t;
    }
    printf("%-34s        : %7.1f GB/s per direction\n", "copy engines (cudaMemcpyPeerAsync)",
           (float)(bytes / (ms * 1e-3) / 1e9));
  }
  return 0;
}
