// Global-atomic latency / contention probe (sm_100a): one phase of S1 issues
// ~1 atomicAdd-with-return per distinct id per CTA; how long does a burst of
// them take when many CTAs hit the same (Zipf-head) addresses?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ap tools/atomic_probe.cu && /tmp/ap
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void k_atom(uint32_t* cnt, int per_thread, int naddr, int ret, uint32_t* out,
                       unsigned long long* t) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  uint32_t acc = 0;
  for (int i = 0; i < per_thread; ++i) {
    const uint32_t a = (uint32_t)(blockIdx.x * 7919u + threadIdx.x * 104729u + i * 31u) % naddr;
    if (ret)
      acc += atomicAdd(cnt + a, 1u);
    else
      atomicAdd(cnt + a, 1u);  // result unused: RED
  }
  __syncthreads();
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) {
    atomicMin(t, t0);
    atomicMax(t + 1, t1);
  }
  if (acc == 0xdeadbeef) out[0] = acc;
}

int main() {
  uint32_t* cnt;
  cudaMalloc(&cnt, 64 << 20);
  cudaMemset(cnt, 0, 64 << 20);
  uint32_t* out;
  cudaMalloc(&out, 64);
  unsigned long long* t;
  cudaMalloc(&t, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int ret : {1, 0})
    for (int naddr : {1, 16, 150, 4096, 1 << 20})
      for (int pt : {1, 8}) {
        for (int blocks : {148, 32}) {
          float best = 1e9;
          for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            k_atom<<<blocks, 512>>>(cnt, pt, naddr, ret, out, t);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
          }
          printf("ret=%d addrs=%8d atomics/thread=%d ctas=%3d total=%7d : %8.2f us\n", ret, naddr,
                 pt, blocks, blocks * 512 * pt, best * 1e3);
        }
      }
  return 0;
}
