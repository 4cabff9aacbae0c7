// seeding.cu -- Sec. 3.2: sampled-softmax candidates drawn from a
// seed shared by a group of GPUs, so the group's candidates coincide and the
// output-embedding exchange keeps a small global unique set.
//
// Draw stream (R16): x_i = floor(u_i * V / 2^64), u_i = mix64(A + i),
// A = mix64(seed ^ mix64(step)); the candidates are the first S distinct x_i in
// stream order (uniform without replacement).  One CTA: each round draws 1024
// stream values, keeps those whose value was not drawn at a smaller stream
// index (a shared-memory hash set holding, per value, the smallest index),
// and appends the kept ones in stream order (block prefix sum) until S are
// accepted.  S is small (1024 per GPU in the paper): latency-bound.
#include <cstdint>
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace lms {

namespace {

constexpr int DR_THREADS = 1024;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Shared-memory hash set of the values drawn so far, each with the smallest
// stream index that drew it (atomicMin).  A draw i with value x is new iff,
// after the round's insertions, the slot of x holds i: values accepted in an
// earlier round keep their smaller index, and within a round only the first
// occurrence matches.  Kept draws are appended in stream order (block scan).
constexpr int DR_HBITS = 14;
constexpr int DR_HSIZE = 1 << DR_HBITS;  // >= 2 * (DRAW_MAX_S + DR_THREADS)
constexpr uint32_t DR_EMPTY = 0xffffffffu;  // ids are < vocab <= 2^32 - 1
static_assert(DR_HSIZE >= DRAW_MAX_S + DR_THREADS, "hash set too small");

__global__ void __launch_bounds__(DR_THREADS) k_draw_samples(uint64_t seed, uint64_t step,
                                                             int S, uint64_t V,
                                                             uint32_t* __restrict__ out) {
  extern __shared__ uint32_t dsm[];
  uint32_t* hkey = dsm;             // DR_HSIZE values
  uint32_t* hidx = dsm + DR_HSIZE;  // smallest stream index per value
  __shared__ uint32_t s_scan[DR_THREADS / 32 + 1];
  const int tid = threadIdx.x;
  for (int i = tid; i < DR_HSIZE; i += DR_THREADS) {
    hkey[i] = DR_EMPTY;
    hidx[i] = 0xffffffffu;
  }
  __syncthreads();
  const uint64_t A = mix64(seed ^ mix64(step));
  int count = 0;
  uint32_t base = 0;
  while (count < S) {
    const uint32_t i = base + (uint32_t)tid;
    const uint32_t x = (uint32_t)__umul64hi(mix64(A + i), V);
    uint32_t h = (x * 0x9E3779B1u) >> (32 - DR_HBITS);
    for (;;) {
      const uint32_t prev = atomicCAS(hkey + h, DR_EMPTY, x);
      if (prev == DR_EMPTY || prev == x) break;
      h = (h + 1) & (DR_HSIZE - 1);
    }
    atomicMin(hidx + h, i);
    __syncthreads();
    const bool fresh = hidx[h] == i;
    uint32_t total;
    const uint32_t pos = block_excl_scan(fresh ? 1u : 0u, s_scan, &total);
    if (fresh && count + (int)pos < S) out[count + pos] = x;
    count = min(S, count + (int)total);
    base += DR_THREADS;
  }
}

}  // namespace

cudaError_t launch_draw_samples(uint64_t seed, uint64_t step, int S, uint64_t V, uint32_t* out,
                                cudaStream_t s) {
  constexpr size_t smem = 2 * DR_HSIZE * sizeof(uint32_t);
  static bool once = (cudaFuncSetAttribute(k_draw_samples,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem), true);
  (void)once;
  k_draw_samples<<<1, DR_THREADS, smem, s>>>(seed, step, S, V, out);
  return cudaGetLastError();
}

// Seed-group plan (R16): number of groups by policy, ranks in
// contiguous near-equal blocks, seed of group q = mix64(master + q).
int plan_seed_groups(int world, int policy, double alpha, uint64_t master, uint64_t* seeds) {
  int n = 0;
  switch (policy) {
    case 0: n = world; break;                                            // all distinct
    case 1: n = 1; break;                                                // all same
    case 2: n = (int)std::floor(std::log((double)world) / std::log(2.0) + 0.5); break;
    case 3: n = (int)std::floor(std::log((double)world) + 0.5); break;   // ln
    case 4: n = (int)std::floor(std::log((double)world) / std::log(10.0) + 0.5); break;
    case 5:
      if (!(alpha > 0.0 && alpha <= 1.0)) return -1;
      n = (int)std::ceil(std::pow((double)world, alpha));
      break;
    default: return -1;
  }
  if (n < 1) n = 1;
  if (n > world) n = world;
  for (int r = 0; r < world; ++r)
    seeds[r] = mix64(master + (uint64_t)(((int64_t)r * n) / world));
  return n;
}

}  // namespace lms
