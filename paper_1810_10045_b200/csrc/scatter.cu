// scatter.cu -- S6, the duplicate-free row update of step 7 (P:421,
// P:433-435) for the staged path, the S0 dense comparison scatter
// (P:313-319), the compression codec (R15), the consistency checksum and the
// forward lookup, for sm_100a.  (S4 is in segsum.cu.)
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace lms {

namespace {

// Vector traits: float4 (128-bit path, dim % 4 == 0) or float (any dim).
template <typename T>
struct Vec;
template <>
struct Vec<float4> {
  static constexpr int W = 4;
  __device__ __forceinline__ static float4 zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ __forceinline__ static float4 ld_once(const float4* p) { return ld_stream(p); }
  __device__ __forceinline__ static float4 ld_l2(const float4* p) { return ld_cg(p); }
  __device__ __forceinline__ static void st(float4* p, float4 v) { st_v4(p, v); }
  __device__ __forceinline__ static float4 add(float4 a, float4 b) { return f4add(a, b); }
  __device__ __forceinline__ static float4 fma(float s, float4 a, float4 b) {
    return make_float4(__fmaf_rn(s, a.x, b.x), __fmaf_rn(s, a.y, b.y), __fmaf_rn(s, a.z, b.z),
                       __fmaf_rn(s, a.w, b.w));
  }
};
template <>
struct Vec<float> {
  static constexpr int W = 1;
  __device__ __forceinline__ static float zero() { return 0.f; }
  __device__ __forceinline__ static float ld_once(const float* p) { return __ldcs(p); }
  __device__ __forceinline__ static float ld_l2(const float* p) { return __ldcg(p); }
  __device__ __forceinline__ static void st(float* p, float v) { *p = v; }
  __device__ __forceinline__ static float add(float a, float b) { return a + b; }
  __device__ __forceinline__ static float fma(float s, float a, float b) {
    return __fmaf_rn(s, a, b);
  }
};

}  // namespace

// ------------------------------------------------------------------- S6
// table[ids[r]] = fma(-lr, rows[r], table[ids[r]]) for r < n.  One warp per
// row at a time (rows are disjoint: P:433-435), 128-bit accesses.
template <typename T>
__global__ void __launch_bounds__(256) k_update(float* __restrict__ table, int D,
                                                const uint32_t* __restrict__ ids,
                                                const float* __restrict__ rows, int64_t n,
                                                const Sc3* __restrict__ n_dev, float lr) {
  using V = Vec<T>;
  if (n_dev) {  // device-side count (no host round trip); nothing on an id error
    if (n_dev->err & 1u) return;
    n = min(n, n_dev->u_global);
  }
  const int C = D / V::W;
  const int lane = (int)lane_id();
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T* R = reinterpret_cast<const T*>(rows);
  T* E = reinterpret_cast<T*>(table);
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nwarps) {
    const uint32_t w = __ldg(ids + r);
    const T* src = R + (size_t)r * C;
    T* dst = E + (size_t)w * C;
    int col = lane;
    for (; col + 96 < C; col += 128) {
      T m0 = V::ld_once(src + col), m1 = V::ld_once(src + col + 32);
      T m2 = V::ld_once(src + col + 64), m3 = V::ld_once(src + col + 96);
      T e0 = dst[col], e1 = dst[col + 32], e2 = dst[col + 64], e3 = dst[col + 96];
      V::st(dst + col, V::fma(-lr, m0, e0));
      V::st(dst + col + 32, V::fma(-lr, m1, e1));
      V::st(dst + col + 64, V::fma(-lr, m2, e2));
      V::st(dst + col + 96, V::fma(-lr, m3, e3));
    }
    for (; col < C; col += 32) V::st(dst + col, V::fma(-lr, V::ld_once(src + col), dst[col]));
  }
}

void launch_update(float* table, int D, const uint32_t* ids, const float* rows, int64_t n,
                   const Sc3* n_dev, float lr, int num_sms, cudaStream_t s) {
  if (n <= 0) return;
  int64_t blocks = (n + 7) / 8;
  const int64_t cap = (int64_t)num_sms * 8;
  if (blocks > cap) blocks = cap;
  const bool v4 = D % 4 == 0 && (uintptr_t)table % 16 == 0 && (uintptr_t)rows % 16 == 0;
  static bool once = (max_carveout((const void*)k_update<float4>),
                      max_carveout((const void*)k_update<float>), true);
  (void)once;
  if (v4)
    k_update<float4><<<(unsigned)blocks, 256, 0, s>>>(table, D, ids, rows, n, n_dev, lr);
  else
    k_update<float><<<(unsigned)blocks, 256, 0, s>>>(table, D, ids, rows, n, n_dev, lr);
}

// ------------------------------------------------------------------- S0
// Dense comparison path: table[ids[q]] += -lr * grad[q] for every one of the
// n gathered tokens, 128-bit vector reductions at L2 (red.global.add.v4.f32):
// the GPU analogue of the paper's locked row updates.
__global__ void __launch_bounds__(256) k_dense_v4(float* __restrict__ table, int D,
                                                  const uint32_t* __restrict__ ids,
                                                  const float* __restrict__ grad, int64_t n,
                                                  float lr, uint32_t vocab) {
  const int C = D / 4;
  const int lane = (int)lane_id();
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float4* G4 = reinterpret_cast<const float4*>(grad);
  float4* E4 = reinterpret_cast<float4*>(table);
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < n; q += nwarps) {
    const uint32_t w = __ldg(ids + q);
    if (w >= vocab) continue;
    const float4* src = G4 + (size_t)q * C;
    float4* dst = E4 + (size_t)w * C;
    for (int col = lane; col < C; col += 32) {
      float4 v = ld_stream(src + col);
      red_add_v4(dst + col, make_float4(-lr * v.x, -lr * v.y, -lr * v.z, -lr * v.w));
    }
  }
}
__global__ void __launch_bounds__(256) k_dense_s(float* __restrict__ table, int D,
                                                 const uint32_t* __restrict__ ids,
                                                 const float* __restrict__ grad, int64_t n,
                                                 float lr, uint32_t vocab) {
  const int lane = (int)lane_id();
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < n; q += nwarps) {
    const uint32_t w = __ldg(ids + q);
    if (w >= vocab) continue;
    for (int col = lane; col < D; col += 32)
      atomicAdd(table + (size_t)w * D + col, -lr * __ldcs(grad + (size_t)q * D + col));
  }
}

void launch_dense(float* table, int D, const uint32_t* ids, const float* grad, int64_t n,
                  float lr, uint32_t vocab, int num_sms, cudaStream_t s) {
  if (n <= 0) return;
  int64_t blocks = (n + 7) / 8;
  const int64_t cap = (int64_t)num_sms * 8;
  if (blocks > cap) blocks = cap;
  const bool v4 = D % 4 == 0 && (uintptr_t)table % 16 == 0 && (uintptr_t)grad % 16 == 0;
  if (v4)
    k_dense_v4<<<(unsigned)blocks, 256, 0, s>>>(table, D, ids, grad, n, lr, vocab);
  else
    k_dense_s<<<(unsigned)blocks, 256, 0, s>>>(table, D, ids, grad, n, lr, vocab);
}

}  // namespace lms

namespace lms {
// ------------------------------------------------------------ codec (R15)
// q[i] = binary16 bits of RNE(fp32(F * x[i])), saturated.
__global__ void __launch_bounds__(256) k_compress(const float* __restrict__ x, int64_t n, float F,
                                                  int bf, uint16_t* __restrict__ q) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    q[i] = enc1(__ldcs(x + i), F, bf);
}
// x[i] = fp32(q[i]) / F.
__global__ void __launch_bounds__(256) k_decompress(const uint16_t* __restrict__ q, int64_t n,
                                                    float F, int bf, float* __restrict__ x) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = dec1(q[i], F, bf);
}

cudaError_t launch_codec(bool down, const void* in, int64_t n, float F, int bf, void* out,
                         int num_sms, cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
  if (blocks < 1) blocks = 1;
  if (down)
    k_compress<<<(unsigned)blocks, 256, 0, s>>>((const float*)in, n, F, bf, (uint16_t*)out);
  else
    k_decompress<<<(unsigned)blocks, 256, 0, s>>>((const uint16_t*)in, n, F, bf, (float*)out);
  return cudaGetLastError();
}
}  // namespace lms

namespace lms {
// ------------------------------------------- consistency check (debug)
// out[0] = U_g, out[1] = sum over r < U_g of mix(I^[r] + r * 2^32): every
// rank computes I^ redundantly, so the pairs must agree everywhere.
__device__ __forceinline__ uint64_t ck_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void __launch_bounds__(1024) k_checksum(const uint32_t* __restrict__ ihat,
                                                   const Sc3* __restrict__ sc3,
                                                   unsigned long long* __restrict__ out) {
  __shared__ unsigned long long part[32];
  const int64_t ug = sc3->u_global;
  unsigned long long h = 0;
  for (int64_t r = threadIdx.x; r < ug; r += blockDim.x)
    h += ck_mix((uint64_t)ihat[r] + ((uint64_t)r << 32));
  for (int o = 16; o; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = h;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
    out[0] = (unsigned long long)ug;
    out[1] = t;
  }
}
cudaError_t launch_checksum(const uint32_t* ihat, const Sc3* sc3, unsigned long long* out,
                            cudaStream_t s) {
  k_checksum<<<1, 1024, 0, s>>>(ihat, sc3, out);
  return cudaGetLastError();
}

// ------------------------------------------------ forward lookup
// out[p, :] = E[ids[p], :] -- the input-embedding projection of the K tokens
// (SURVEY 8(f) row 4).  Warp per row, grid-stride, 128-bit accesses when the
// rows allow; an id >= vocab gives a zero row.
template <typename T>
__global__ void __launch_bounds__(256) k_lookup(const float* __restrict__ table, int D,
                                                const uint32_t* __restrict__ ids, int64_t n,
                                                uint32_t vocab, float* __restrict__ out) {
  const int C = D / (int)(sizeof(T) / sizeof(float));
  const int lane = threadIdx.x & 31;
  const T* E = reinterpret_cast<const T*>(table);
  T* O = reinterpret_cast<T*>(out);
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n; p += nw) {
    const uint32_t w = __ldg(ids + p);
    const T* src = E + (size_t)w * C;
    T* dst = O + (size_t)p * C;
    if (w < vocab) {
      int c = lane;
      for (; c + 96 < C; c += 128) {
        const T a0 = __ldg(src + c), a1 = __ldg(src + c + 32), a2 = __ldg(src + c + 64),
                a3 = __ldg(src + c + 96);
        __stcs(dst + c, a0);
        __stcs(dst + c + 32, a1);
        __stcs(dst + c + 64, a2);
        __stcs(dst + c + 96, a3);
      }
      for (; c < C; c += 32) __stcs(dst + c, __ldg(src + c));
    } else {
      for (int c = lane; c < C; c += 32) dst[c] = T{};
    }
  }
}

cudaError_t launch_lookup(const float* table, int D, const uint32_t* ids, int64_t n,
                          uint32_t vocab, float* out, int num_sms, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 7) / 8;
  if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
  const bool v4 = D % 4 == 0 && (uintptr_t)table % 16 == 0 && (uintptr_t)out % 16 == 0;
  if (v4)
    k_lookup<float4><<<(unsigned)blocks, 256, 0, s>>>(table, D, ids, n, vocab, out);
  else
    k_lookup<float><<<(unsigned)blocks, 256, 0, s>>>(table, D, ids, n, vocab, out);
  return cudaGetLastError();
}
}  // namespace lms
