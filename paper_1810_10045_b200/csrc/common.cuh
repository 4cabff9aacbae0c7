// common.cuh -- device helpers shared by the lmscale kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

// Device-side bounds checks of the checked build (LMSCALE_DEVICE_CHECKS,
// `python -m paper_1810_10045_b200._build --checked` -> liblmscale_checked.so):
// the stand-in for compute-sanitizer, which is closed on this GPU pool.  A
// failed check prints the condition and traps (the launch fails with an
// error); in the product build the checks compile to nothing.
#ifdef LMSCALE_DEVICE_CHECKS
#define LMS_CHECK(cond)                                                              \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      printf("LMS_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                            \
      __trap();                                                                      \
    }                                                                                \
  } while (0)
#else
#define LMS_CHECK(cond) ((void)0)
#endif

namespace lms {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Decoupled look-back publication (gpu scope, release / acquire).
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// system scope (peer GPUs over NVLink)
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// relaxed (strong) sys-scope store / load: with one fence before the stores
// (or after the polling loads) they form the release (acquire) pattern, and a
// loaded memory system does not pay a fence per access
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Look-back words: bits 31..30 = flag (1 aggregate, 2 inclusive prefix), 29..0 = count.
constexpr uint32_t LB_AGG = 1u << 30;
constexpr uint32_t LB_INC = 2u << 30;
constexpr uint32_t LB_MASK = (1u << 30) - 1u;

// 128-bit loads/stores.  Gradient rows are read exactly once (no L1
// allocation).  The load asm is NOT volatile so the compiler may batch and
// schedule independent loads (volatile asm pins them in program order, which
// serialised the row loads behind their register moves).
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 v;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_cg(const float4* p) { return __ldcg(p); }
__device__ __forceinline__ void st_v4(float4* p, float4 v) { *p = v; }
__device__ __forceinline__ void red_add_v4(float4* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

// Block-wide exclusive scan of one uint32 per thread (blockDim.x <= 1024,
// multiple of 32).  `warp_tot` is shared scratch of >= 32 words.  Returns the
// exclusive prefix; *total receives the block sum (all threads).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* warp_tot,
                                                    uint32_t* total) {
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= (unsigned)o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t t = lane < nwarps ? warp_tot[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(FULL, t, o);
      if (lane >= (unsigned)o) t += y;
    }
    warp_tot[lane] = t;  // inclusive prefix over warps
  }
  __syncthreads();
  uint32_t base = warp ? warp_tot[warp - 1] : 0u;
  *total = warp_tot[nwarps - 1];
  __syncthreads();
  return base + x - v;
}

// Decoupled look-back over tiles for a single running count.  Called by ONE
// thread of the tile; `state` has one word per tile (zeroed before the
// launch).  Returns the exclusive prefix of all earlier tiles.
__device__ __forceinline__ uint32_t lookback_one(uint32_t* state, uint32_t tile,
                                                 uint32_t agg) {
  if (tile == 0) {
    st_release(state, LB_INC | agg);
    return 0u;
  }
  st_release(state + tile, LB_AGG | agg);
  uint32_t excl = 0;
  int t = (int)tile - 1;
  while (true) {
    uint32_t s = ld_acquire(state + t);
    if ((s & ~LB_MASK) == 0u) continue;  // predecessor not published yet
    excl += s & LB_MASK;
    if (s & LB_INC) break;
    --t;
  }
  st_release(state + tile, LB_INC | (excl + agg));
  return excl;
}

// Grid-wide barrier for a normally-launched kernel whose grid is sized to fit
// co-resident (<= occupancy x SMs): a sense-reversing counter in global
// memory, reused across launches (count returns to 0, gen only grows).  Avoids
// cudaLaunchCooperativeKernel, whose launch was measured at ~15-20 us.
struct GridBar {
  uint32_t count;
  uint32_t gen;
};
__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v)
               : "memory");
  return old;
}
// Arrival: atom.inc with wrap-around (the last arriver's increment returns
// the count to 0, no separate reset store) and release semantics; the last
// arriver (acquire: every arrival is in the count's release sequence) bumps
// gen with a release store; the others poll gen with relaxed loads and then
// acquire it with one ld.acquire (SASS: the strong load + CCTL.IVALL) -- a
// fence.acq_rel there (MEMBAR.ALL.GPU) cost ~0.8 us per barrier (S1 1b:
// barrier 2 2.6 -> 1.8 us, step 49.1 -> 47.1 us).  (An acquire load per poll
// and a reset store before the release left ~2.2 us between the last arrival
// and the others passing.)
// gen is loaded BEFORE the CTA's __syncthreads, so its round trip overlaps
// the wait for the CTA's other warps: it cannot change before this CTA
// arrives, and thread 0 has already seen the previous release (coherence).
__device__ __forceinline__ void grid_barrier(GridBar* b) {
  uint32_t gen = 0;
  if (threadIdx.x == 0)
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(&b->gen) : "memory");
  __syncthreads();  // the CTA's writes happen-before thread 0's release below
  if (threadIdx.x == 0) {
    const uint32_t nb = gridDim.x * gridDim.y * gridDim.z;
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;"
                 : "=r"(old) : "l"(&b->count), "r"(nb - 1u) : "memory");
    if (old == nb - 1u) {
      st_release(&b->gen, gen + 1u);
    } else {
      uint32_t g;
      do {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&b->gen) : "memory");
      } while (g == gen);
      // one acquire load of the released gen (synchronises with the last
      // arriver's release store) instead of a fence.acq_rel
      g = ld_acquire(&b->gen);
      asm volatile("" ::"r"(g) : "memory");  // wait for it before the CTA sync
    }
  }
  __syncthreads();  // thread 0's acquire happens-before the CTA's reads
}

// ---- mbarrier + 1-D bulk copies (TMA engine, cp.async.bulk; SASS UBLKCP) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// L2 policy for data read exactly once (gradient rows)
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// global -> shared bulk copy of `bytes` (multiple of 16, both ends 16-byte
// aligned) completing on mbarrier `bar`
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes,
                                              uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// One carveout for every kernel of the library (max shared memory): the SMs
// are then never reconfigured between the step's kernels.
inline void max_carveout(const void* f) {
  static const bool off = getenv("LMSCALE_NO_CARVEOUT") != nullptr;
  if (!off) cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

// ---- compression codec (Sec. 3.3; R15) -------------
// down-cast: round-to-nearest-even of the fp32 product F * x to a 16-bit
// format, saturated to its largest finite value; up-cast: exact widening, then
// one fp32 division by F.  bf == 0: binary16 (the paper's FP16); bf == 1:
// bfloat16.  Payloads travel as raw 16-bit patterns.
__device__ __forceinline__ uint16_t enc1(float x, float F, int bf) {
  const float p = __fmul_rn(F, x);
  if (bf) {
    const float m = 3.3895313892515355e38f;  // largest finite bfloat16
    return __bfloat16_as_ushort(__float2bfloat16_rn(fminf(fmaxf(p, -m), m)));
  }
  return __half_as_ushort(__float2half_rn(fminf(fmaxf(p, -65504.f), 65504.f)));
}
__device__ __forceinline__ float dec1(uint16_t u, float F, int bf) {
  const float v = bf ? __bfloat162float(__ushort_as_bfloat16(u)) : __half2float(__ushort_as_half(u));
  return __fdiv_rn(v, F);
}
__device__ __forceinline__ uint2 enc4(float4 v, float F, int bf) {
  return make_uint2((uint32_t)enc1(v.x, F, bf) | ((uint32_t)enc1(v.y, F, bf) << 16),
                    (uint32_t)enc1(v.z, F, bf) | ((uint32_t)enc1(v.w, F, bf) << 16));
}
__device__ __forceinline__ float4 dec4(uint2 u, float F, int bf) {
  return make_float4(dec1((uint16_t)(u.x & 0xffffu), F, bf), dec1((uint16_t)(u.x >> 16), F, bf),
                     dec1((uint16_t)(u.y & 0xffffu), F, bf), dec1((uint16_t)(u.y >> 16), F, bf));
}

}  // namespace lms
