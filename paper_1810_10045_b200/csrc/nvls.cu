// nvls.cu -- S5 + S6 fused over NVLink SHARP multicast (NVLS): the all-reduce
// of M (step 6) and the duplicate-free row update of E (step 7,
// P:421) in ONE kernel, through NCCL 2.28's device API.
//
// M (U_g x D, one copy per rank) sits in an NCCL symmetric window with a
// multicast (multimem) mapping on the NVSwitch.  Rank i owns rows r = i mod G:
//   1. LSA barrier: every rank's M_g is complete (S4 ran before on each rank);
//   2. for each owned row: multimem.ld_reduce (the switch sums the G copies),
//      e' = fma(-lr, m, E[I^[r]]) written to the local E, and multimem.st of e'
//      into M[r] of every rank (the owner's result is the only one, so the
//      replicas stay bit-identical);
//   3. LSA barrier: all broadcasts landed;
//   4. for every row of the other slices: E[I^[r]] = M[r] (local copy).
// Per GPU that is ~1x the payload each way over NVLink (a ring all-reduce
// moves 2(G-1)/G x), no separate 12*U_g*D update pass, and no host round trip:
// U_g is read on the device.  Barriers are per CTA index: CTA k of every rank
// handles the same relative rows of every slice, so CTA k only has to meet the
// CTAs k of the other ranks.
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace lms {

namespace {

constexpr int NV_THREADS = 512;
constexpr int NV_WARPS = NV_THREADS / 32;

__device__ __forceinline__ float4 mm_ld_reduce(const float4* p) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ float mm_ld_reduce(const float* p) {
  float v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mm_st(float4* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mm_st(float* p, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ float4 fma4(float s, float4 a, float4 b) {
  return make_float4(__fmaf_rn(s, a.x, b.x), __fmaf_rn(s, a.y, b.y), __fmaf_rn(s, a.z, b.z),
                     __fmaf_rn(s, a.w, b.w));
}
__device__ __forceinline__ float fma4(float s, float a, float b) { return __fmaf_rn(s, a, b); }
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float add4(float a, float b) { return a + b; }
__device__ __forceinline__ float4 dech(uint2 u, float F, int bf) { return dec4(u, F, bf); }
__device__ __forceinline__ float dech(uint16_t h, float F, int bf) { return dec1(h, F, bf); }
__device__ __forceinline__ uint2 ench(float4 v, float F, int bf) { return enc4(v, F, bf); }
__device__ __forceinline__ uint16_t ench(float v, float F, int bf) { return enc1(v, F, bf); }

}  // namespace

struct NvlsKernelArgs {
  ncclDevComm dev;
  ncclWindow_t win;
  const uint32_t* ihat;
  const Sc3* sc3;
  float* table;
  const float* M;  // local view of this rank's M
  int D;
  float lr;
  int rank, world;
  unsigned long long* trace;
  int diag;  // timing diagnostics only (LMSCALE_NVLS_DIAG): 1 no broadcast, 2 no reduce
  size_t lbits_off;  // byte offset of each rank's local presence bitmap in the M window
  ncclWindow_t twin;  // non-null: the table is in a symmetric window; updated rows are
                      // multicast straight into every replica of E (no copy phase)
  float cF;           // compression scale F (k_p2p_update_c)
  int cbf;            // codec: 0 binary16, 1 bfloat16
  size_t mhat_off;    // byte offset of the compressed M^ rows in the M window
  size_t lrank_off;   // local-slot layout: byte offset of lrank in the window
  int local_m;        // 1: M_j rows are at rank j's local index (lrank + popcount), else at r
  int pb_slots;       // k_p2p_bulk: shared-memory ring slots
  int pb_rows;        // k_p2p_bulk: rows per presence-table batch (<= PB_MAXROWS)
  int64_t mcap;       // rows of every rank's M (bounds of the checked build)
  uint32_t vocab;
  // emulation (lmscale_emulate_step): each rank's M-window base and table
  char* emu_m[8];
  float* emu_t[8];
};

// Peer access of the P2P kernels.  Product (EMU = false): the NCCL symmetric
// windows (LSA pointers over NVLink) and per-CTA-index LSA barriers.
// Emulation (EMU = true, lmscale_emulate_step): the G ranks are G contexts on
// one GPU whose kernels run one after the other, the window bases are those
// contexts' buffers, and the launch order gives what the barriers give (every
// rank's S4 before any exchange; compressed: every phase 1 before any phase 2).
template <bool EMU>
__device__ __forceinline__ char* peer_m(const NvlsKernelArgs& a, int j) {
  if constexpr (EMU)
    return a.emu_m[j];
  else
    return reinterpret_cast<char*>(ncclGetLsaPointer(a.win, 0, j));
}
template <bool EMU>
__device__ __forceinline__ float* peer_t(const NvlsKernelArgs& a, int j) {
  if constexpr (EMU)
    return a.emu_t[j];
  else
    return reinterpret_cast<float*>(ncclGetLsaPointer(a.twin, 0, j));
}
template <bool EMU>
struct PeerBar;
template <>
struct PeerBar<false> {
  ncclCoopCta cta;
  ncclLsaBarrierSession<ncclCoopCta> s;
  __device__ explicit PeerBar(const NvlsKernelArgs& a)
      : s(cta, a.dev, ncclTeamTagLsa{}, blockIdx.x, /*multimem=*/true) {}
  __device__ void sync() { s.sync(cta, cuda::memory_order_acq_rel); }
};
template <>
struct PeerBar<true> {
  __device__ explicit PeerBar(const NvlsKernelArgs&) {}
  __device__ void sync() { __syncthreads(); }
};

__device__ __forceinline__ void nv_stamp(unsigned long long* tr, int i) {
  if (tr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[i] = t;
  }
}
// latest over the CTAs (trace slot reset by the host before the step)
__device__ __forceinline__ void nv_stamp_max(unsigned long long* tr, int i) {
  if (tr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(tr + i, t);
  }
}

template <typename T>
__global__ void __launch_bounds__(NV_THREADS, 1) k_nvls_update(NvlsKernelArgs a) {
  constexpr int W = sizeof(T) / sizeof(float);
  nv_stamp(a.trace, 48);
  ncclCoopCta cta;
  ncclLsaBarrierSession<ncclCoopCta> bar(cta, a.dev, ncclTeamTagLsa{}, blockIdx.x,
                                         /*multimem=*/true);
  bar.sync(cta, cuda::memory_order_acq_rel);  // every rank's M_g is complete
  // an id >= vocab on any rank (S3's error bit is the OR over ranks): every
  // rank leaves here, no table row is touched (lmscale_sync semantics)
  if (__ldcg(&a.sc3->err) & 1u) return;
  nv_stamp(a.trace, 49);

  const int64_t Ug = a.sc3->u_global;
  const int C = a.D / W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * NV_WARPS + warp;
  const int64_t nw = (int64_t)gridDim.x * NV_WARPS;
  T* mc = reinterpret_cast<T*>(ncclGetLsaMultimemPointer(a.win, 0, a.dev));
  T* E = reinterpret_cast<T*>(a.table);
  T* mcE = a.twin ? reinterpret_cast<T*>(ncclGetLsaMultimemPointer(a.twin, 0, a.dev)) : nullptr;
  const T* Ml = reinterpret_cast<const T*>(a.M);

  // owned rows r = rank + G*t (interleaved over the id space, so every rank
  // gets the same mix of hot and cold rows): reduce through the switch,
  // update, broadcast the new rows
  {
    for (int64_t t = gw; a.rank + a.world * t < Ug; t += nw) {
      const int64_t r = a.rank + a.world * t;
      const size_t wrow = (size_t)__ldg(a.ihat + r) * C;
      T* er = E + wrow;
      T* mr = mc + (size_t)r * C;
      T* dst = mcE ? mcE + wrow : mr;  // multicast target: E replicas, or M
      int c = lane;
      // 8 independent multicast reductions (+ 8 local E loads) in flight per lane
      for (; c + 224 < C; c += 256) {
        T m[8], e[8];
        if (a.diag == 2) {
#pragma unroll
          for (int q = 0; q < 8; ++q) m[q] = __ldcg(reinterpret_cast<const T*>(a.M) + (mr - mc) + c + 32 * q);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) m[q] = mm_ld_reduce(mr + c + 32 * q);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) e[q] = er[c + 32 * q];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          e[q] = fma4(-a.lr, m[q], e[q]);
          if (!mcE) er[c + 32 * q] = e[q];
        }
        if (a.diag != 1) {
#pragma unroll
          for (int q = 0; q < 8; ++q) mm_st(dst + c + 32 * q, e[q]);
        }
      }
      for (; c < C; c += 32) {
        const T e = fma4(-a.lr, mm_ld_reduce(mr + c), er[c]);
        if (!mcE) er[c] = e;
        mm_st(dst + c, e);
      }
    }
  }
  nv_stamp(a.trace, 50);
  bar.sync(cta, cuda::memory_order_acq_rel);  // the other ranks' rows have landed
  nv_stamp(a.trace, 51);
  if (mcE) {  // every replica already holds every updated row
    nv_stamp(a.trace, 52);
    return;
  }

  // rows owned by the other ranks: copy the broadcast result into E
  for (int j = 0; j < a.world; ++j) {
    if (j == a.rank) continue;
    for (int64_t t = gw; j + a.world * t < Ug; t += nw) {
      const int64_t r = j + a.world * t;
      T* er = E + (size_t)__ldg(a.ihat + r) * C;
      const T* mr = Ml + (size_t)r * C;
      int c = lane;
      for (; c + 96 < C; c += 128) {
        const T v0 = __ldcg(mr + c), v1 = __ldcg(mr + c + 32);
        const T v2 = __ldcg(mr + c + 64), v3 = __ldcg(mr + c + 96);
        er[c] = v0;
        er[c + 32] = v1;
        er[c + 64] = v2;
        er[c + 96] = v3;
      }
      for (; c < C; c += 32) er[c] = __ldcg(mr + c);
    }
  }
  nv_stamp(a.trace, 52);
}

// S5+S6 over direct NVLink loads/stores (LSA peer pointers) for small G:
// rank i owns rows r = i mod G; per owned row it loads the G copies of M[r]
// (its own and the peers', summed in rank order -- the order of S:142), forms
// e' = fma(-lr, m, E[I^[r]]) and stores e' into every rank's table window.
// Per GPU and direction that is (G-1)/G x payload for the loads plus the same
// for the stores -- 1x at G = 2, where multicast needs (1 + 1/G) = 1.5x.
template <typename T, bool EMU>
__global__ void __launch_bounds__(NV_THREADS, 1) k_p2p_update(NvlsKernelArgs a) {
  constexpr int W = sizeof(T) / sizeof(float);
  constexpr int MAXG = 8;
  PeerBar<EMU> bar(a);
  bar.sync();  // every rank's M_g is complete
  // an id >= vocab on any rank (S3's error bit is the OR over ranks): every
  // rank leaves here, no table row is touched (lmscale_sync semantics)
  if (__ldcg(&a.sc3->err) & 1u) return;
  const int64_t Ug = a.sc3->u_global;
  const int C = a.D / W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * NV_WARPS + warp;
  const int64_t nw = (int64_t)gridDim.x * NV_WARPS;
  const T* pm[MAXG];
  T* pe[MAXG];
#pragma unroll
  for (int j = 0; j < MAXG; ++j) {
    pm[j] = j < a.world ? reinterpret_cast<const T*>(peer_m<EMU>(a, j)) : nullptr;
    pe[j] = j < a.world ? reinterpret_cast<T*>(peer_t<EMU>(a, j)) : nullptr;
  }
  const uint32_t* pb[MAXG];  // each rank's local presence bitmap (S1's lbits)
  const uint32_t* pr[MAXG];  // each rank's lrank (local-slot layout)
#pragma unroll
  for (int j = 0; j < MAXG; ++j) {
    const char* base = j < a.world ? peer_m<EMU>(a, j) : nullptr;
    pb[j] = reinterpret_cast<const uint32_t*>(base + a.lbits_off);
    pr[j] = reinterpret_cast<const uint32_t*>(base + a.lrank_off);
  }
  const T* E = reinterpret_cast<const T*>(a.table);
  for (int64_t t = gw; a.rank + a.world * t < Ug; t += nw) {
    const int64_t r = a.rank + a.world * t;
    const uint32_t w = __ldg(a.ihat + r);
    const size_t wrow = (size_t)w * C;
    const size_t mrow = (size_t)r * C;
    // which ranks hold word w: only their copies of M[r] are loaded (absent
    // ranks' rows are never written: S4 skips the zero-fill on this path)
    uint32_t has = 0;
    size_t lrow[MAXG];  // row of word w in rank j's M
#pragma unroll
    for (int j = 0; j < MAXG; ++j) {
      lrow[j] = mrow;
      if (j < a.world) {
        const uint32_t bits = __ldcg(pb[j] + (w >> 5));
        has |= ((bits >> (w & 31u)) & 1u) << j;
        if (a.local_m)
          lrow[j] = (size_t)(__ldcg(pr[j] + (w >> 5)) + __popc(bits & ((1u << (w & 31u)) - 1u))) * C;
      }
    }
    for (int c = lane; c < C; c += 128) {
      T m[4], e[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) m[q] = T{};
#pragma unroll
      for (int j = 0; j < MAXG; ++j) {
        if ((has >> j) & 1u) {
          T v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            v[q] = (c + 32 * q < C) ? __ldcg(pm[j] + lrow[j] + c + 32 * q) : T{};
#pragma unroll
          for (int q = 0; q < 4; ++q) m[q] = add4(m[q], v[q]);  // rank order
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c + 32 * q < C) e[q] = fma4(-a.lr, m[q], E[wrow + c + 32 * q]);
#pragma unroll
      for (int j = 0; j < MAXG; ++j) {
        if (j < a.world) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (c + 32 * q < C) __stcg(pe[j] + wrow + c + 32 * q, e[q]);
        }
      }
    }
  }
  bar.sync();  // every replica holds every updated row
}


// S5+S6 over NVLink with the row traffic on the TMA engine (default P2P
// kernel for dim % 4 == 0): each CTA owns every gridDim-th of this rank's
// rows r = rank + G t.  After the first LSA barrier, the CTA looks up, for all
// its rows at once, which ranks hold word I^[r] (peers' presence bitmaps) and
// where (lrank + popcount); then a producer warp streams, per (row, column
// block of <= 2 KB), the present copies of M[r] from the peers' windows and
// the local E block into a shared-memory slot with cp.async.bulk (one
// mbarrier per slot), while consumer threads sum the copies in rank order,
// form fma(-lr, m, e) and store it into every replica of the table.  Bytes in
// flight cost no registers, and no per-row chain of remote loads remains.
constexpr int PB_CB = 512;        // floats per column block (2 KB)
constexpr int PB_MAXROWS = 1024;  // owned rows per CTA (presence table in smem)
constexpr int PB_THREADS = PB_CB / 4 + 32;
constexpr int PB_MAXSLOTS = 16;
constexpr int PB_MAX_CPS = 4;     // k_p2p_bulk CTAs per SM (LSA barrier count)

template <bool EMU>
__global__ void __launch_bounds__(PB_THREADS) k_p2p_bulk(NvlsKernelArgs a) {
  constexpr int MAXG = 8;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[2 * PB_MAXSLOTS];
  __shared__ uint32_t s_w[PB_MAXROWS];
  __shared__ uint8_t s_has[PB_MAXROWS];
  const int G = a.world, tid = threadIdx.x, nct = PB_CB / 4;
  const int NS = a.pb_slots;
  const uint32_t SB = (uint32_t)(G + 1) * PB_CB * 4;  // a slot: <= G copies + the E block
  uint32_t* s_lrow = reinterpret_cast<uint32_t*>(smem + (size_t)NS * SB);  // [rows][G]
  (void)0;
  const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8u * PB_MAXSLOTS;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full0 + 8u * s, 1u);
      mbar_init(empty0 + 8u * s, (uint32_t)(nct / 32));
    }
    fence_mbar_init();
  }
  nv_stamp(a.trace, 48);
  const bool err = __ldcg(&a.sc3->err) & 1u;  // id error on some rank (OR over ranks)
  const int64_t Ug = a.sc3->u_global;
  const int64_t T = Ug > a.rank ? (Ug - a.rank + G - 1) / G : 0;  // this rank's rows
  // this CTA's rows: t = blockIdx.x + i * gridDim.x (interleaved: the Zipf head
  // -- rows held by every rank, the most copies to load -- is spread over all
  // CTAs; contiguous blocks left the first CTAs 40 % behind at tieba G = 2)
  const int64_t nb = gridDim.x;
  const int64_t nmine = T > (int64_t)blockIdx.x ? (T - blockIdx.x + nb - 1) / nb : 0;
  const int D = a.D;
  const int ncb = (D + PB_CB - 1) / PB_CB;
  const int lane = tid & 31;
  const uint32_t* pbits[MAXG];
  const uint32_t* prank[MAXG];
#pragma unroll
  for (int j = 0; j < MAXG; ++j) {
    const char* base = j < G ? peer_m<EMU>(a, j) : nullptr;
    pbits[j] = reinterpret_cast<const uint32_t*>(base + a.lbits_off);
    prank[j] = reinterpret_cast<const uint32_t*>(base + a.lrank_off);
  }
  // ---- presence and row of word I^[r] on every rank, for a batch of rows:
  // the G ranks' presence bitmaps and per-word local prefixes, all of a row's
  // loads issued together (a chain of 2G remote loads per row cost 12 us at
  // 1b G = 2)
  auto presence = [&](int64_t b0, int nrows) {
    for (int i = tid; i < nrows; i += blockDim.x) {
      const int64_t r = a.rank + (int64_t)G * ((int64_t)blockIdx.x + (b0 + i) * nb);
      const uint32_t w = __ldg(a.ihat + r);
      uint32_t bw[MAXG], lw[MAXG];
#pragma unroll
      for (int j = 0; j < MAXG; ++j) {
        bw[j] = j < G ? __ldcg(pbits[j] + (w >> 5)) : 0u;
        lw[j] = (j < G && a.local_m) ? __ldcg(prank[j] + (w >> 5)) : 0u;
      }
      uint32_t has = 0;
#pragma unroll
      for (int j = 0; j < MAXG; ++j) {
        if (j >= G) break;
        const uint32_t bits = bw[j];
        has |= ((bits >> (w & 31u)) & 1u) << j;
        uint32_t lrow = (uint32_t)r;
        if (a.local_m) lrow = lw[j] + __popc(bits & ((1u << (w & 31u)) - 1u));
        LMS_CHECK(lrow < (uint32_t)a.mcap);
        s_lrow[i * G + j] = lrow;
      }
      LMS_CHECK(w < a.vocab);
      s_w[i] = w;
      s_has[i] = (uint8_t)has;
    }
  };
  // In the local-slot layout (peer S3) every rank's S1 -- the bitmaps and
  // prefixes read here -- completed before S3's handshake, so the first
  // batch's table is built while the barrier waits for the peers' S4.
  const bool early = a.local_m && !err;
  nv_stamp(a.trace, 44);
  const int BR = a.pb_rows;
  if (early) presence(0, (int)(nmine < BR ? nmine : BR));
  nv_stamp(a.trace, 45);
  PeerBar<EMU> bar(a);
  bar.sync();  // every rank's M_g is complete
  // the peers' generic-proxy stores of M_g, now acquired, are read below by
  // bulk copies (async proxy)
  asm volatile("fence.proxy.async.global;" ::: "memory");
  nv_stamp(a.trace, 49);
  if (err) return;  // all ranks leave, no table row is touched
  int it0 = 0;  // items issued / consumed before this batch (ring phase continuity)
  for (int64_t b0 = 0; b0 < nmine; b0 += BR) {
    const int nrows = (int)(nmine - b0 < BR ? nmine - b0 : BR);
    if (b0 > 0 || !early) presence(b0, nrows);
    __syncthreads();
    if (b0 == 0) nv_stamp_max(a.trace, 47);
    const int items = nrows * ncb;
    if (tid >= nct) {
      // -------------------------------------------------------- producer warp
      const char* pm =
          (lane < G) ? peer_m<EMU>(a, lane) : nullptr;
      for (int q = 0; q < items; ++q) {
        const int it = it0 + q;
        const int s = it % NS, ph = it / NS;
        if (ph > 0) mbar_wait(empty0 + 8u * s, (uint32_t)(ph - 1) & 1u);
        const int i = q / ncb, cb = q % ncb;
        const int cw = min(PB_CB, D - cb * PB_CB);
        const uint32_t bytes = (uint32_t)cw * 4u;
        const uint32_t has = s_has[i];
        const int n = __popc(has);
        if (lane == 0) mbar_arrive_tx(full0 + 8u * s, (uint32_t)(n + 1) * bytes);
        __syncwarp();
        const uint32_t dst = smem_u32(smem) + (uint32_t)s * SB;
        if (lane < G && ((has >> lane) & 1u)) {
          const int k = __popc(has & ((1u << lane) - 1u));  // rank order
          bulk_g2s(dst + (uint32_t)k * PB_CB * 4,
                   pm + ((size_t)s_lrow[i * G + lane] * D + (size_t)cb * PB_CB) * 4, bytes,
                   full0 + 8u * s);
        }
        if (lane == 31)
          bulk_g2s(dst + (uint32_t)n * PB_CB * 4,
                   a.table + (size_t)s_w[i] * D + (size_t)cb * PB_CB, bytes, full0 + 8u * s);
      }
    } else {
      // ----------------------------------------------------------- consumers
      float4* pe[MAXG];
#pragma unroll
      for (int j = 0; j < MAXG; ++j)
        pe[j] = j < G ? reinterpret_cast<float4*>(peer_t<EMU>(a, j)) : nullptr;
      const int t = tid;
      for (int q = 0; q < items; ++q) {
        const int it = it0 + q;
        const int s = it % NS, ph = it / NS;
        const int i = q / ncb, cb = q % ncb;
        const int cw = min(PB_CB, D - cb * PB_CB) / 4;
        mbar_wait(full0 + 8u * s, (uint32_t)ph & 1u);
        if (t < cw) {
          const float4* slot = reinterpret_cast<const float4*>(smem + (size_t)s * SB);
          const int n = __popc((uint32_t)s_has[i]);
          float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int k = 0; k < n; ++k) m = add4(m, slot[k * (PB_CB / 4) + t]);  // rank order
          const float4 e = fma4(-a.lr, m, slot[n * (PB_CB / 4) + t]);
          const size_t off = ((size_t)s_w[i] * D + (size_t)cb * PB_CB) / 4 + t;
#pragma unroll
          for (int j = 0; j < MAXG; ++j)
            if (j < G) __stcg(pe[j] + off, e);
        }
        __syncwarp();
        if ((t & 31) == 0) mbar_arrive(empty0 + 8u * s);
      }
    }
    it0 += items;
    __syncthreads();  // the batch's presence table is no longer read
  }
  nv_stamp(a.trace, 50);
  nv_stamp_max(a.trace, 53);
  bar.sync();  // every replica holds every updated row
  nv_stamp(a.trace, 51);
  nv_stamp(a.trace, 52);
}


// Compressed S5+S6 (Sec. 3.3; R15): the all-reduce as a
// reduce-scatter and an all-gather, each carrying binary16 payloads.
//   1. LSA barrier: every rank's compressed M_g (written by S4) is complete;
//   2. rank i owns rows r = i mod G: it loads the copies of the ranks that hold
//      word I^[r] (peers' presence bitmaps), up-casts, divides by F, sums in
//      fp32 in rank order, compresses the sum and stores it into every rank's
//      M^ region (P2P stores, half the bytes of fp32 rows);
//      (the owner also updates its own E row right away from the decoded
//      compressed sum, the value every other rank will apply);
//   3. LSA barrier: every compressed row of M^ has landed;
//   4. every rank updates the other ranks' rows of its own E from its local
//      M^: E[I^[r]] = fma(-lr, dec(M^[r]), E[I^[r]]) -- the same instruction on
//      the same bits on every rank, so the replicas stay bit-identical.
// Per GPU and direction: (G-1)/G x (present rows + U_g rows) x 2 bytes x D.
// PH: 0 the product kernel (both phases, LSA barriers); emulation: 1 phase
// 1 only, 2 phase 2 only (every rank's phase 1 is launched first).
template <typename T, int PH>
__global__ void __launch_bounds__(NV_THREADS, 1) k_p2p_update_c(NvlsKernelArgs a) {
  constexpr int W = sizeof(T) / sizeof(float);
  using H = typename std::conditional<W == 4, uint2, uint16_t>::type;
  constexpr int MAXG = 8;
  constexpr bool EMU = PH != 0;
  PeerBar<EMU> bar(a);
  bar.sync();  // every rank's compressed M_g is complete
  // an id >= vocab on any rank (S3's error bit is the OR over ranks): every
  // rank leaves here, no table row is touched (lmscale_sync semantics)
  if (__ldcg(&a.sc3->err) & 1u) return;
  const int64_t Ug = a.sc3->u_global;
  const int C = a.D / W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * NV_WARPS + warp;
  const int64_t nw = (int64_t)gridDim.x * NV_WARPS;
  const float F = a.cF;
  const H* pm[MAXG];
  H* pq[MAXG];
  const uint32_t* pb[MAXG];
  const uint32_t* pr[MAXG];
#pragma unroll
  for (int j = 0; j < MAXG; ++j) {
    char* base = j < a.world ? peer_m<EMU>(a, j) : nullptr;
    pm[j] = reinterpret_cast<const H*>(base);
    pq[j] = reinterpret_cast<H*>(base + a.mhat_off);
    pb[j] = reinterpret_cast<const uint32_t*>(base + a.lbits_off);
    pr[j] = reinterpret_cast<const uint32_t*>(base + a.lrank_off);
  }
  T* Eo = reinterpret_cast<T*>(a.table);
  for (int64_t t = gw; PH != 2 && a.rank + a.world * t < Ug; t += nw) {
    const int64_t r = a.rank + a.world * t;
    const uint32_t w = __ldg(a.ihat + r);
    const size_t mrow = (size_t)r * C;
    uint32_t has = 0;
    size_t lrow[MAXG];  // row of word w in rank j's M
#pragma unroll
    for (int j = 0; j < MAXG; ++j) {
      lrow[j] = mrow;
      if (j < a.world) {
        const uint32_t bits = __ldcg(pb[j] + (w >> 5));
        has |= ((bits >> (w & 31u)) & 1u) << j;
        if (a.local_m)
          lrow[j] = (size_t)(__ldcg(pr[j] + (w >> 5)) + __popc(bits & ((1u << (w & 31u)) - 1u))) * C;
      }
    }
    T* er = Eo + (size_t)w * C;  // this rank's own row of E (updated here, not in phase 2)
    for (int c = lane; c < C; c += 128) {
      T m[4], ev[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        m[q] = T{};
        if (c + 32 * q < C) ev[q] = er[c + 32 * q];
      }
#pragma unroll
      for (int j = 0; j < MAXG; ++j) {
        if ((has >> j) & 1u) {
          H v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (c + 32 * q < C) v[q] = pm[j][lrow[j] + c + 32 * q];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (c + 32 * q < C) m[q] = add4(m[q], dech(v[q], F, a.cbf));  // rank order, fp32
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (c + 32 * q < C) {
          const H e = ench(m[q], F, a.cbf);
#pragma unroll
          for (int j = 0; j < MAXG; ++j)
            if (j < a.world && j != a.rank) pq[j][mrow + c + 32 * q] = e;
          // the owner applies the same decoded value every other rank applies
          er[c + 32 * q] = fma4(-a.lr, dech(e, F, a.cbf), ev[q]);
        }
      }
    }
  }
  if (PH == 1) return;
  if (PH == 0) bar.sync();  // every compressed row of M^ has landed
  const H* Q = reinterpret_cast<const H*>(reinterpret_cast<const char*>(a.M) + a.mhat_off);
  T* E = reinterpret_cast<T*>(a.table);
  // rows in the same (owner, t) order as phase 1: the barrier above is per
  // CTA index, so CTA k may only read the rows that CTAs k wrote
  for (int j = 0; j < a.world; ++j) {
  if (j == a.rank) continue;  // own rows were updated in phase 1
  for (int64_t t = gw; j + a.world * t < Ug; t += nw) {
    const int64_t r = j + a.world * t;
    T* er = E + (size_t)__ldg(a.ihat + r) * C;
    const H* qr = Q + (size_t)r * C;
    for (int c = lane; c < C; c += 128) {
      H v[4];
      T e[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c + 32 * q < C) {
          v[q] = __ldcg(qr + c + 32 * q);
          e[q] = er[c + 32 * q];
        }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c + 32 * q < C) er[c + 32 * q] = fma4(-a.lr, dech(v[q], F, a.cbf), e[q]);
    }
  }
  }
}

// ---------------------------------------------------------------- host side

struct NvlsState {
  ncclWindow_t win = nullptr;
  ncclDevComm dev{};
  bool dev_ok = false;
  int ctas = 0;
};

NvlsState* nvls_create(ncclComm_t comm, void* M, size_t bytes, int num_sms, char* err,
                       size_t errlen) {
  NvlsState* st = new NvlsState();
  st->ctas = num_sms;  // one CTA per SM (measured: 128 -> 148 CTAs, 1b G=4 264 -> 260 us)
  if (const char* e = getenv("LMSCALE_NVLS_CTAS")) st->ctas = atoi(e);
  ncclResult_t r = ncclCommWindowRegister(comm, M, bytes, &st->win, NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess) {
    snprintf(err, errlen, "ncclCommWindowRegister: %s", ncclGetErrorString(r));
    delete st;
    return nullptr;
  }
  ncclDevCommRequirements req{};
  req.lsaMultimem = true;
  req.lsaBarrierCount = PB_MAX_CPS * st->ctas;  // k_p2p_bulk runs up to PB_MAX_CPS CTAs per SM
  r = ncclDevCommCreate(comm, &req, &st->dev);
  if (r != ncclSuccess) {
    snprintf(err, errlen, "ncclDevCommCreate(lsaMultimem): %s", ncclGetErrorString(r));
    ncclCommWindowDeregister(comm, st->win);
    delete st;
    return nullptr;
  }
  if (!st->dev.lsaMultimem.mcBasePtr) {
    snprintf(err, errlen, "no multimem (NVLS) mapping on this communicator");
    ncclDevCommDestroy(comm, &st->dev);
    ncclCommWindowDeregister(comm, st->win);
    delete st;
    return nullptr;
  }
  st->dev_ok = true;
  return st;
}

void nvls_destroy(ncclComm_t comm, NvlsState* st) {
  if (!st) return;
  if (st->dev_ok) ncclDevCommDestroy(comm, &st->dev);
  if (st->win) ncclCommWindowDeregister(comm, st->win);
  delete st;
}

__global__ void k_peer_bases(ncclWindow_t win, int world, void** out) {
  if ((int)threadIdx.x < world) out[threadIdx.x] = ncclGetLsaPointer(win, 0, (int)threadIdx.x);
}

// LSA base address of every rank's M window (plain device pointers over
// NVLink), for kernels outside this file that read peer memory directly.
bool nvls_peer_bases(NvlsState* st, int world, void** out_host) {
  void** d = nullptr;
  if (cudaMalloc(&d, 8 * sizeof(void*)) != cudaSuccess) return false;
  k_peer_bases<<<1, 32>>>(st->win, world, d);
  const bool ok = cudaMemcpy(out_host, d, world * sizeof(void*), cudaMemcpyDeviceToHost) ==
                  cudaSuccess;
  cudaFree(d);
  return ok;
}

bool nvls_use_p2p(int world) {
  static const int p2p_max =
      getenv("LMSCALE_P2P_MAX_G") ? atoi(getenv("LMSCALE_P2P_MAX_G")) : 8;
  return world <= p2p_max && world <= 8;
}

ncclWindow_t nvls_register_table(ncclComm_t comm, void* table, size_t bytes, char* err,
                                 size_t errlen) {
  ncclWindow_t w = nullptr;
  ncclResult_t r = ncclCommWindowRegister(comm, table, bytes, &w, NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess) {
    snprintf(err, errlen, "ncclCommWindowRegister(table): %s", ncclGetErrorString(r));
    return nullptr;
  }
  return w;
}

void nvls_deregister_table(ncclComm_t comm, ncclWindow_t w) {
  if (w) ncclCommWindowDeregister(comm, w);
}

// The P2P fused kernel: k_p2p_bulk (rows staged by bulk copies) when rows
// are 16-byte vectors, else k_p2p_update (warp loads).
template <bool EMU>
void p2p_launch(NvlsKernelArgs& a, int ctas, const float* M, cudaStream_t s) {
  const int world = a.world;
  const bool v4 = a.D % 4 == 0 && (uintptr_t)a.table % 16 == 0;
  static const bool no_bulk = getenv("LMSCALE_NO_P2P_BULK") != nullptr;
  const bool bulk = v4 && !no_bulk && (uintptr_t)M % 16 == 0;
  if (!bulk) {
    if (v4)
      k_p2p_update<float4, EMU><<<ctas, NV_THREADS, 0, s>>>(a);
    else
      k_p2p_update<float, EMU><<<ctas, NV_THREADS, 0, s>>>(a);
    return;
  }
  // ring: (G + 1) x 2 KB per slot; the rest of the CTA's share of shared
  // memory after the presence table
  const size_t sb = (size_t)(world + 1) * PB_CB * 4;
  static const int cps_env =
      getenv("LMSCALE_P2P_CTAS_PER_SM") ? atoi(getenv("LMSCALE_P2P_CTAS_PER_SM")) : 0;
  const int cps = cps_env >= 1 && cps_env <= PB_MAX_CPS ? cps_env : 4;  // measured best (tools/ab_p2p.sh)
  // presence-table batch: this rank's most rows per CTA (U_g <= mcap), so
  // one batch normally covers them, and the table leaves room for slots
  static const int rows_env =
      getenv("LMSCALE_P2P_BATCH_ROWS") ? atoi(getenv("LMSCALE_P2P_BATCH_ROWS")) : 0;
  int64_t br = rows_env > 0 ? rows_env
                            : (a.mcap / world + (int64_t)cps * ctas - 1) / ((int64_t)cps * ctas);
  br = (br + 31) / 32 * 32;
  br = br < 32 ? 32 : br > PB_MAXROWS ? PB_MAXROWS : br;
  a.pb_rows = (int)br;
  const size_t lrow_bytes = 4 * (size_t)br * world;
  int slots = (int)(((size_t)200 * 1024 / cps - lrow_bytes) / sb);
  slots = slots < 2 ? 2 : slots > PB_MAXSLOTS ? PB_MAXSLOTS : slots;
  a.pb_slots = slots;
  const size_t smem = (size_t)slots * sb + lrow_bytes;
  static size_t set = 0;
  if (smem > set) {
    cudaFuncSetAttribute(k_p2p_bulk<EMU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    set = smem;
  }
  // several CTAs per SM (one CTA's bulk-copy stream saturates below the
  // SM's share: tools/gather_probe.cu)
  // every CTA resident (the LSA barriers pair CTA k of every rank)
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_p2p_bulk<EMU>, PB_THREADS, smem) !=
          cudaSuccess || occ < 1)
    occ = 1;
  k_p2p_bulk<EMU><<<std::min(cps, occ) * ctas, PB_THREADS, smem, s>>>(a);
}

cudaError_t launch_p2p_emulated(char* const* m_bases, float* const* tables, int world, int rank,
                                const uint32_t* ihat, const Sc3* sc3, const float* M, int D,
                                float lr, size_t lbits_off, size_t lrank_off, size_t mhat_off,
                                float cF, int cbf, int phase, int64_t mcap, uint32_t vocab,
                                int num_sms, cudaStream_t s) {
  NvlsKernelArgs a{};
  a.mcap = mcap;
  a.vocab = vocab;
  a.cbf = cbf;
  a.lrank_off = lrank_off;
  a.local_m = 1;
  a.lbits_off = lbits_off;
  a.cF = cF;
  a.mhat_off = mhat_off;
  a.ihat = ihat;
  a.sc3 = sc3;
  a.table = tables[rank];
  a.M = M;
  a.D = D;
  a.lr = lr;
  a.rank = rank;
  a.world = world;
  for (int j = 0; j < world && j < 8; ++j) {
    a.emu_m[j] = m_bases[j];
    a.emu_t[j] = tables[j];
  }
  const bool v4 = D % 4 == 0 && (uintptr_t)a.table % 16 == 0;
  if (cF > 0.f) {
    if (phase == 1) {
      if (v4)
        k_p2p_update_c<float4, 1><<<num_sms, NV_THREADS, 0, s>>>(a);
      else
        k_p2p_update_c<float, 1><<<num_sms, NV_THREADS, 0, s>>>(a);
    } else {
      if (v4)
        k_p2p_update_c<float4, 2><<<num_sms, NV_THREADS, 0, s>>>(a);
      else
        k_p2p_update_c<float, 2><<<num_sms, NV_THREADS, 0, s>>>(a);
    }
  } else {
    p2p_launch<true>(a, num_sms, M, s);
  }
  return cudaGetLastError();
}

void launch_nvls_update(NvlsState* st, const uint32_t* ihat, const Sc3* sc3, float* table,
                        const float* M, int D, float lr, int rank, int world,
                        unsigned long long* trace, ncclWindow_t twin, size_t lbits_off,
                        float cF, int cbf, size_t mhat_off, size_t lrank_off, int local_m,
                        int64_t mcap, uint32_t vocab, cudaStream_t s) {
  NvlsKernelArgs a;
  a.mcap = mcap;
  a.vocab = vocab;
  a.cbf = cbf;
  a.lrank_off = lrank_off;
  a.local_m = local_m;
  a.lbits_off = lbits_off;
  a.cF = cF;
  a.mhat_off = mhat_off;
  a.twin = twin;
  a.trace = trace;
  static const int diag = getenv("LMSCALE_NVLS_DIAG") ? atoi(getenv("LMSCALE_NVLS_DIAG")) : 0;
  a.diag = diag;
  a.dev = st->dev;
  a.win = st->win;
  a.ihat = ihat;
  a.sc3 = sc3;
  a.table = table;
  a.M = M;
  a.D = D;
  a.lr = lr;
  a.rank = rank;
  a.world = world;
  const bool v4 = D % 4 == 0 && (uintptr_t)table % 16 == 0;
  static bool once = (max_carveout((const void*)k_nvls_update<float4>),
                      max_carveout((const void*)k_nvls_update<float>),
                      max_carveout((const void*)k_p2p_update<float4, false>),
                      max_carveout((const void*)k_p2p_update<float, false>),
                      max_carveout((const void*)k_p2p_update_c<float4, 0>),
                      max_carveout((const void*)k_p2p_update_c<float, 0>), true);
  (void)once;
  if (cF > 0.f) {  // compressed exchange (any table; G <= 8)
    if (v4)
      k_p2p_update_c<float4, 0><<<st->ctas, NV_THREADS, 0, s>>>(a);
    else
      k_p2p_update_c<float, 0><<<st->ctas, NV_THREADS, 0, s>>>(a);
  } else if (twin && nvls_use_p2p(world)) {
    p2p_launch<false>(a, st->ctas, M, s);
  } else if (v4) {
    k_nvls_update<float4><<<st->ctas, NV_THREADS, 0, s>>>(a);
  } else {
    k_nvls_update<float><<<st->ctas, NV_THREADS, 0, s>>>(a);
  }
}

}  // namespace lms
