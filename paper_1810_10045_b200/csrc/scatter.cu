// scatter.cu -- S4 segmented scatter-add (steps 2+5),
// S6 duplicate-free row update (step 7) and the S0 dense
// comparison scatter for sm_100a.
//
// S4 layout: the K gradient rows are visited in sorted-id order through the
// stable permutation from S1.  Work items are (chunk of 32 sorted positions,
// column block) pairs, one warp each, in a persistent grid: every warp reads
// its 32 rows with 128-bit streaming loads (4-row software pipeline), sums the
// runs of equal ids in registers and writes each finished run ONCE to its
// global slot of M.  Runs cut by a chunk boundary write a partial row instead
// (head / tail partial of the chunk); a second launch sums each cut run's
// partials in a fixed order (deterministic, no atomics) and writes its M row.
// Slots whose word is absent on this rank are written as zeros by extra work
// items, so every one of the U_g rows is stored exactly once (no memset).
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

constexpr int SC_THREADS = 256;
constexpr unsigned FULL_MASK = 0xffffffffu;

// Store element block `col` of M row `slot`: fp32, or compressed binary16
// (the payload of the compressed exchange) when a.m16.
__device__ __forceinline__ void st_m(const ScatterArgs& a, size_t slot, int C, int col, float4 v) {
  if (a.m16) {
    reinterpret_cast<uint2*>(a.M)[slot * C + col] = enc4(v, a.cF, a.cbf);
  } else {
    st_v4(reinterpret_cast<float4*>(a.M) + slot * C + col, v);
  }
}
__device__ __forceinline__ void st_m(const ScatterArgs& a, size_t slot, int C, int col, float v) {
  if (a.m16)
    reinterpret_cast<uint16_t*>(a.M)[slot * C + col] = enc1(v, a.cF, a.cbf);
  else
    a.M[slot * C + col] = v;
}


// World 1 with S6 folded in (a.apply): a finished row m of word w goes straight
// into the table, E[w] = fma(-lr, m, E[w]) -- the same instruction k_update
// runs, so the bits equal the separate-launch path; M is never written.
template <typename T>
__device__ __forceinline__ void apply_e(const ScatterArgs& a, uint32_t w, int C, int col, T m);
template <>
__device__ __forceinline__ void apply_e<float4>(const ScatterArgs& a, uint32_t w, int C, int col,
                                                float4 m) {
  float4* e = reinterpret_cast<float4*>(a.table) + (size_t)w * C + col;
  const float4 x = *e;
  st_v4(e, make_float4(__fmaf_rn(-a.lr, m.x, x.x), __fmaf_rn(-a.lr, m.y, x.y),
                       __fmaf_rn(-a.lr, m.z, x.z), __fmaf_rn(-a.lr, m.w, x.w)));
}
template <>
__device__ __forceinline__ void apply_e<float>(const ScatterArgs& a, uint32_t w, int C, int col,
                                               float m) {
  float* e = a.table + (size_t)w * C + col;
  *e = __fmaf_rn(-a.lr, m, *e);
}

// A finished row of slot `slot` (word w): into M, or into E (a.apply).
template <typename T, int NV, bool FULLC>
__device__ __forceinline__ void emit_row(const ScatterArgs& a, size_t slot, uint32_t w, int C,
                                         int col0, const T (&acc)[NV]) {
  if (a.apply) {
    T* e = reinterpret_cast<T*>(a.table) + (size_t)w * C;
    T x[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (FULLC || col0 + v * 32 < C) x[v] = e[col0 + v * 32];
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (FULLC || col0 + v * 32 < C) Vec<T>::st(e + col0 + v * 32, Vec<T>::fma(-a.lr, acc[v], x[v]));
  } else {
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (FULLC || col0 + v * 32 < C) st_m(a, slot, C, col0 + v * 32, acc[v]);
  }
}
}  // namespace

// ------------------------------------------------------------------- S4

// One chunk of sorted positions [i0, i0 + n) for one column block.  Runs of
// <= FX_SHORT tokens belong entirely to the chunk where they start: a short
// run cut by the chunk's right edge is finished by reading on (at most
// FX_SHORT - 1 positions past the edge) and the next chunk skips its tail.
// Only long runs (the Zipf head) are cut into partial rows (P[2c] head piece,
// P[2c+1] tail piece) and listed for the fix-up phase by the chunk holding
// their start.  FULLC: the column block lies inside the row (no predicates).
// ---- last-arriver fix-up of runs cut by chunk boundaries (no grid barrier)
// A run spanning chunks c0..c1 leaves np = c1 - c0 + 1 partial rows: k = 0 is
// the tail piece of c0 (P[2c0+1]), k >= 1 the head piece of c0+k (P[2(c0+k)]).
// They are summed in parts of FXP partials: the warp that stores the last
// partial of a part (atomic counter per (part, column block)) sums that part
// in k order; with one part it emits the row, else it stores a level-2 row
// and the last part to finish sums the level-2 rows in part order.  Fixed
// summation order: deterministic.  Counters reset themselves for the next
// launch.

// partial rows k in [k0, k0 + n) of the run starting at chunk c0, summed in k order
template <typename T, int NV>
__device__ __forceinline__ void sum_partials(const T* base, int c0, int k0, int n, int col0, int C,
                                             T (&acc)[NV]) {
  using V = Vec<T>;
  constexpr int FU = NV >= 4 ? 2 : 4;  // rows in flight (register budget of the 4-vector path)
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = V::zero();
  for (int i = 0; i < n; i += FU) {
    T r[FU][NV];
#pragma unroll
    for (int q = 0; q < FU; ++q) {
      const int kk = k0 + i + q;
      const size_t row = kk == 0 ? (size_t)(2 * c0 + 1) : (size_t)(2 * (c0 + kk));
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int col = col0 + v * 32;
        r[q][v] = V::zero();
        if (i + q < n && col < C) r[q][v] = V::ld_l2(base + row * C + col);
      }
    }
#pragma unroll
    for (int q = 0; q < FU; ++q)
      if (i + q < n)
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] = V::add(acc[v], r[q][v]);
  }
}

template <typename T, int NV>
__device__ __forceinline__ void fix_arrive(const ScatterArgs& a, int u, int c0, int k, int np, int cb,
                                        int ncb, int col0, int C, int lane) {
  using V = Vec<T>;
  uint32_t* pcnt = a.fxcnt;
  uint32_t* rcnt = a.fxcnt + a.fx_stride;
  const int FXP = a.fxp;  // partials per part
  const int j = k / FXP, nparts = (np + FXP - 1) / FXP;
  // ids of a part / a run = the partial-row index of its first piece (unique:
  // every partial row belongs to exactly one run): counter and level-2 row
  const int pc = j == 0 ? 2 * c0 + 1 : 2 * (c0 + j * FXP);
  const int rc = 2 * c0 + 1;
  const int cnt = min(FXP, np - j * FXP);
  __syncwarp();
  __threadfence();
  uint32_t old = 0;
  if (lane == 0) old = atomicAdd(pcnt + (size_t)pc * ncb + cb, 1u);
  old = __shfl_sync(FULL_MASK, old, 0);
  if ((int)old != cnt - 1) return;
  if (lane == 0) pcnt[(size_t)pc * ncb + cb] = 0u;
  __threadfence();
  T acc[NV];
  sum_partials<T, NV>(reinterpret_cast<const T*>(a.partial), c0, j * FXP, cnt, col0, C, acc);
  if (nparts > 1) {
    T* L2 = reinterpret_cast<T*>(a.part2) + (size_t)pc * C;
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (col0 + v * 32 < C) V::st(L2 + col0 + v * 32, acc[v]);
    __syncwarp();
    __threadfence();
    if (lane == 0) old = atomicAdd(rcnt + (size_t)rc * ncb + cb, 1u);
    old = __shfl_sync(FULL_MASK, old, 0);
    if ((int)old != nparts - 1) return;
    if (lane == 0) rcnt[(size_t)rc * ncb + cb] = 0u;
    __threadfence();
    const T* L2b = reinterpret_cast<const T*>(a.part2);
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = V::zero();
    for (int jj = 0; jj < nparts; jj += 2) {
      T r2[2][NV];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int jq = jj + q;
        const size_t row = jq == 0 ? (size_t)(2 * c0 + 1) : (size_t)(2 * (c0 + jq * FXP));
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          r2[q][v] = V::zero();
          if (jq < nparts && col0 + v * 32 < C) r2[q][v] = V::ld_l2(L2b + row * C + col0 + v * 32);
        }
      }
#pragma unroll
      for (int q = 0; q < 2; ++q)
        if (jj + q < nparts)
#pragma unroll
          for (int v = 0; v < NV; ++v) acc[v] = V::add(acc[v], r2[q][v]);
    }
  }
  const int slot = a.zero_rows ? __ldcg(a.l2g + u) : u;
  if (slot < 0) return;
  const uint32_t w = a.apply ? __ldg(a.ihat + slot) : 0u;
  emit_row<T, NV, false>(a, (size_t)slot, w, C, col0, acc);
}

template <typename T, int NV, int UNR, bool FULLC, bool PRE, bool FXL>
__device__ __forceinline__ void scatter_chunk(const ScatterArgs& a, const T* __restrict__ g,
                                              T* __restrict__ M, T* __restrict__ P, int c,
                                              int n, int col0, int C, int lane) {
  using V = Vec<T>;
  const int K = a.K;
  const int i0 = c * SC_CHUNK;
  int my_pos = 0, my_u = -1;
  if (lane < n) {
    my_pos = __ldg(a.perm + i0 + lane);
    my_u = __ldg(a.segidx + i0 + lane);
  }
  const int prev_u = i0 > 0 ? __ldg(a.segidx + i0 - 1) : -1;
  const int next_u = i0 + n < K ? __ldg(a.segidx + i0 + n) : -1;
  const int up = __shfl_up_sync(FULL_MASK, my_u, 1);
  const unsigned hmask = __ballot_sync(FULL_MASK, lane < n && (lane == 0 || my_u != up));
  const int u_first = __shfl_sync(FULL_MASK, my_u, 0);
  const int u_last = __shfl_sync(FULL_MASK, my_u, n - 1);
  const bool split_left = u_first == prev_u;
  const bool split_right = u_last == next_u;
  // run extents of the cut runs: lanes 0..3 load lstart[u_first], lstart[u_first+1],
  // lstart[u_last], lstart[u_last+1]
  int ls = 0;
  if ((lane < 2 && split_left) || (lane >= 2 && lane < 4 && split_right))
    ls = __ldg(a.lstart + (lane < 2 ? u_first + lane : u_last + lane - 2));
  // world 1: I^ = J^, so the slot is the run index itself (no dependent load)
  int my_slot = -1;
  if (lane < n) my_slot = a.zero_rows ? __ldg(a.l2g + my_u) : my_u;
  uint32_t my_w = 0;  // the run's word (world-1 S6 folded in)
  if (a.apply && lane < n) my_w = __ldg(a.ihat + my_slot);
  const int f_start = __shfl_sync(FULL_MASK, ls, 0), f_end = __shfl_sync(FULL_MASK, ls, 1);
  const int l_start = __shfl_sync(FULL_MASK, ls, 2), l_end = __shfl_sync(FULL_MASK, ls, 3);
  // without short-run handling (small K, where the fix-up is cheap) every cut
  // run is treated as long: no run-extent lookup before the row loop
  const bool first_long = split_left && (!a.short_runs || f_end - f_start > FX_SHORT);
  const bool last_long = split_right && (!a.short_runs || l_end - l_start > FX_SHORT);
  // [p_begin, p_end): positions this chunk sums (p_end may pass n for a short
  // run started here and cut by the right edge)
  const int p_begin = (split_left && !first_long) ? min(n, f_end - i0) : 0;
  if (p_begin >= n) return;  // the whole chunk is the tail of a short run owned earlier
  const bool extend = split_right && !last_long;
  const int p_end = extend ? l_end - i0 : n;
  int ext_pos = 0;
  if (extend && SC_CHUNK + lane < p_end) ext_pos = __ldg(a.perm + i0 + SC_CHUNK + lane);
  T acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = V::zero();
  bool seg_first = (p_begin == 0);  // the run being accumulated is the chunk's first
  bool pend_head = false, pend_tail = false;  // partial rows stored (fix-ups after the loop)
  for (int p0 = p_begin; p0 < p_end; p0 += UNR) {
    T r[UNR][NV];
#pragma unroll
    for (int q = 0; q < UNR; ++q) {
      const int p = p0 + q;
      const int pos = p < SC_CHUNK ? __shfl_sync(FULL_MASK, my_pos, p & 31)
                                   : __shfl_sync(FULL_MASK, ext_pos, p & 31);
      const T* row = g + (size_t)pos * C;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int col = col0 + v * 32;
        r[q][v] = V::zero();
        if (p < p_end && (FULLC || col < C)) r[q][v] = V::ld_once(row + col);
      }
    }
    // PRE (world-1 folded S6, small K): the E rows of the runs ending in this
    // group are loaded together with the gradient rows, so the row update at
    // a run's end does not wait for a dependent load (p_end <= n here)
    T x[PRE ? UNR : 1][NV];
    if constexpr (PRE) {
      const T* E = reinterpret_cast<const T*>(a.table);
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const int p = p0 + q;
        const bool endp = p < p_end && (p == p_end - 1 || (p + 1 < n && ((hmask >> (p + 1)) & 1u)));
        const uint32_t wq = __shfl_sync(FULL_MASK, my_w, min(p, n - 1));
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int col = col0 + v * 32;
          x[q][v] = V::zero();
          if (endp && (FULLC || col < C)) x[q][v] = E[(size_t)wq * C + col];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < UNR; ++q) {
      const int p = p0 + q;
      if (p < p_end) {
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] = V::add(acc[v], r[q][v]);
        const bool last = (p == p_end - 1);
        if (last || (p + 1 < n && ((hmask >> (p + 1)) & 1u))) {
          const int slot = __shfl_sync(FULL_MASK, my_slot, min(p, n - 1));
          T* dst;
          if (seg_first && split_left) {  // long run continuing from the left
            dst = P + (size_t)(2 * c) * C;
            pend_head = true;
          } else if (last && split_right && last_long) {
            dst = P + (size_t)(2 * c + 1) * C;
            pend_tail = true;
            // this chunk holds the start of a long run cut by its end: it owns
            // the run's fix-up, listed (by column block 0) as ceil(np / FX_PART)
            // contiguous parts so that the Zipf head is summed by many CTAs
            if (!FXL && col0 == lane) {
              int ent = 0, nparts = 0;
              if (lane == 0) {
                const int np = (l_end - 1) / SC_CHUNK - c + 1;
                nparts = (np + FX_PART - 1) / FX_PART;
                ent = (int)atomicAdd(&a.sc1w->fixcount, (uint32_t)nparts);
                if (nparts > 1) atomicOr(&a.sc1w->err, 2u);  // phase 2b needed
              }
              ent = __shfl_sync(FULL_MASK, ent, 0);
              nparts = __shfl_sync(FULL_MASK, nparts, 0);
              for (int j = lane; j < nparts; j += 32)
                if (ent + j < a.fix_cap) a.fixent[ent + j] = make_int2(c, j | (nparts << 16));
            }
          } else {
            dst = nullptr;
            const uint32_t wv = __shfl_sync(FULL_MASK, my_w, min(p, n - 1));
            if constexpr (PRE) {
              T* e = reinterpret_cast<T*>(a.table) + (size_t)wv * C;
#pragma unroll
              for (int v = 0; v < NV; ++v)
                if (FULLC || col0 + v * 32 < C)
                  V::st(e + col0 + v * 32, V::fma(-a.lr, acc[v], x[q][v]));
            } else if (slot >= 0) {
              emit_row<T, NV, FULLC>(a, (size_t)slot, wv, C, col0, acc);
            }
          }
          if (dst) {
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              const int col = col0 + v * 32;
              if (FULLC || col < C) V::st(dst + col, acc[v]);
            }
          }
#pragma unroll
          for (int v = 0; v < NV; ++v) acc[v] = V::zero();
          seg_first = false;
        }
      }
    }
  }
  // last-arriver fix-ups of the cut runs this chunk stored pieces of (after
  // the row loop: no registers of the loop are live across the call)
  if (FXL && (pend_head || pend_tail)) {
    const int cb = (col0 - lane) / (32 * NV), ncb = (C + 32 * NV - 1) / (32 * NV);
    if (pend_head) {
      const int c0 = f_start / SC_CHUNK;
      fix_arrive<T, NV>(a, __shfl_sync(FULL_MASK, my_u, 0), c0, c - c0,
                        (f_end - 1) / SC_CHUNK - c0 + 1, cb, ncb, col0, C, lane);
    }
    if (pend_tail)
      fix_arrive<T, NV>(a, __shfl_sync(FULL_MASK, my_u, n - 1), c, 0,
                        (l_end - 1) / SC_CHUNK - c + 1, cb, ncb, col0, C, lane);
  }
}

// Phase 2a (fix-up part) for one listed entry (owner chunk c, part j of
// nparts) and column block: sum partials k in [64j, min(np, 64j + 64)) of the
// run -- k = 0 is P[2c+1] (tail of c), k >= 1 is P[2(c+k)] (head of c+k) --
// in a fixed order (warp w sums k = w, w+8, ...; warps combined in warp order
// through shared memory).  One part: the sum is the run's row of M.  More
// parts: it goes to level-2 row `e` and phase 2b adds the parts in order.
template <typename T, int NV>
__device__ __forceinline__ void fixup_part(const ScatterArgs& a, T (*red)[32 * NV], int e,
                                           int cb, int C) {
  using V = Vec<T>;
  constexpr int NWF = SC_THREADS / 32;
  constexpr int UNR = 4;
  const int lane = (int)lane_id(), warp = threadIdx.x >> 5;
  const T* P = reinterpret_cast<const T*>(a.partial);
  const int2 en = __ldcg(a.fixent + e);
  const int c = en.x, j = en.y & 0xffff, nparts = en.y >> 16;
  const int iend = min(a.K, (c + 1) * SC_CHUNK);
  const int u = __ldcg(a.segidx + iend - 1);
  const int np = (__ldcg(a.lstart + u + 1) - 1) / SC_CHUNK - c + 1;
  const int k_lo = j * FX_PART, k_hi = min(np, k_lo + FX_PART);
  const int col0 = cb * 32 * NV + lane;
  T acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = V::zero();
  for (int k0 = k_lo + warp; k0 < k_hi; k0 += NWF * UNR) {
    T r[UNR][NV];
#pragma unroll
    for (int q = 0; q < UNR; ++q) {
      const int k = k0 + q * NWF;
      const size_t prow = k == 0 ? (size_t)(2 * c + 1) : (size_t)(2 * (c + k));
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int col = col0 + v * 32;
        r[q][v] = V::zero();
        if (k < k_hi && col < C) r[q][v] = V::ld_l2(P + prow * C + col);
      }
    }
#pragma unroll
    for (int q = 0; q < UNR; ++q)
#pragma unroll
      for (int v = 0; v < NV; ++v) acc[v] = V::add(acc[v], r[q][v]);
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) red[warp][v * 32 + lane] = acc[v];
  __syncthreads();
  if (warp == 0) {
    const int slot = nparts == 1 ? (a.zero_rows ? __ldcg(a.l2g + u) : u) : -1;
    const uint32_t word = (a.apply && slot >= 0) ? __ldg(a.ihat + slot) : 0u;
    T* dst = nparts == 1 ? nullptr : reinterpret_cast<T*>(a.part2) + (size_t)e * C;
    if (dst || slot >= 0) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        T sum = red[0][v * 32 + lane];
#pragma unroll
        for (int w = 1; w < NWF; ++w) sum = V::add(sum, red[w][v * 32 + lane]);
        const int col = col0 + v * 32;
        if (col < C) {
          if (dst)
            V::st(dst + col, sum);
          else if (a.apply)
            apply_e<T>(a, word, C, col, sum);
          else
            st_m(a, (size_t)slot, C, col, sum);
        }
      }
    }
  }
  __syncthreads();
}

// Phase 2b: a run listed as nparts > 1 parts (entries e0 .. e0+nparts-1,
// contiguous): add its level-2 rows in entry order, store the run's M row.
template <typename T, int NV>
__device__ __forceinline__ void fixup_final(const ScatterArgs& a, int e0, int cb, int C) {
  using V = Vec<T>;
  const int lane = (int)lane_id();
  const int2 en = __ldcg(a.fixent + e0);
  const int c = en.x, nparts = en.y >> 16;
  const int iend = min(a.K, (c + 1) * SC_CHUNK);
  const int u = __ldcg(a.segidx + iend - 1);
  const int slot = a.zero_rows ? __ldcg(a.l2g + u) : u;
  if (slot < 0) return;
  const T* L2 = reinterpret_cast<const T*>(a.part2);
  const int col0 = cb * 32 * NV + lane;
  const uint32_t w = a.apply ? __ldg(a.ihat + slot) : 0u;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int col = col0 + v * 32;
    if (col >= C) continue;
    T sum = V::ld_l2(L2 + (size_t)e0 * C + col);
    for (int j = 1; j < nparts; ++j) sum = V::add(sum, V::ld_l2(L2 + (size_t)(e0 + j) * C + col));
    if (a.apply)
      apply_e<T>(a, w, C, col, sum);
    else
      st_m(a, (size_t)slot, C, col, sum);
  }
}

__device__ __forceinline__ void sstamp(unsigned long long* tr, int i) {
  if (tr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x == 0) tr[i] = t;
    atomicMax(tr + i + 4, t);  // latest CTA
  }
}

template <typename T, int NV, int UNR, bool PRE, bool FXL>
__global__ void __launch_bounds__(SC_THREADS, (PRE || FXL) ? 1 : 2) k_scatter(ScatterArgs a) {
  using V = Vec<T>;
  sstamp(a.trace, 54);
  if (a.trace && threadIdx.x == 0) {  // earliest start over all CTAs (as ~t)
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(a.trace + 63, ~t);
  }
  __shared__ T red[SC_THREADS / 32][32 * NV];
  // launched as a programmatic dependent of S1: wait for S1's grid to
  // complete (and its memory to be visible) before reading its outputs
  if (a.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  // an id >= vocab: no table row is touched (the error surfaces at the next
  // host sync); every CTA reads the same flag, so all leave together
  if (a.apply && (__ldcg(&a.sc3->err) & 1u)) return;
  const int K = a.K;
  const int C = a.D / V::W;  // vectors per row
  const int ncb = (C + 32 * NV - 1) / (32 * NV);
  const int nchunks = (K + SC_CHUNK - 1) / SC_CHUNK;
  const int64_t Ug = a.sc3->u_global;
  const int64_t nz = a.zero_rows && a.fill_absent ? (Ug + SC_ZGROUP - 1) / SC_ZGROUP : 0;
  const int64_t items = ((int64_t)nchunks + nz) * ncb;
  const int lane = (int)lane_id();
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T* g = reinterpret_cast<const T*>(a.grad);
  T* M = reinterpret_cast<T*>(a.M);
  T* P = reinterpret_cast<T*>(a.partial);

  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items;
       it += nwarps) {
    const int cb = (int)(it % ncb);
    const int64_t unit = it / ncb;
    const int col0 = cb * 32 * NV + lane;
    if (unit < nchunks) {
      const int c = (int)unit;
      const int n = min(SC_CHUNK, K - c * SC_CHUNK);
      if ((cb + 1) * 32 * NV <= C)
        scatter_chunk<T, NV, UNR, true, PRE, FXL>(a, g, M, P, c, n, col0, C, lane);
      else
        scatter_chunk<T, NV, UNR, false, PRE, FXL>(a, g, M, P, c, n, col0, C, lane);
    } else {
      // ---- zero rows: slots [r0, r0 + 32) whose word is absent on this rank
      const int64_t r0 = (unit - nchunks) * SC_ZGROUP;
      const int64_t r = r0 + lane;
      bool absent = false;
      if (r < Ug) {
        const uint32_t w = __ldg(a.ihat + r);
        absent = !((__ldg(a.lbits + (w >> 5)) >> (w & 31u)) & 1u);
      }
      unsigned am = __ballot_sync(FULL, absent);
      while (am) {
        const int b = __ffs(am) - 1;
        am &= am - 1;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int col = col0 + v * 32;
          if (col < C) st_m(a, (size_t)(r0 + b), C, col, V::zero());
        }
      }
    }
  }
  sstamp(a.trace, 55);
  if constexpr (FXL) return;  // cut runs were finished by their last arriving piece
  if constexpr (!FXL) {
  grid_barrier(a.bar);
  sstamp(a.trace, 56);

  // phase 2a: parts of the runs cut by chunk boundaries (balanced: <= FX_PART
  // partials per CTA item)
  const int nfix = (int)min(__ldcg(&a.sc1w->fixcount), (uint32_t)a.fix_cap);
  for (int64_t it = blockIdx.x; it < (int64_t)nfix * ncb; it += gridDim.x)
    fixup_part<T, NV>(a, red, (int)(it / ncb), (int)(it % ncb), C);
  sstamp(a.trace, 57);
  if (!(__ldcg(&a.sc1w->err) & 2u)) return;  // no run was split into parts
  grid_barrier(a.bar);
  // phase 2b: runs split into several parts, one warp per (run, column block)
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t it = gwarp; it < (int64_t)nfix * ncb; it += nwarps) {
    const int e = (int)(it / ncb);
    const int2 en = __ldcg(a.fixent + e);
    if ((en.y & 0xffff) == 0 && (en.y >> 16) > 1) fixup_final<T, NV>(a, e, (int)(it % ncb), C);
  }

  }
  if (!a.table || a.apply) return;
  grid_barrier(a.bar);

  // phase 3 (world 1): S6 row update, warp per row
  T* E = reinterpret_cast<T*>(a.table);
  const float lr = a.lr;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < Ug; r += nwarps) {
    const uint32_t w = __ldg(a.ihat + r);
    const T* src = M + (size_t)r * C;
    T* dst = E + (size_t)w * C;
    int col = lane;
    for (; col + 96 < C; col += 128) {
      const T m0 = V::ld_l2(src + col), m1 = V::ld_l2(src + col + 32);
      const T m2 = V::ld_l2(src + col + 64), m3 = V::ld_l2(src + col + 96);
      const T e0 = dst[col], e1 = dst[col + 32], e2 = dst[col + 64], e3 = dst[col + 96];
      V::st(dst + col, V::fma(-lr, m0, e0));
      V::st(dst + col + 32, V::fma(-lr, m1, e1));
      V::st(dst + col + 64, V::fma(-lr, m2, e2));
      V::st(dst + col + 96, V::fma(-lr, m3, e3));
    }
    for (; col < C; col += 32) V::st(dst + col, V::fma(-lr, V::ld_l2(src + col), dst[col]));
  }
}

namespace {
template <typename T>
bool vec_ok(const ScatterArgs& a) {
  if (sizeof(T) == 4) return true;
  return (a.D % 4 == 0) && ((uintptr_t)a.grad % 16 == 0) && ((uintptr_t)a.M % 16 == 0) &&
         ((uintptr_t)a.partial % 16 == 0);
}
}  // namespace

template <typename T, int NV, int UNR, bool PRE = false, bool FXL = false>
static cudaError_t scatter_t(const ScatterArgs& a, cudaStream_t s) {
  static int occ = 0;  // resident CTAs per SM for this instantiation (persistent grid)
  if (!occ) {
    max_carveout((const void*)k_scatter<T, NV, UNR, PRE, FXL>);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_scatter<T, NV, UNR, PRE, FXL>, SC_THREADS,
                                                      0) != cudaSuccess || occ < 1)
      occ = 1;
  }
  const int C = a.D / Vec<T>::W;
  const int ncb = (C + 32 * NV - 1) / (32 * NV);
  const int64_t nchunks = (a.K + SC_CHUNK - 1) / SC_CHUNK;
  const int64_t nz = a.zero_rows && a.fill_absent ? (a.ug_cap + SC_ZGROUP - 1) / SC_ZGROUP : 0;
  int64_t blocks = ((nchunks + nz) * ncb * 32 + SC_THREADS - 1) / SC_THREADS;
  const int64_t cap = (int64_t)a.num_sms * occ;
  if (blocks > cap) blocks = cap;
  if (blocks < a.num_sms) blocks = a.num_sms < cap ? a.num_sms : cap;  // phases 2/3 want a wide grid
  // grid <= occupancy x SMs: every CTA is co-resident, so the in-kernel
  // grid barrier is safe with a normal launch
  if (a.pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(SC_THREADS);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_scatter<T, NV, UNR, PRE, FXL>, a);
  }
  k_scatter<T, NV, UNR, PRE, FXL><<<(unsigned)blocks, SC_THREADS, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_scatter(const ScatterArgs& a, cudaStream_t s) {
  if (vec_ok<float4>(a)) {
    const int C = a.D / 4;
    // experiment knob: column-block width x row loads in flight per warp
    static const int var = getenv("LMSCALE_S4_VARIANT") ? atoi(getenv("LMSCALE_S4_VARIANT")) : 0;
    // folded S6 at small K (no short-run extension): E rows preloaded per group
    static const bool no_pre = getenv("LMSCALE_NO_PRE") != nullptr;
    if (a.apply && !a.short_runs && !no_pre) {
      if (a.fx_last) {
        if (C >= 128) return scatter_t<float4, 4, 4, true, true>(a, s);
        if (C >= 64) return scatter_t<float4, 2, 4, true, true>(a, s);
        return scatter_t<float4, 1, 4, true, true>(a, s);
      }
      if (C >= 128) return scatter_t<float4, 4, 4, true>(a, s);
      if (C >= 64) return scatter_t<float4, 2, 4, true>(a, s);
      return scatter_t<float4, 1, 4, true>(a, s);
    }
    if (a.fx_last && !a.short_runs) {  // small K: last-arriver fix-up
      if (C >= 128) return scatter_t<float4, 4, 4, false, true>(a, s);
      if (C >= 64) return scatter_t<float4, 2, 4, false, true>(a, s);
      return scatter_t<float4, 1, 4, false, true>(a, s);
    }
    if (var == 1) return scatter_t<float4, 2, 8>(a, s);
    if (var == 2) return scatter_t<float4, 1, 16>(a, s);
    if (var == 3) return scatter_t<float4, 1, 8>(a, s);
    if (C >= 128) return scatter_t<float4, 4, 4>(a, s);
    if (C >= 64) return scatter_t<float4, 2, 4>(a, s);
    return scatter_t<float4, 1, 4>(a, s);
  }
  return scatter_t<float, 4, 4>(a, s);
}

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
