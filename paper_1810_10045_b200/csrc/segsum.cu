// segsum.cu -- S4, the segmented scatter-add of steps 2 + 5 (P:405-406,
// P:415-418), and at world 1 the row update of step 7 folded into it.
//
// The K gradient rows are walked in the grouped order of S1 (perm): runs of
// equal ids are contiguous.  The grouped positions are cut into nR
// contiguous, equal-length ranges, one CTA each (x a column block when a row
// is wider than 8 KB), so every CTA reads the same number of gradient rows.
//
// Inside a CTA (warp-specialised, mbarrier rings in shared memory):
//   * producer warp: for each group of GR positions, one elected lane arms
//     the slot's `full` mbarrier with the byte count and lanes issue one 1-D
//     bulk copy (cp.async.bulk, the TMA engine) per gradient row into the
//     slot; at world 1 also one per E row of every run that ends whole inside
//     the group, behind the group's rows.
//     Bytes in flight cost no registers.  2-4 CTAs per SM: one CTA's copy
//     stream was measured to saturate at 20-40 GB/s (tools/gather_probe.cu).
//   * consumer warps: thread t owns one float4 column of the row; it waits
//     on the slot's `full` barrier, adds the group's rows into its running
//     sum, and at the end of each run emits the run's row -- world 1: E[w] =
//     fma(-lr, m, E[w]) from the staged E row, one store, no atomics
//     (P:433-435); otherwise M_g[slot] (fp32, or binary16 under compression,
//     R15) -- then releases the slot through its `empty` barrier.
//   * a run cut by a range edge (the Zipf head spans many ranges) leaves one
//     partial row per range; the CTAs that store the last partial of each
//     group of 8 consecutive partials, then of the run's group sums (counters,
//     self-resetting), sum them in range order and emit the row.  No grid
//     barrier, no atomics on data.
//
// Non-16-byte-aligned rows (dim % 4 != 0) take the same kernel without the
// producer: consumers load their scalar columns directly.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace lms {

namespace {

constexpr uint32_t F_END = 1u << 31;   // the last position of a segment in this range
constexpr uint32_t F_FULL = 1u << 30;  // ... and the segment is a whole run (emit here)
constexpr uint32_t F_ROW = (1u << 30) - 1u;

template <typename T>
struct VT;
template <>
struct VT<float4> {
  static constexpr int W = 4;
  __device__ __forceinline__ static float4 zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ __forceinline__ static float4 add(float4 a, float4 b) { return f4add(a, b); }
  __device__ __forceinline__ static float4 fma(float s, float4 a, float4 b) {
    return make_float4(__fmaf_rn(s, a.x, b.x), __fmaf_rn(s, a.y, b.y), __fmaf_rn(s, a.z, b.z),
                       __fmaf_rn(s, a.w, b.w));
  }
  __device__ __forceinline__ static float4 ld_once(const float4* p) { return ld_stream(p); }
  __device__ __forceinline__ static void st_m(float* M, size_t off, float4 v, int m16, float F,
                                              int bf) {
    if (m16)
      *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(M) + off) = enc4(v, F, bf);
    else
      *reinterpret_cast<float4*>(M + off) = v;
  }
};
template <>
struct VT<float> {
  static constexpr int W = 1;
  __device__ __forceinline__ static float zero() { return 0.f; }
  __device__ __forceinline__ static float add(float a, float b) { return a + b; }
  __device__ __forceinline__ static float fma(float s, float a, float b) {
    return __fmaf_rn(s, a, b);
  }
  __device__ __forceinline__ static float ld_once(const float* p) { return __ldcs(p); }
  __device__ __forceinline__ static void st_m(float* M, size_t off, float v, int m16, float F,
                                              int bf) {
    if (m16)
      reinterpret_cast<uint16_t*>(M)[off] = enc1(v, F, bf);
    else
      M[off] = v;
  }
};

// range of grouped position q (ranges of seg_len positions)
__device__ __forceinline__ int range_of(int q, uint32_t seg_len) { return (int)((uint32_t)q / seg_len); }

struct Meta {
  int u_first, u_last;
  int cut_l, cut_r;
  int ls_first, le_first, ls_last, le_last;  // lstart[u], lstart[u + 1]
  int last;                                  // broadcast: this CTA is the last arriver
};

}  // namespace

// Sum rows row_of(0..n-1) of `base` (column `col`) in index order, up to 8
// loads in flight.
template <typename T, typename RowOf>
__device__ __forceinline__ T sum_rows(const float* base, int n, size_t D, size_t col, RowOf row_of) {
  using V = VT<T>;
  T s = V::zero();
  for (int k = 0; k < n; k += 8) {
    T r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      r[q] = k + q < n ? __ldcg(reinterpret_cast<const T*>(base + row_of(k + q) * D + col))
                       : V::zero();
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (k + q < n) s = V::add(s, r[q]);
  }
  return s;
}

// One segment end that is a piece of a run cut by range edges.  Piece k of a
// run that starts in range b0 and spans np ranges: k = 0 is the tail of b0
// (partial row 2 b0 + 1), k >= 1 the head of b0 + k (row 2 (b0 + k)).  Pieces
// are summed in groups of SEG_FXP consecutive pieces by the CTA that stores
// the group's last piece (counter per group); with several groups, each group
// sum goes to a level-2 row and the last group to finish sums those in group
// order.  Fixed summation order, no grid barrier, counters reset themselves.
template <typename T>
__device__ __forceinline__ void cut_piece(const SegArgs& a, Meta& m, bool head, T acc, int b,
                                          int cb, int ncb, int nct, int t, int cw) {
  using V = VT<T>;
  constexpr int VW = V::W;
  const size_t D = (size_t)a.D;
  const size_t col = (size_t)cb * a.cbw + (size_t)t * VW;  // first float of this thread
  const bool act = t < cw;
  const int u = head ? m.u_first : m.u_last;
  const int ls = head ? m.ls_first : m.ls_last, le = head ? m.le_first : m.le_last;
  const int b0 = range_of(ls, a.seg_len), b1 = range_of(le - 1, a.seg_len);
  const int np = b1 - b0 + 1;
  const int k = b - b0;  // this piece
  const size_t prow = k == 0 ? (size_t)(2 * b0 + 1) : (size_t)(2 * b);
  LMS_CHECK(k >= 0 && np >= 1 && prow < (size_t)a.part_rows && b1 < (int)gridDim.x);
  if (act) __stcg(reinterpret_cast<T*>(a.part + prow * D + col), acc);
  const int j = k / SEG_FXP, ng = (np + SEG_FXP - 1) / SEG_FXP;
  const int gn = min(SEG_FXP, np - j * SEG_FXP);
  named_bar_sync(1, nct);
  if (t == 0) {
    __threadfence();
    uint32_t* c = a.cnt + ((size_t)(2 * b0 + j) * ncb + cb);
    const uint32_t old = atomicAdd(c, 1u);
    m.last = (int)old == gn - 1;
    if (m.last) *c = 0u;  // the group is complete: reset for the next launch
  }
  named_bar_sync(1, nct);
  if (!m.last) return;
  __threadfence();
  const int k0 = j * SEG_FXP;
  T s = V::zero();
  if (act)
    s = sum_rows<T>(a.part, gn, D, col, [&](int q) {
      const int kk = k0 + q;
      return kk == 0 ? (size_t)(2 * b0 + 1) : (size_t)(2 * (b0 + kk));
    });
  if (ng > 1) {
    if (act) __stcg(reinterpret_cast<T*>(a.part2 + (size_t)(2 * b0 + j) * D + col), s);
    named_bar_sync(1, nct);
    if (t == 0) {
      __threadfence();
      uint32_t* c = a.cnt2 + ((size_t)b0 * ncb + cb);
      const uint32_t old = atomicAdd(c, 1u);
      m.last = (int)old == ng - 1;
      if (m.last) *c = 0u;
    }
    named_bar_sync(1, nct);
    if (!m.last) return;
    __threadfence();
    if (act) s = sum_rows<T>(a.part2, ng, D, col, [&](int q) { return (size_t)(2 * b0 + q); });
  }
  if (!act) return;
  if (a.apply) {
    const uint32_t w = __ldg(a.word + u);
    T* e = reinterpret_cast<T*>(a.table + (size_t)w * D + col);
    *e = V::fma(-a.lr, s, *e);
  } else {
    const int slot = a.l2g ? __ldg(a.l2g + u) : u;
    if (slot >= 0) V::st_m(a.M, (size_t)slot * D + col, s, a.m16, a.cF, a.cbf);
  }
}

// LMSCALE_PHASE_TRACE: [54] ~earliest CTA start, [55] latest CTA start,
// [56] latest prologue end, [57] ~earliest consumer end, [58] latest consumer end
__device__ __forceinline__ void seg_stamp(unsigned long long* tr, int i, bool earliest) {
  if (tr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(tr + i, earliest ? ~t : t);
  }
}

template <typename T, bool TMA>
__global__ void __launch_bounds__(SEG_MAX_THREADS) k_seg(SegArgs a) {
  using V = VT<T>;
  constexpr int VW = V::W;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ Meta m;
  __shared__ __align__(8) uint64_t bars[4 * SEG_MAX_SLOTS];

  const int tid = threadIdx.x;
  const int nct = a.nct;                      // consumer threads
  const int cb = blockIdx.y, ncb = gridDim.y;
  const int b = blockIdx.x, nR = gridDim.x;
  const int K = a.K, D = a.D;
  const int cw = min(a.cbw, D - cb * a.cbw) / VW;  // active columns (T units) of this block
  const uint32_t rbytes = (uint32_t)(cw * VW * 4);
  const int GR = a.gr, NS = a.nslot;
  const uint32_t RB = (uint32_t)a.cbw * 4u;   // slot stride of one row
  // one slot = a group of GR gradient rows, then (world 1) the E rows of the
  // runs that end whole inside the group (at most GR)
  const uint32_t SB = (uint32_t)(a.apply ? 2 * GR : GR) * RB;
  // [ring NS x SB][s_pos lmax][s_w lmax]
  uint32_t* s_pos = reinterpret_cast<uint32_t*>(smem + (size_t)NS * SB);
  uint32_t* s_w = s_pos + a.lmax;
  const uint32_t ring = smem_u32(smem);
  const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8u * SEG_MAX_SLOTS;

  if (TMA && tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full0 + 8u * s, 1u);
      mbar_init(empty0 + 8u * s, (uint32_t)(nct / 32));
    }
    fence_mbar_init();
  }
  if (a.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  seg_stamp(a.trace, 54, true);
  seg_stamp(a.trace, 55, false);
  if (a.clear_bits) {  // world 1: nobody reads the presence bits after S1
    for (int64_t w = ((int64_t)b * ncb + cb) * blockDim.x + tid; w < a.W;
         w += (int64_t)nR * ncb * blockDim.x)
      a.lbits[w] = 0u;
  }
  // an id >= vocab: no row of M or E is touched (every CTA reads the same flag)
  if (__ldcg(&a.sc1->err) & 1u) return;

  const int p0 = (int)((uint32_t)b * a.seg_len), p1 = min(K, p0 + (int)a.seg_len);
  const int L = p1 - p0;
  // ---- prologue: the range's rows, its runs (from S1's run starts), the
  // segment ends and what each end emits to
  for (int i = tid; i < L; i += blockDim.x) {
    s_pos[i] = (uint32_t)__ldg(a.perm + p0 + i);
    LMS_CHECK(s_pos[i] < (uint32_t)K);
  }
  const int u0 = __ldg(a.runfirst + b);
  const int un = __ldg(a.runfirst + b + 1);  // run holding p1 (or U at the end)
  const int ul = __ldg(a.lstart + un) == p1 ? un - 1 : un;  // run holding p1 - 1
  __syncthreads();
  for (int r = tid; r <= ul - u0; r += blockDim.x) {
    const int u = u0 + r;
    const int st = __ldg(a.lstart + u), en = __ldg(a.lstart + u + 1);
    const int e = min(en, p1) - 1 - p0;  // this range's last position of run u
    LMS_CHECK(e >= 0 && e < L && st < en && st <= p1 - 1);
    uint32_t f = F_END;
    if (st >= p0 && en <= p1) {
      f |= F_FULL;
      s_w[e] = a.apply ? __ldg(a.word + u) : (a.l2g ? (uint32_t)__ldg(a.l2g + u) : (uint32_t)u);
    }
    s_pos[e] |= f;
    if (r == 0) {
      m.u_first = u;
      m.ls_first = st;
      m.le_first = en;
      m.cut_l = st < p0;
    }
    if (u == ul) {
      m.u_last = u;
      m.ls_last = st;
      m.le_last = en;
      m.cut_r = en > p1;
    }
  }
  __syncthreads();

  seg_stamp(a.trace, 56, false);
  const int ng = (L + GR - 1) / GR;
  if (TMA && tid >= nct) {
    // ---------------------------------------------------------- producer warp
    // per group: arm the slot's barrier with the group's bytes, then lane j
    // copies gradient row j and (world 1) lane j's run end copies its E row
    // behind the group's rows, in run order
    const int lane = tid & 31;
    const uint64_t pol = policy_evict_first();
    const float* gsrc = a.grad + (size_t)cb * a.cbw;
    const float* esrc = a.table + (size_t)cb * a.cbw;
    for (int g = 0; g < ng; ++g) {
      const int s = g % NS, it = g / NS;
      if (it > 0) mbar_wait(empty0 + 8u * s, (uint32_t)(it - 1) & 1u);
      const int i0 = g * GR, n = min(GR, L - i0);
      const uint32_t f = lane < n ? s_pos[i0 + lane] : 0u;
      const bool e = a.apply && lane < n && (f & F_FULL);
      const unsigned em = __ballot_sync(FULL, e);
      if (lane == 0) mbar_arrive_tx(full0 + 8u * s, (uint32_t)(n + __popc(em)) * rbytes);
      __syncwarp();
      const uint32_t dst = ring + (uint32_t)s * SB;
      if (lane < n)
        bulk_g2s_hint(dst + (uint32_t)lane * RB, gsrc + (size_t)(f & F_ROW) * D, rbytes,
                      full0 + 8u * s, pol);
      if (e)
        bulk_g2s(dst + (uint32_t)(n + __popc(em & lanemask_lt())) * RB,
                 esrc + (size_t)s_w[i0 + lane] * D, rbytes, full0 + 8u * s);
    }
    return;
  }

  // ------------------------------------------------------------- consumers
  const int t = tid;
  const bool act = t < cw;
  const size_t col = (size_t)cb * a.cbw + (size_t)t * VW;
  T acc = V::zero();
  bool first_seg = true;
  for (int g = 0; g < ng; ++g) {
    const int s = TMA ? g % NS : 0, it = TMA ? g / NS : 0;
    const int i0 = g * GR, n = min(GR, L - i0);
    const T* slot = reinterpret_cast<const T*>(smem + (size_t)s * SB);
    if (TMA) mbar_wait(full0 + 8u * s, (uint32_t)it & 1u);
    int ne = 0;  // E rows of this group consumed so far
    for (int j = 0; j < n; ++j) {
      const uint32_t f = s_pos[i0 + j];
      if (act) {
        T x;
        if (TMA)
          x = slot[(size_t)j * (RB / sizeof(T)) + t];
        else
          x = V::ld_once(reinterpret_cast<const T*>(a.grad + (size_t)(f & F_ROW) * D + col));
        acc = V::add(acc, x);
      }
      if (f & F_END) {
        if (f & F_FULL) {
          const uint32_t wv = s_w[i0 + j];
          LMS_CHECK(a.apply ? wv < a.vocab : (int)wv < 0 || (int64_t)wv < a.mrows);
          if (a.apply) {
            T* dst = reinterpret_cast<T*>(a.table + (size_t)wv * D + col);
            if (act)
              *dst = V::fma(-a.lr, acc,
                            TMA ? slot[(size_t)(n + ne) * (RB / sizeof(T)) + t] : *dst);
            ++ne;
          } else if (act && (int)wv >= 0) {
            V::st_m(a.M, (size_t)wv * D + col, acc, a.m16, a.cF, a.cbf);
          }
        } else {
          // a piece of a run cut by this range's left or right edge
          const bool head = first_seg && m.cut_l;
          cut_piece<T>(a, m, head, acc, b, cb, ncb, nct, t, cw);
        }
        acc = V::zero();
        first_seg = false;
      }
    }
    if (TMA) {
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(empty0 + 8u * s);
    }
  }
  seg_stamp(a.trace, 57, true);
  seg_stamp(a.trace, 58, false);
}

// M rows of slots whose word is absent on this rank are exactly +0:
// the staged path and the NCCL all-reduce need every one of the U_g rows.
__global__ void __launch_bounds__(256) k_zero_absent(float* __restrict__ M, int D,
                                                     const uint32_t* __restrict__ ihat,
                                                     const uint32_t* __restrict__ lbits,
                                                     const Sc3* __restrict__ sc3,
                                                     const Sc1* __restrict__ sc1) {
  if ((sc1->err | sc3->err) & 1u) return;
  const int64_t ug = sc3->u_global;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < ug; r += nw) {
    const uint32_t w = __ldg(ihat + r);
    if ((__ldg(lbits + (w >> 5)) >> (w & 31u)) & 1u) continue;
    float* row = M + (size_t)r * D;
    for (int c = lane; c < D; c += 32) row[c] = 0.f;
  }
}

namespace {
template <typename T, bool TMA>
void seg_attrs(size_t smem) {
  static size_t set = 0;
  if (smem > set) {
    cudaFuncSetAttribute(k_seg<T, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    max_carveout((const void*)k_seg<T, TMA>);
    set = smem;
  }
}
}  // namespace

// CTAs per SM for rows of D floats (the vector path's 8 KB column blocks).
// fold: the world-1 kernel with S6 folded in (E rows staged beside the
// gradient rows); otherwise M rows are written (G > 1, staged calls).
static int seg_occ(int64_t D, bool fold) {
  static const int occ_env = getenv("LMSCALE_S4_OCC") ? atoi(getenv("LMSCALE_S4_OCC")) : 0;
  if (occ_env > 0) return std::min(occ_env, SEG_MAX_OCC);
  // measured best on B200: fold (tools/ab_s4.sh) 2 KB rows 4, 4 KB rows 3,
  // 8 KB rows 2; M rows (tools/ab_seg_emu.sh) 4 / 3 / 4
  const int64_t rb = std::min<int64_t>(D, 2048) * 4;
  return rb <= 2048 ? 4 : rb <= 4096 ? 3 : fold ? 2 : 4;
}

// ranges: one per CTA of seg_occ per SM, at most SEG_MAX_L positions each,
// at least 8 positions each; fixed length (the last one shorter), so a
// position's range is one 32-bit division
int seg_ranges(int64_t K, int64_t D, int num_sms, bool fold, uint32_t* seg_len) {
  const int64_t ncb = (D + 2047) / 2048;
  const int64_t cap = std::max<int64_t>(1, (int64_t)num_sms * seg_occ(D, fold) / ncb);
  const int64_t by_len = (K + SEG_MAX_L - 1) / SEG_MAX_L;
  const int64_t by_min = (K + 7) / 8;
  const int64_t n = std::max<int64_t>(1, std::max<int64_t>(by_len, std::min<int64_t>(cap, by_min)));
  const int64_t len = (K + n - 1) / n;
  if (seg_len) *seg_len = (uint32_t)len;
  return (int)((K + len - 1) / len);
}

// Launch geometry.  Measured on B200 (tools/gather_probe.cu, randomly
// permuted 2-8 KB rows): one CTA's bulk-copy stream saturates at 20-40 GB/s
// whatever its ring depth, so the SM's share of HBM (~44 GB/s) needs 2-4
// CTAs per SM with groups of 4-8 rows per mbarrier.
SegPlan seg_plan(int64_t K, int64_t D, bool vec, bool apply, bool fold, int num_sms) {
  SegPlan p{};
  p.tma = vec;
  const int vw = vec ? 4 : 1;
  p.cbw = (int)std::min<int64_t>(D, vec ? 2048 : 512);
  const int cols = (p.cbw + vw - 1) / vw;
  p.nct = (cols + 31) / 32 * 32;
  p.threads = p.nct + (vec ? 32 : 0);
  p.ncb = (int)((D + p.cbw - 1) / p.cbw);
  const int rb = p.cbw * 4;
  p.occ = seg_occ(D, fold);
  uint32_t len = 0;
  p.nr = seg_ranges(K, D, num_sms, fold, &len);
  p.lmax = (int)len;
  const size_t meta = 8 * (size_t)p.lmax;
  if (vec) {
    static const int gr_env = getenv("LMSCALE_S4_GR") ? atoi(getenv("LMSCALE_S4_GR")) : 0;
    // measured with seg_occ: fold 4 / 4 / 2 rows per group (2 / 4 / 8 KB
    // rows), M rows 8 / 4 / 4
    p.gr = gr_env > 0 ? gr_env : fold ? (rb <= 4096 ? 4 : 2) : (rb <= 2048 ? 8 : 4);
    const size_t budget = (size_t)(224 * 1024) / p.occ - meta - 1024;
    // a slot holds GR gradient rows and, at world 1, up to GR E rows
    // at least 2 slots, and the whole ring within one SM's shared memory
    while (p.gr > 1 && (size_t)2 * (apply ? 2 : 1) * p.gr * rb + meta > (size_t)(200 * 1024))
      p.gr /= 2;
    const size_t per_slot = (size_t)(apply ? 2 : 1) * p.gr * rb;
    p.nslot = (int)std::max<size_t>(2, std::min<size_t>(SEG_MAX_SLOTS, budget / per_slot));
  } else {
    p.gr = 8;
    p.nslot = 0;
  }
  p.neslot = 0;
  const size_t ring = vec ? (size_t)p.nslot * (apply ? 2 : 1) * p.gr * rb : 0;
  p.smem = ring + meta;
  return p;
}

int64_t seg_max_ranges(int64_t K, int num_sms) {
  return std::max<int64_t>((int64_t)num_sms * SEG_MAX_OCC, (K + SEG_MAX_L - 1) / SEG_MAX_L) + 1;
}

cudaError_t launch_seg(const SegArgs& a0, cudaStream_t s) {
  SegArgs a = a0;
  const bool vec = a.D % 4 == 0 && (uintptr_t)a.grad % 16 == 0 &&
                   (!a.apply || (uintptr_t)a.table % 16 == 0) &&
                   (a.apply || (uintptr_t)a.M % 16 == 0) && (uintptr_t)a.part % 16 == 0;
  const SegPlan p = seg_plan(a.K, a.D, vec, a.apply != 0, a.fold != 0, a.num_sms);
  a.cbw = p.cbw;
  a.nct = p.nct;
  a.gr = p.gr;
  a.nslot = p.nslot;
  a.neslot = p.neslot;
  a.lmax = p.lmax;
  a.seg_len = (uint32_t)p.lmax;
  const dim3 grid((unsigned)p.nr, (unsigned)p.ncb);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3((unsigned)p.threads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = a.pdl ? 1 : 0;
  if (vec) {
    seg_attrs<float4, true>(p.smem);
    return cudaLaunchKernelEx(&cfg, k_seg<float4, true>, a);
  }
  seg_attrs<float, false>(p.smem);
  return cudaLaunchKernelEx(&cfg, k_seg<float, false>, a);
}

cudaError_t launch_zero_absent(float* M, int D, const uint32_t* ihat, const uint32_t* lbits,
                               const Sc3* sc3, const Sc1* sc1, int64_t ug_cap, int num_sms,
                               cudaStream_t s) {
  if (ug_cap <= 0) return cudaSuccess;
  int64_t blocks = (ug_cap + 7) / 8;
  if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
  k_zero_absent<<<(unsigned)blocks, 256, 0, s>>>(M, D, ihat, lbits, sc3, sc1);
  return cudaGetLastError();
}

}  // namespace lms
