// group.cu -- S1, the local unique of step 1 with the grouping of
// step 2, as ONE launch over every SM: a counting sort keyed by
// the vocabulary itself instead of a comparison or radix sort of the ids.
//
// The K ids of a rank index a |V|-entry count array and a |V|-bit presence
// bitmap, so the sorted distinct set J^ is simply the set bits of the bitmap
// in ascending order and the rank of an id in J^ is a popcount:
//
//   PA  CTA b takes a contiguous chunk of tokens and counts its ids in a
//       shared-memory hash table (each token gets its rank among the chunk's
//       equal ids); then one global atomicAdd per distinct id per chunk,
//       wcount[id] += c, returns the chunk's base, and a token's ticket is
//       base + rank.  The chunk that draws base 0 sets the id's presence bit.
//       Per-range totals (present ids, tokens) for PC's word ranges are
//       accumulated on the way.  The Zipf head costs one global atomic per
//       chunk, not one per token.                           -- grid barrier --
//   PC  CTA b owns a contiguous range of 32-id bitmap words: prefix of the
//       range totals, then warp per word (lane = bit): lrank[w] (index in J^
//       of the first present id of word w) and, per present id, J^[u],
//       counts[u] and lstart[u] (first grouped position of its run).
//                                                           -- grid barrier --
//   PD  per token p: u = lrank[w] + popc(bits below) (the inverse map),
//       grouped position lstart[u] + ticket[p]: perm, the grouped order that
//       S4 walks; the token at the first position of an S4 range records the
//       range's first run (runfirst).  (wcount returns to zero in PC, once per
//       present id.)
//
// Two grid barriers in a normally-launched kernel sized to co-residency (one
// CTA per SM).  The grouping is a counting sort, so the tokens of one word are
// contiguous in perm but in ticket order, not position order (R18):
// S4 sums each run in that order.  Every integer output -- J^, counts,
// inverse, lstart, U_i -- is unique and bit-exact.
//
// Invariants between launches: wcount and the range totals are all zero (PC
// and PD clear what PA set).  lbits must be zero on entry; a.zero_bits asks
// this kernel to clear it first (one more barrier) -- at world 1 the S4 kernel
// clears it after use.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace lms {

namespace {

constexpr int GT = G1_THREADS;

__device__ __forceinline__ void gstamp(unsigned long long* tr, int i) {
  if (tr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[i] = t;
  }
}

// latest over the CTAs of a phase end (slot i), and (slot i + 3) the CTA that
// set it (diagnostic; racy between near-equal times)
__device__ __forceinline__ void gstamp_last(unsigned long long* tr, int i) {
  if (tr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (atomicMax(tr + i, t) < t) tr[i + 3] = blockIdx.x;
  }
}

// Block-wide exclusive scan of (a, b) pairs; totals returned through *ta, *tb.
__device__ __forceinline__ void block_scan2(uint32_t a, uint32_t b, uint32_t& ea, uint32_t& eb,
                                            uint32_t& ta, uint32_t& tb, uint32_t* s_a,
                                            uint32_t* s_b) {
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t xa = a, xb = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t ya = __shfl_up_sync(FULL, xa, o), yb = __shfl_up_sync(FULL, xb, o);
    if (lane >= (unsigned)o) {
      xa += ya;
      xb += yb;
    }
  }
  if (lane == 31) {
    s_a[warp] = xa;
    s_b[warp] = xb;
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t va = lane < nw ? s_a[lane] : 0u, vb = lane < nw ? s_b[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t ya = __shfl_up_sync(FULL, va, o), yb = __shfl_up_sync(FULL, vb, o);
      if (lane >= (unsigned)o) {
        va += ya;
        vb += yb;
      }
    }
    s_a[lane] = va;
    s_b[lane] = vb;
  }
  __syncthreads();
  ea = (warp ? s_a[warp - 1] : 0u) + xa - a;
  eb = (warp ? s_b[warp - 1] : 0u) + xb - b;
  ta = s_a[nw - 1];
  tb = s_b[nw - 1];
  __syncthreads();
}

constexpr int HS = 4096;          // hash slots per CTA (load factor <= 1/2)
constexpr int SUB = 2048;         // tokens per hash round
constexpr int TPT = SUB / GT;     // tokens per thread per round
constexpr uint32_t EMPTY = 0xffffffffu;

__device__ __forceinline__ uint32_t hslot(uint32_t id) { return (id * 0x9E3779B1u) >> 20; }

// wcount is stored transposed (index (id % 32) * W + id / 32): consecutive ids
// -- the Zipf head of a frequency-ordered vocabulary -- fall in different
// cache lines, so the chunks' atomics on hot ids do not queue on one line,
// and PC's loads of a 32-word chunk (lane = word, fixed bit) stay coalesced.
// (A multiplicative-hash layout spread the atomics further -- tieba PA 6.3 ->
// 5.1 us -- but made every PC load scattered: amazon PC 10 -> 37 us.)
__device__ __forceinline__ size_t widx(uint32_t id, int64_t W) {
  return (size_t)(id & 31u) * (size_t)W + (id >> 5);
}
constexpr int NST = G1_STRIPES;  // range-total stripes (chunk b adds into stripe b % NST)

}  // namespace

__global__ void __launch_bounds__(G1_THREADS, 1) k_group(G1Args a) {
  __shared__ uint32_t s_a[32], s_b[32];
  // PA: hash table + range totals; PC: one 32 x 33 count tile per warp
  extern __shared__ __align__(16) uint32_t g_smem[];
  uint32_t* h_key = g_smem;
  uint32_t* h_cnt = g_smem + HS;
  uint32_t* s_ru = g_smem + 2 * HS;
  uint32_t* s_rt = s_ru + G1_MAX_GRID;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t gtid = (int64_t)blockIdx.x * GT + tid;
  const int64_t gthreads = (int64_t)gridDim.x * GT;
  const int K = a.K, nb = gridDim.x;
  const uint32_t per = (uint32_t)((a.W + nb - 1) / nb);  // bitmap words per PC range
  gstamp(a.trace, 0);

  if (gtid == 0) {
    a.sc->err = 0u;
    a.sc->u_local = 0;
    a.sc->fixcount = 0u;
    if (a.sc3) {
      a.sc3->err = 0u;
      a.sc3->u_global = 0;
    }
  }
  for (int i = tid; i < HS; i += GT) {
    h_key[i] = EMPTY;
    h_cnt[i] = 0u;
  }
  for (int i = tid; i < nb; i += GT) s_ru[i] = s_rt[i] = 0u;
  if (a.zero_bits) {
    for (int64_t w = gtid; w < a.W; w += gthreads) a.lbits[w] = 0u;
    grid_barrier(a.bar);
  }
  __syncthreads();

  gstamp(a.trace, 10);
  // ---- PA: tickets, presence bits, range totals
  const int q0 = (int)((int64_t)blockIdx.x * K / nb), q1 = (int)((int64_t)(blockIdx.x + 1) * K / nb);
  bool bad = false;
  for (int sub = q0; sub < q1; sub += SUB) {
    const int n = min(SUB, q1 - sub);
    uint32_t id[TPT], slot[TPT], rk[TPT];
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      const int i = tid + k * GT;
      id[k] = i < n ? __ldg(a.ids + sub + i) : EMPTY;
    }
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      slot[k] = EMPTY;
      const int i = tid + k * GT;
      if (i < n && id[k] >= a.vocab) bad = true;
      if (i < n && id[k] < a.vocab) {
        uint32_t h = hslot(id[k]);
        while (true) {
          const uint32_t prev = atomicCAS(h_key + h, EMPTY, id[k]);
          if (prev == EMPTY || prev == id[k]) break;
          h = (h + 1) & (HS - 1);
        }
        slot[k] = h;
        rk[k] = atomicAdd(h_cnt + h, 1u);
      }
    }
    __syncthreads();
    gstamp(a.trace, 11);
    // one global atomic per distinct id of the round: base of this chunk
    // (all of a thread's slots issued together)
    {
      constexpr int SPT = HS / GT;
      uint32_t key[SPT], cnt[SPT], base[SPT];
#pragma unroll
      for (int q = 0; q < SPT; ++q) {
        key[q] = h_key[tid + q * GT];
        cnt[q] = h_cnt[tid + q * GT];
      }
#pragma unroll
      for (int q = 0; q < SPT; ++q)
        base[q] = key[q] != EMPTY ? atomicAdd(a.wcount + widx(key[q], a.W), cnt[q]) : 0u;
#pragma unroll
      for (int q = 0; q < SPT; ++q)
        if (key[q] != EMPTY) h_cnt[tid + q * GT] = base[q];
      gstamp(a.trace, 13);
#pragma unroll
      for (int q = 0; q < SPT; ++q) {
        if (key[q] == EMPTY) continue;
        LMS_CHECK(key[q] < a.vocab && base[q] + cnt[q] <= (uint32_t)a.K);
        const int r = (int)((key[q] >> 5) / per);  // 32-bit division
        if (base[q] == 0u) {
          atomicOr(a.lbits + (key[q] >> 5), 1u << (key[q] & 31u));
          atomicAdd(s_ru + r, 1u);
        }
        atomicAdd(s_rt + r, cnt[q]);
      }
    }
    __syncthreads();
    gstamp(a.trace, 12);
#pragma unroll
    for (int k = 0; k < TPT; ++k)
      if (slot[k] != EMPTY) a.tick[sub + tid + k * GT] = h_cnt[slot[k]] + rk[k];
    __syncthreads();
    for (int e = tid; e < HS; e += GT) {
      h_key[e] = EMPTY;
      h_cnt[e] = 0u;
    }
    __syncthreads();
  }
  {
    uint32_t* st = a.ctot + (size_t)(blockIdx.x % NST) * 2 * nb;
    for (int r = tid; r < nb; r += GT) {
      if (s_ru[r]) atomicAdd(st + 2 * r, s_ru[r]);
      if (s_rt[r]) atomicAdd(st + 2 * r + 1, s_rt[r]);
    }
  }
  if (bad) {
    atomicOr(&a.sc->err, 1u);
    if (a.sc3) atomicOr(&a.sc3->err, 1u);
  }
  gstamp(a.trace, 1);
  gstamp_last(a.trace, 16);
  grid_barrier(a.bar);
  gstamp(a.trace, 2);

  // ---- PC: J^, counts, lstart, lrank over this CTA's word range
  {
    const int64_t w0 = (int64_t)blockIdx.x * per;
    const int64_t w1 = min(a.W, w0 + (int64_t)per);
    // this range's prefix: the totals of every earlier range (all stripes)
    uint32_t pu = 0, pt = 0;
    for (int c = tid; c < (int)blockIdx.x; c += GT) {
#pragma unroll
      for (int sI = 0; sI < NST; ++sI) {
        pu += __ldcg(a.ctot + (size_t)sI * 2 * nb + 2 * c);
        pt += __ldcg(a.ctot + (size_t)sI * 2 * nb + 2 * c + 1);
      }
    }
    uint32_t ea, eb, ta, tb;
    block_scan2(pu, pt, ea, eb, ta, tb, s_a, s_b);
    const uint32_t cta_u = ta, cta_t = tb;
    gstamp(a.trace, 7);
    const int nwarps = GT / 32;
    const int64_t nw = w1 > w0 ? w1 - w0 : 0;
    const int64_t ws = (nw + nwarps - 1) / nwarps;
    const int64_t x0 = w0 + warp * ws, x1 = min(w1, x0 + ws);
    // The counts of a 32-word chunk are loaded lane = word (wcount is
    // transposed: for a fixed bit i the 32 words' counts are contiguous, so
    // each load is coalesced) into a padded 32 x 33 tile, then read back
    // lane = bit for the scans and the coalesced emission.
    uint32_t* tile = g_smem + warp * (32 * 33);
    // (the counts are returned to zero right after they are read, once per
    // id -- zeroing them per token in PD queued thousands of stores on the
    // Zipf head's counters: 15 us at tieba)
    // The tile holds, per (bit i, word), the INCLUSIVE prefix of the word's
    // counts over bits 0..i, summed by the word's lane in registers: the
    // emission below reads a run's start and count from two tile entries
    // instead of a per-word warp scan (its shuffle chain serialised the
    // words: ~3 us of the Zipf head's ranges at 1b).
    auto load_chunk = [&](int64_t xc, uint32_t& mybits, bool zero) -> uint32_t {
      const int64_t myw = xc + lane;
      mybits = myw < x1 ? __ldcg(a.lbits + myw) : 0u;
      uint32_t v[32], tot = 0;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        v[i] = ((mybits >> i) & 1u) ? __ldcg(a.wcount + (size_t)i * a.W + myw) : 0u;
      if (zero) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if ((mybits >> i) & 1u) a.wcount[(size_t)i * a.W + myw] = 0u;
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        tot += v[i];
        tile[i * 33 + lane] = tot;
      }
      __syncwarp();
      return tot;  // this lane's word total
    };
    // pass 1: this warp's totals
    uint32_t wu = 0, wt = 0, bits0 = 0, tot0 = 0;
    const bool one_chunk = x1 - x0 <= 32;
    for (int64_t xc = x0; xc < x1; xc += 32) {
      uint32_t mybits;
      tot0 = load_chunk(xc, mybits, one_chunk);
      wt += tot0;
      wu += __popc(mybits);
      bits0 = mybits;
      __syncwarp();
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      wu += __shfl_xor_sync(FULL, wu, o);
      wt += __shfl_xor_sync(FULL, wt, o);
    }
    gstamp(a.trace, 8);
    // exclusive prefix over the CTA's warps (one contribution per warp: lane 0)
    block_scan2(lane == 0 ? wu : 0u, lane == 0 ? wt : 0u, ea, eb, ta, tb, s_a, s_b);
    uint32_t bu = cta_u + __shfl_sync(FULL, ea, 0), bt = cta_t + __shfl_sync(FULL, eb, 0);
    gstamp(a.trace, 9);
    // pass 2: emit J^, counts, lstart, lrank (lane = bit: coalesced stores)
    for (int64_t xc = x0; xc < x1; xc += 32) {
      uint32_t mybits = bits0, mytot = tot0;
      if (!one_chunk) mytot = load_chunk(xc, mybits, true);
      // per-word bases (lane = word): exclusive scans of ids and tokens
      uint32_t su = __popc(mybits), stt = mytot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t yu = __shfl_up_sync(FULL, su, o), yt = __shfl_up_sync(FULL, stt, o);
        if (lane >= o) {
          su += yu;
          stt += yt;
        }
      }
      const uint32_t wbu = bu + su - __popc(mybits), wbt = bt + stt - mytot;
      const int nwc = (int)(x1 - xc < 32 ? x1 - xc : 32);
      for (int j = 0; j < nwc; ++j) {
        const int64_t w = xc + j;
        const uint32_t bits = __shfl_sync(FULL, mybits, j);
        const uint32_t ubase = __shfl_sync(FULL, wbu, j), tbase = __shfl_sync(FULL, wbt, j);
        const bool has = (bits >> lane) & 1u;
        const uint32_t inc = tile[lane * 33 + j];
        const uint32_t exc = lane ? tile[(lane - 1) * 33 + j] : 0u;
        if (lane == 0) a.lrank[w] = ubase;
        if (has) {
          const uint32_t id = (uint32_t)(w * 32 + lane);
          const uint32_t u = ubase + __popc(bits & lanemask_lt());
          LMS_CHECK(u < (uint32_t)a.K && tbase + inc <= (uint32_t)a.K && id < a.vocab);
          a.luniq[u] = id;
          a.counts[u] = (int32_t)(inc - exc);
          a.lstart[u] = (int32_t)(tbase + exc);
          if (a.ihat) {
            a.ihat[u] = id;
            a.l2g[u] = (int32_t)u;
          }
        }
      }
      bu += __shfl_sync(FULL, su, 31);
      bt += __shfl_sync(FULL, stt, 31);
      __syncwarp();
    }
    // the last range ends at U_i (ids) and the valid token count
    if (blockIdx.x == nb - 1 && warp == nwarps - 1 && lane == 0) {
      a.sc->u_local = bu;
      a.lstart[bu] = (int32_t)bt;
      a.runfirst[a.nr] = (int32_t)bu;
      if (a.nu_out) *a.nu_out = bu;
      if (a.sc3) a.sc3->u_global = bu;
    }
  }
  gstamp(a.trace, 3);
  gstamp_last(a.trace, 17);
  grid_barrier(a.bar);
  gstamp(a.trace, 4);
  if (tid < NST) {  // this range's totals return to zero for the next launch
    a.ctot[(size_t)tid * 2 * nb + 2 * blockIdx.x] = 0u;
    a.ctot[(size_t)tid * 2 * nb + 2 * blockIdx.x + 1] = 0u;
  }

  // ---- PD: inverse map and the grouped order, TPT tokens per thread in flight
  for (int sub = q0; sub < q1; sub += SUB) {
    const int n = min(SUB, q1 - sub);
    uint32_t id[TPT], bits[TPT], base[TPT], t[TPT];
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      const int i = tid + k * GT;
      id[k] = i < n ? __ldg(a.ids + sub + i) : EMPTY;
      t[k] = i < n ? __ldcg(a.tick + sub + i) : 0u;
    }
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      bits[k] = 0u;
      base[k] = 0u;
      if (id[k] < a.vocab) {
        bits[k] = __ldca(a.lbits + (id[k] >> 5));
        base[k] = __ldca(a.lrank + (id[k] >> 5));
      }
    }
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      const int i = tid + k * GT;
      if (i >= n) continue;
      if (id[k] >= a.vocab) {
        a.inverse[sub + i] = -1;
        continue;
      }
      const uint32_t u = base[k] + __popc(bits[k] & ((1u << (id[k] & 31u)) - 1u));
      a.inverse[sub + i] = (int32_t)u;
      base[k] = u;
    }
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      const int i = tid + k * GT;
      if (i < n && id[k] < a.vocab) {
        const uint32_t spos = (uint32_t)__ldca(a.lstart + base[k]) + t[k];
        LMS_CHECK(spos < (uint32_t)a.K && spos / a.seg_len <= (uint32_t)a.nr);
        a.perm[spos] = sub + i;
        // the S4 range starting here begins inside run u
        if (spos % a.seg_len == 0u) a.runfirst[spos / a.seg_len] = (int32_t)base[k];
      }
    }
  }
  gstamp(a.trace, 5);
  gstamp_last(a.trace, 18);
}

constexpr size_t G1_SMEM = std::max<size_t>(4 * (2 * HS + 2 * G1_MAX_GRID),
                                             4 * (GT / 32) * 32 * 33);

int group_grid(int num_sms) {
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(k_group, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G1_SMEM);
    max_carveout((const void*)k_group);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_group, GT, G1_SMEM) != cudaSuccess ||
        occ < 1)
      occ = 1;
  }
  static const int want = getenv("LMSCALE_S1_CTAS") ? atoi(getenv("LMSCALE_S1_CTAS")) : 0;
  const int cap = std::min(num_sms * occ, G1_MAX_GRID);
  const int g = want > 0 ? want : num_sms;
  return g < cap ? g : cap;
}

cudaError_t launch_group(const G1Args& a, int num_sms, cudaStream_t s) {
  // grid <= co-resident capacity: the in-kernel barrier is safe with a normal launch
  const int grid = group_grid(num_sms);
  k_group<<<grid, GT, G1_SMEM, s>>>(a);
  return cudaGetLastError();
}

}  // namespace lms
