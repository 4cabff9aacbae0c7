// coop.cu -- S1 (local unique, step 1) and S3 (global unique +
// remap, step 4) as ONE launch each: a normal launch sized to
// co-residency, phases separated by an in-kernel grid barrier.
//
// Both steps touch at most a few MB (ids, bitmaps), so they are bound by
// latency, not bandwidth: a chain of dependent launches or a serial
// decoupled look-back costs more than the data movement.  Each step is
// therefore a single persistent cooperative kernel whose phases are separated
// by grid-wide barriers, and every cross-tile prefix is a parallel read of the
// per-tile counts (digit-major, vector loads) instead of a look-back chain.
//
// S1: stable LSD radix sort of (id, position) with up to 11-bit digits (two
//     passes for |V| <= 4M), warp multisplit ranking via __match_any_sync,
//     then run-length flags over the sorted ids -> J^ (ascending), run starts,
//     sorted-position -> u map, inverse map, local presence bitmap, U_i.
// S3: warp-aggregated test-then-set of a |V|-bit presence bitmap over the
//     gathered ids I (hot Zipf words cost one load per warp, not one atomic per
//     token), a popcount scan over the bitmap that emits I^ in ascending order
//     and the per-word rank table, U_g, and the J^ -> I^ map l2g.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace lms {

namespace {

constexpr int CT = CO_THREADS;
constexpr int NW = CO_THREADS / 32;
constexpr int IT = CO_ITEMS;

__device__ __forceinline__ void stamp(unsigned long long* tr, int i) {
  if (tr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[i] = t;
  }
}

// Block-wide sum (all threads get the result).
__device__ __forceinline__ uint32_t block_sum(uint32_t v, uint32_t* scratch) {
  uint32_t tot;
  block_excl_scan(v, scratch, &tot);
  return tot;
}

// Rank one tile of 4096 keys by the digit (key >> shift) & (ndig - 1).
// Striped warp layout: warp w owns tile keys w*256 + j*32 + lane, so the
// (w, j, lane) order is input order and the multisplit rank is stable.
// On return s_cnt[w][d] holds this warp's count of digit d and rank[j] the
// key's rank among equal digits of its warp.
__device__ __forceinline__ void rank_tile(const uint32_t* __restrict__ kin,
                                          const int32_t* __restrict__ vin, int K, int tile,
                                          int shift, int ndig, uint32_t* s_cnt,
                                          uint32_t (&key)[IT], int32_t (&val)[IT],
                                          uint32_t (&rank)[IT], uint32_t (&dig)[IT]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < NW * ndig; i += CT) s_cnt[i] = 0;
  const int base = tile * CO_TILE + warp * (32 * IT);
#pragma unroll
  for (int j = 0; j < IT; ++j) {
    const int idx = base + j * 32 + lane;
    if (idx < K) {
      key[j] = __ldcg(kin + idx);
      val[j] = vin ? __ldcg(vin + idx) : idx;
    } else {
      key[j] = 0;
      val[j] = -1;
    }
  }
  __syncthreads();
  uint32_t* wc = s_cnt + warp * ndig;
#pragma unroll
  for (int j = 0; j < IT; ++j) {
    const int idx = base + j * 32 + lane;
    const uint32_t d = idx < K ? ((key[j] >> shift) & (uint32_t)(ndig - 1)) : 0xffffffffu;
    dig[j] = d;
    const unsigned m = __match_any_sync(FULL, d);
    const uint32_t before = d != 0xffffffffu ? wc[d] : 0u;
    rank[j] = before + __popc(m & lanemask_lt());
    __syncwarp();
    if (d != 0xffffffffu && lane == (__ffs(m) - 1)) wc[d] = before + __popc(m);
    __syncwarp();
  }
  __syncthreads();
}

// Turn s_cnt[w][d] into exclusive offsets over warps; return nothing, write
// the tile's digit totals to cT[d][tile] when cT != nullptr.
__device__ __forceinline__ void warp_offsets(uint32_t* s_cnt, int ndig, uint32_t* cT,
                                             int ntp, int tile) {
  for (int d = threadIdx.x; d < ndig; d += CT) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t c = s_cnt[w * ndig + d];
      s_cnt[w * ndig + d] = run;
      run += c;
    }
    if (cT) cT[(size_t)d * ntp + tile] = run;
  }
}

}  // namespace

// --------------------------------------------------------------------- S1

__global__ void __launch_bounds__(CO_THREADS, 1) k_s1(S1Args a) {
  extern __shared__ uint32_t smem[];
  __shared__ uint32_t s_scan[32];
  const int ndig = 1 << a.bits;
  uint32_t* s_cnt = smem;                 // [NW][ndig]
  uint32_t* s_base = smem + NW * ndig;    // [ndig]
  const int tid = threadIdx.x;
  const int K = a.K;
  const bool single = a.ntiles <= (int)gridDim.x;

  stamp(a.trace, 0);
  // phase 0: zero the local bitmap and scalars (ordered by the first grid.sync)
  for (int64_t w = (int64_t)blockIdx.x * CT + tid; w < a.W; w += (int64_t)gridDim.x * CT)
    a.lbits[w] = 0u;
  if (blockIdx.x == 0 && tid == 0) {
    a.sc->err = 0u;
    a.sc->u_local = 0;
    a.sc->fixcount = 0u;
    if (a.sc3) {
      a.sc3->err = 0u;
      a.sc3->u_global = 0;
    }
  }
  bool bad = false;

  uint32_t key[IT], rank[IT], dig[IT];
  int32_t val[IT];
  const uint32_t* kin = a.ids;
  const int32_t* vin = nullptr;
  for (int p = 0; p < a.passes; ++p) {
    uint32_t* kout = (p & 1) ? a.kb : a.ka;
    int32_t* vout = (p & 1) ? a.vb : a.va;
    const int shift = p * a.bits;
    uint32_t* cT = a.cT + (size_t)p * ndig * a.ntp;
    // P1: per-tile digit counts (block 0 also zeroes the row padding)
    if (blockIdx.x == 0)
      for (int i = tid; i < ndig * (a.ntp - a.ntiles); i += CT)
        cT[(size_t)(i / (a.ntp - a.ntiles)) * a.ntp + a.ntiles + i % (a.ntp - a.ntiles)] = 0u;
    for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
      rank_tile(kin, vin, K, t, shift, ndig, s_cnt, key, val, rank, dig);
      if (p == 0) {
#pragma unroll
        for (int j = 0; j < IT; ++j) bad |= (dig[j] != 0xffffffffu) && key[j] >= a.vocab;
      }
      warp_offsets(s_cnt, ndig, cT, a.ntp, t);
      __syncthreads();
    }
    stamp(a.trace, 1 + 4 * p);
    grid_barrier(a.bar);
    stamp(a.trace, 2 + 4 * p);
    // Bases, distributed: CTA b owns digits [r0, r1).  A warp per digit scans
    // the digit's per-tile counts (one coalesced row of cT) into per-tile
    // exclusive prefixes; the CTA scans its digits' totals; range offsets are
    // combined across CTAs; every tile's bases land tile-major in bT.
    {
      const int nb = (int)gridDim.x;
      const int r0 = (int)((int64_t)ndig * blockIdx.x / nb);
      const int r1 = (int)((int64_t)ndig * (blockIdx.x + 1) / nb);
      const int warp = tid >> 5, lane = tid & 31;
      for (int d = r0 + warp; d < r1; d += NW) {
        const uint32_t* row = cT + (size_t)d * a.ntp;
        uint32_t carry = 0;
        for (int t0 = 0; t0 < a.ntiles; t0 += 32) {
          const int t = t0 + lane;
          const uint32_t v = t < a.ntiles ? __ldcg(row + t) : 0u;
          uint32_t x = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
          }
          if (t < a.ntiles) a.bT[(size_t)t * ndig + d] = carry + x - v;  // exclusive over tiles
          carry += __shfl_sync(FULL, x, 31);
        }
        if (lane == 0) s_base[d - r0] = carry;  // digit total
      }
      __syncthreads();
      // exclusive scan of this range's digit totals (<= 2048 / nb digits)
      const int nr = r1 - r0;
      const int dpt2 = (nr + CT - 1) / CT;
      uint32_t dt[8], my = 0;
      for (int k = 0; k < dpt2 && k < 8; ++k) {
        const int dl = tid * dpt2 + k;
        dt[k] = dl < nr ? s_base[dl] : 0u;
        my += dt[k];
      }
      uint32_t rtot;
      uint32_t ex = block_excl_scan(my, s_scan, &rtot);
      __syncthreads();
      for (int k = 0; k < dpt2 && k < 8; ++k) {
        const int dl = tid * dpt2 + k;
        if (dl < nr) s_base[dl] = ex;
        ex += dt[k];
      }
      if (tid == 0) a.rtot[blockIdx.x] = rtot;
      stamp(a.trace, 9 + 3 * p);
      grid_barrier(a.bar);
      uint32_t part = 0;
      for (int c = tid; c < (int)blockIdx.x; c += CT) part += __ldcg(a.rtot + c);
      const uint32_t roff = block_sum(part, s_scan);
      for (int i = tid; i < nr * a.ntiles; i += CT) {
        const int t = i / nr, dl = i % nr;
        uint32_t* pb = a.bT + (size_t)t * ndig + r0 + dl;
        *pb = __ldcg(pb) + roff + s_base[dl];
      }
      stamp(a.trace, 10 + 3 * p);
      grid_barrier(a.bar);
      stamp(a.trace, 11 + 3 * p);
    }
    // P2: this tile's bases (one coalesced row), then the stable scatter
    for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
      if (!single) {
        rank_tile(kin, vin, K, t, shift, ndig, s_cnt, key, val, rank, dig);
        warp_offsets(s_cnt, ndig, nullptr, a.ntp, t);
      }
      for (int d = tid; d < ndig; d += CT) s_base[d] = __ldcg(a.bT + (size_t)t * ndig + d);
      __syncthreads();
      const int warp = tid >> 5;
#pragma unroll
      for (int j = 0; j < IT; ++j) {
        const uint32_t d = dig[j];
        if (d != 0xffffffffu) {
          const uint32_t pos = s_base[d] + s_cnt[warp * ndig + d] + rank[j];
          kout[pos] = key[j];
          vout[pos] = val[j];
        }
      }
      __syncthreads();
    }
    stamp(a.trace, 3 + 4 * p);
    grid_barrier(a.bar);
    stamp(a.trace, 4 + 4 * p);
    kin = kout;
    vin = vout;
  }
  if (bad) {
    atomicOr(&a.sc->err, 1u);
    if (a.sc3) atomicOr(&a.sc3->err, 1u);
  }

  // ---- run-length flags over the sorted ids (blocked: 8 per thread)
  uint32_t heads = 0;
  uint32_t sk[IT];
  int32_t sv[IT];
  uint32_t prev_first = 0;  // key before this thread's slice (word heads)
  auto load_sorted = [&](int t) {
    const int i0 = t * CO_TILE + tid * IT;
    uint32_t prev = (i0 > 0 && i0 <= K) ? __ldcg(kin + i0 - 1) : 0u;
    prev_first = prev;
    heads = 0;
#pragma unroll
    for (int j = 0; j < IT; ++j) {
      const int i = i0 + j;
      sk[j] = i < K ? __ldcg(kin + i) : 0u;
      sv[j] = i < K ? __ldcg(vin + i) : 0;
      const bool h = i < K && (i == 0 || sk[j] != prev);
      heads |= (uint32_t)h << j;
      prev = sk[j];
    }
  };
  for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    load_sorted(t);
    const uint32_t tot = block_sum(__popc(heads), s_scan);
    if (tid == 0) a.heads[t] = tot;
  }
  stamp(a.trace, 20);
  grid_barrier(a.bar);
  stamp(a.trace, 21);
  for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    if (!single) load_sorted(t);
    uint32_t part = 0;
    for (int t2 = tid; t2 < t; t2 += CT) part += __ldcg(a.heads + t2);
    const uint32_t tile_excl = block_sum(part, s_scan);
    uint32_t dummy;
    uint32_t u_run = tile_excl + block_excl_scan(__popc(heads), s_scan, &dummy);
    const int i0 = t * CO_TILE + tid * IT;
    bool bad2 = false;
#pragma unroll
    for (int j = 0; j < IT; ++j) {
      const int i = i0 + j;
      if (i < K) {
        if ((heads >> j) & 1u) {
          a.luniq[u_run] = sk[j];
          a.lstart[u_run] = i;
          if (a.ihat) {
            a.ihat[u_run] = sk[j];
            a.l2g[u_run] = (int32_t)u_run;
          }
          if (sk[j] < a.vocab) {
            atomicOr(a.lbits + (sk[j] >> 5), 1u << (sk[j] & 31u));
            const uint32_t pkey = j == 0 ? prev_first : sk[j > 0 ? j - 1 : 0];
            if (a.lrank && (i == 0 || (pkey >> 5) != (sk[j] >> 5))) a.lrank[sk[j] >> 5] = u_run;
          } else {
            bad2 = true;
          }
          ++u_run;
        }
        a.segidx[i] = (int32_t)u_run - 1;
        a.inverse[sv[j]] = (int32_t)u_run - 1;
        if (i == K - 1) {
          a.sc->u_local = u_run;
          a.lstart[u_run] = K;
          if (a.nu_out) *a.nu_out = u_run;
          if (a.sc3) a.sc3->u_global = u_run;
        }
      }
    }
    if (bad2) {
      atomicOr(&a.sc->err, 1u);
      if (a.sc3) atomicOr(&a.sc3->err, 1u);
    }
    __syncthreads();
  }
  stamp(a.trace, 22);
}

// --------------------------------------------------------------------- S3

__global__ void __launch_bounds__(CO_THREADS, 1) k_s3(S3Args a) {
  __shared__ uint32_t s_scan[32];
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t gtid = (int64_t)blockIdx.x * CT + tid;
  const int64_t gthreads = (int64_t)gridDim.x * CT;

  stamp(a.trace, 32);
  if (a.peer_mode) {
    // handshake: this rank's S1 (the previous kernel on this stream) is
    // complete; tell every peer, then wait until every peer has said so
    // (flag = 2 * epoch + this rank's id-error bit: every rank learns every
    // rank's error, so all of them report it and none enters a collective alone)
    if (gtid == 0) {
      const uint32_t e = *a.epoch + 1u;
      *a.epoch = e;
      const uint32_t f = 2u * e + (__ldcg(&a.sc1->err) & 1u);
      __threadfence_system();
      for (int j = 0; j < a.world; ++j)
        st_release_sys(reinterpret_cast<uint32_t*>(a.peer_base[j] + a.flags_off) + a.rank, f);
      const uint32_t* mine = reinterpret_cast<const uint32_t*>(a.peer_base[a.rank] + a.flags_off);
      uint32_t err = 0u;
      for (int j = 0; j < a.world; ++j) {
        uint32_t v;
        while ((int32_t)((v = ld_acquire_sys(mine + j)) - 2u * e) < 0) __nanosleep(64);
        err |= v & 1u;
      }
      a.sc->err = err;
      a.sc->u_global = 0;
    }
    grid_barrier(a.bar);
    stamp(a.trace, 33);
    // phase A': the global presence bitmap = OR of the G local bitmaps
    for (int64_t w = gtid; w < a.W; w += gthreads) {
      uint32_t g = 0u;
#pragma unroll 8
      for (int j = 0; j < a.world; ++j)
        g |= __ldcv(reinterpret_cast<const uint32_t*>(a.peer_base[j] + a.lbits_off) + w);
      a.gbits[w] = g;
    }
    stamp(a.trace, 35);
    grid_barrier(a.bar);
    stamp(a.trace, 36);
  } else {
  // phase 0: zero the bitmap and scalars
  for (int64_t w = gtid; w < a.W; w += gthreads) a.gbits[w] = 0u;
  if (gtid == 0) {
    a.sc->err = 0u;
    a.sc->u_global = 0;
  }
  stamp(a.trace, 33);
  grid_barrier(a.bar);
  stamp(a.trace, 34);

  // phase A: presence bits.  Words < CO_HOTW (the head of a frequency-ordered
  // vocabulary, where Zipf puts most tokens) are OR-ed in shared memory first
  // and published with one test-then-set per CTA; the tail dedups equal ids in
  // the warp and does a test-then-set on the global word.
  __shared__ uint32_t s_hot[CO_HOTW];
  const int64_t hotw = a.W < CO_HOTW ? a.W : CO_HOTW;
  for (int i = tid; i < CO_HOTW; i += CT) s_hot[i] = 0u;
  __syncthreads();
  bool bad = false;
  // 4 ids per lane per round, loads issued together; warp-uniform trip count
  const int64_t wbase0 = (gtid >> 5) << 7;
  for (int64_t q0 = wbase0; q0 < a.n; q0 += 4 * gthreads) {
    uint32_t ids4[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t q = q0 + e * 32 + lane;
      ids4[e] = q < a.n ? __ldcs(a.I + q) : 0xffffffffu;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t q = q0 + e * 32 + lane;
      const uint32_t id = ids4[e];
      const bool valid = q < a.n && id < a.vocab;
      bad |= (q < a.n && !valid);
      const uint32_t w = id >> 5, b = 1u << (id & 31u);
      const bool hot = valid && w < hotw;
      // convergent: every lane of the warp takes part in the match
      const unsigned m = __match_any_sync(FULL, (valid && !hot) ? id : 0xffffffffu);
      if (hot) {
        atomicOr(s_hot + w, b);
      } else if (valid && lane == (unsigned)(__ffs(m) - 1)) {
        uint32_t* p = a.gbits + w;
        if (!(__ldcg(p) & b)) atomicOr(p, b);
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < hotw; i += CT) {
    const uint32_t b = s_hot[i];
    if (b && (__ldcg(a.gbits + i) & b) != b) atomicOr(a.gbits + i, b);
  }
  if (bad) atomicOr(&a.sc->err, 1u);
  stamp(a.trace, 35);
  grid_barrier(a.bar);
  stamp(a.trace, 36);
  }  // !peer_mode

  // phase B: popcounts of this CTA's word range (one word per thread per round)
  const int64_t per = (a.W + gridDim.x - 1) / gridDim.x;
  const int64_t w0 = (int64_t)blockIdx.x * per;
  const int64_t w1 = min(a.W, w0 + per);
  uint32_t cnt = 0;
  for (int64_t w = w0 + tid; w < w1; w += CT) cnt += __popc(__ldcg(a.gbits + w));
  const uint32_t cta_tot = block_sum(cnt, s_scan);
  if (tid == 0) a.ctot[blockIdx.x] = cta_tot;
  stamp(a.trace, 37);
  grid_barrier(a.bar);
  stamp(a.trace, 38);

  // phase C: CTA prefix, per-word ranks, ascending I^ emission.  Emission is
  // warp-cooperative: for each of the warp's 32 words, lane b writes id
  // 32w + b at rank r_w + popc(bits below b) -- one coalesced store per word.
  uint32_t part = 0;
  for (int c = tid; c < (int)blockIdx.x; c += CT) part += __ldcg(a.ctot + c);
  uint32_t run = block_sum(part, s_scan);
  if (blockIdx.x == gridDim.x - 1 && tid == 0) a.sc->u_global = run + cta_tot;
  for (int64_t wr = w0; wr < w1; wr += CT) {
    const int64_t w = wr + tid;
    const uint32_t wd = w < w1 ? __ldcg(a.gbits + w) : 0u;
    uint32_t round_tot;
    const uint32_t r = run + block_excl_scan(__popc(wd), s_scan, &round_tot);
    if (w < w1) a.wrank[w] = r;
    for (int src = 0; src < 32; ++src) {
      const uint32_t bits = __shfl_sync(FULL, wd, src);
      const uint32_t rs = __shfl_sync(FULL, r, src);
      if ((bits >> lane) & 1u)
        a.ihat[rs + __popc(bits & lanemask_lt())] = (uint32_t)((wr + (tid & ~31) + src) * 32 + lane);
    }
    run += round_tot;
  }
  stamp(a.trace, 39);
  if (!a.luniq) return;
  grid_barrier(a.bar);
  stamp(a.trace, 40);

  // phase D: l2g[u] = slot of J^[u] in I^ (S1 of this rank has completed)
  const int U = (int)a.sc1->u_local;
  for (int64_t u = gtid; u < U; u += gthreads) {
    const uint32_t w = __ldcg(a.luniq + u);
    int32_t slot = -1;
    if (w < a.vocab) {
      const uint32_t below = __ldcg(a.gbits + (w >> 5)) & ((1u << (w & 31u)) - 1u);
      slot = (int32_t)(__ldcg(a.wrank + (w >> 5)) + __popc(below));
    }
    a.l2g[u] = slot;
  }
  stamp(a.trace, 41);
}

// ------------------------------------------------- counts / staged export

__global__ void k_counts_export(const int32_t* __restrict__ lstart,
                                const uint32_t* __restrict__ luniq,
                                const int32_t* __restrict__ inverse, const Sc1* __restrict__ sc,
                                int K, int32_t* __restrict__ counts,
                                uint32_t* __restrict__ uniq_out, int32_t* __restrict__ counts_out,
                                int32_t* __restrict__ inverse_out) {
  const int U = (int)sc->u_local;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < K; i += gridDim.x * blockDim.x) {
    if (i < U) {
      int c = lstart[i + 1] - lstart[i];
      counts[i] = c;
      if (counts_out) counts_out[i] = c;
      if (uniq_out) uniq_out[i] = luniq[i];
    }
    if (inverse_out) inverse_out[i] = inverse[i];
  }
}

void launch_counts_export(const int32_t* lstart, const uint32_t* luniq, const int32_t* inverse,
                          const Sc1* sc, int K, int32_t* counts, uint32_t* uniq_out,
                          int32_t* counts_out, int32_t* inverse_out, cudaStream_t s) {
  int blocks = (K + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  k_counts_export<<<blocks, 256, 0, s>>>(lstart, luniq, inverse, sc, K, counts, uniq_out,
                                         counts_out, inverse_out);
}

// ------------------------------------------------------------------ launch

SortPlan make_coop_plan(uint64_t vocab) {
  int bits = 1;
  while (bits < 32 && (1ull << bits) < vocab) ++bits;
  SortPlan p;
  p.passes = (bits + CO_MAX_BITS - 1) / CO_MAX_BITS;
  p.bits = (bits + p.passes - 1) / p.passes;
  return p;
}

size_t s1_smem_bytes(int bits) { return (size_t)(NW + 1) * (1u << bits) * 4; }

int coop_grid_s1(int ntiles, int num_sms) {
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(k_s1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)s1_smem_bytes(CO_MAX_BITS));
    max_carveout((const void*)k_s1);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_s1, CO_THREADS,
                                                      s1_smem_bytes(CO_MAX_BITS)) != cudaSuccess ||
        occ < 1)
      occ = 1;
  }
  const int cap = num_sms * occ;
  return ntiles < cap ? ntiles : cap;
}

cudaError_t launch_s1(const S1Args& a, int num_sms, cudaStream_t s) {
  const int grid = coop_grid_s1(a.ntiles, num_sms);
  // grid <= co-resident capacity: the in-kernel barrier is safe with a normal launch
  k_s1<<<grid, CO_THREADS, s1_smem_bytes(a.bits), s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_s3(const S3Args& a, int num_sms, cudaStream_t s) {
  static int occ = -1;
  if (occ < 0) {
    max_carveout((const void*)k_s3);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_s3, CO_THREADS, 0) != cudaSuccess ||
        occ < 1)
      occ = 1;
  }
  // enough CTAs for the id and word volumes, few enough that barriers stay cheap
  int64_t want = (a.n + 4095) / 4096;
  // peer mode: one remote word per thread per peer in the OR phase
  const int64_t ww = a.peer_mode ? (a.W + CO_THREADS - 1) / CO_THREADS : (a.W + 2047) / 2048;
  if (ww > want) want = ww;
  if (want < 1) want = 1;
  const int64_t cap = (int64_t)num_sms * occ;
  const int grid = (int)(want < cap ? want : cap);
  k_s3<<<grid, CO_THREADS, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace lms
