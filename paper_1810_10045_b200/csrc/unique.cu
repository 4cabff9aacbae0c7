// unique.cu -- S1 (local unique) and S3 (global unique + remap,
// P:410-414) for sm_100a.
//
// S1 is a stable LSD radix sort of (id, position) pairs -- one histogram
// launch for every pass, then one single-sweep launch per pass with
// warp-level multisplit ranking (__match_any_sync) and decoupled look-back
// across tiles -- followed by run-length flagging of the sorted ids with a
// block scan + look-back that emits J^, segment starts, the sorted-position ->
// u map and the inverse map.
//
// S3 never sorts the G*K gathered ids: it sets one bit per id in a |V|-bit
// presence bitmap (test-then-atomicOr, so hot Zipf words cost a load, not an
// atomic), then one look-back scan of popcounts over the bitmap yields I^ in
// ascending order (R2), U_g, and a per-word rank table; slot(w) =
// wrank[w/32] + popc(bits below w) is then O(1).
#include "common.cuh"
#include "kernels.cuh"

namespace lms {

SortPlan make_sort_plan(uint64_t vocab) {
  int bits = 1;
  while (bits < 32 && (1ull << bits) < vocab) ++bits;  // ids < vocab need `bits` bits
  int passes = (bits + 7) / 8;
  SortPlan p;
  p.passes = passes;
  p.bits = (bits + passes - 1) / passes;
  return p;
}

// ------------------------------------------------------------------ S1 sort

__global__ void __launch_bounds__(RS_THREADS) k_radix_hist(const uint32_t* __restrict__ keys,
                                                           int K, int passes, int bits,
                                                           uint32_t* __restrict__ hist,
                                                           Sc1* __restrict__ sc,
                                                           uint32_t vocab) {
  __shared__ uint32_t sh[RS_MAX_PASSES][256];
  for (int i = threadIdx.x; i < RS_MAX_PASSES * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  const uint32_t mask = (1u << bits) - 1u;
  bool bad = false;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < K; i += gridDim.x * blockDim.x) {
    uint32_t k = keys[i];
    bad |= (k >= vocab);
    for (int p = 0; p < passes; ++p) atomicAdd(&sh[p][(k >> (p * bits)) & mask], 1u);
  }
  if (__any_sync(FULL, bad) && lane_id() == 0) atomicOr(&sc->err, 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
    uint32_t v = (&sh[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

// One LSD pass: stable scatter of (key, val) by digit (pass * bits).
// Striped warp layout: warp w of tile t owns keys t*4096 + w*512 + j*32 + lane,
// so (j, lane) order is input order and the multisplit rank is stable.
__global__ void __launch_bounds__(RS_THREADS) k_radix_pass(
    const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin,
    uint32_t* __restrict__ kout, int32_t* __restrict__ vout, int K, int shift, int bits,
    const uint32_t* __restrict__ hist, uint32_t* __restrict__ lb, uint32_t* tile_ctr) {
  constexpr int NW = RS_THREADS / 32;
  __shared__ uint32_t s_cnt[NW][256];  // per-warp digit counts -> exclusive offsets
  __shared__ uint32_t s_base[256];     // global start of each digit for this tile
  __shared__ uint32_t s_scan[32];
  __shared__ uint32_t s_tile;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int i = threadIdx.x; i < NW * 256; i += blockDim.x) (&s_cnt[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t mask = (1u << bits) - 1u;
  const int base = (int)tile * RS_TILE + (int)warp * (32 * RS_ITEMS);

  uint32_t key[RS_ITEMS];
  int32_t val[RS_ITEMS];
  uint32_t rank[RS_ITEMS];
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    int idx = base + j * 32 + (int)lane;
    if (idx < K) {
      key[j] = kin[idx];
      val[j] = vin ? vin[idx] : idx;
    } else {
      key[j] = 0;
      val[j] = -1;
    }
  }
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    int idx = base + j * 32 + (int)lane;
    uint32_t d = idx < K ? ((key[j] >> shift) & mask) : 256u;  // 256 = padding
    unsigned m = __match_any_sync(FULL, d);
    uint32_t before = d < 256u ? s_cnt[warp][d] : 0u;
    rank[j] = before + __popc(m & lanemask_lt());
    __syncwarp();
    if (d < 256u && lane == (unsigned)(__ffs(m) - 1)) s_cnt[warp][d] = before + __popc(m);
    __syncwarp();
  }
  __syncthreads();
  // Thread t owns digit t: exclusive offsets over warps, tile total, look-back.
  const uint32_t t = threadIdx.x;  // RS_THREADS == 256
  uint32_t run = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    uint32_t c = s_cnt[w][t];
    s_cnt[w][t] = run;
    run += c;
  }
  uint32_t htot;
  uint32_t dstart = block_excl_scan(hist[t], s_scan, &htot);  // global digit start
  uint32_t* st = lb + (size_t)tile * 256 + t;
  uint32_t excl = 0;
  if (tile == 0) {
    st_release(st, LB_INC | run);
  } else {
    st_release(st, LB_AGG | run);
    int tt = (int)tile - 1;
    while (true) {
      uint32_t sv = ld_acquire(lb + (size_t)tt * 256 + t);
      if ((sv & ~LB_MASK) == 0u) continue;
      excl += sv & LB_MASK;
      if (sv & LB_INC) break;
      --tt;
    }
    st_release(st, LB_INC | (excl + run));
  }
  s_base[t] = dstart + excl;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    int idx = base + j * 32 + (int)lane;
    if (idx < K) {
      uint32_t d = (key[j] >> shift) & mask;
      uint32_t pos = s_base[d] + s_cnt[warp][d] + rank[j];
      kout[pos] = key[j];
      vout[pos] = val[j];
    }
  }
}

void launch_radix_hist(const uint32_t* keys, int K, SortPlan plan, uint32_t* hist, Sc1* sc,
                       uint32_t vocab, cudaStream_t s) {
  int blocks = (K + RS_TILE - 1) / RS_TILE;
  if (blocks < 1) blocks = 1;
  k_radix_hist<<<blocks, RS_THREADS, 0, s>>>(keys, K, plan.passes, plan.bits, hist, sc, vocab);
}

void launch_radix_pass(int pass, const uint32_t* kin, const int32_t* vin, uint32_t* kout,
                       int32_t* vout, int K, SortPlan plan, const uint32_t* hist, uint32_t* lb,
                       Sc1* sc, cudaStream_t s) {
  int tiles = (K + RS_TILE - 1) / RS_TILE;
  k_radix_pass<<<tiles, RS_THREADS, 0, s>>>(kin, vin, kout, vout, K, pass * plan.bits, plan.bits,
                                            hist + pass * 256, lb + (size_t)pass * tiles * 256,
                                            &sc->tile_ctr[pass]);
}

// ------------------------------------------------------------ S1 segments
// Run-length flags over the sorted ids.  Thread t of tile T owns sorted
// positions T*4096 + t*16 .. +15 (blocked).  u(i) = number of run heads at
// positions <= i, minus one.
__global__ void __launch_bounds__(RS_THREADS) k_segments(
    const uint32_t* __restrict__ sk, const int32_t* __restrict__ sv, int K, uint32_t vocab,
    uint32_t* __restrict__ luniq, int32_t* __restrict__ lstart, int32_t* __restrict__ segidx,
    int32_t* __restrict__ inverse, uint32_t* __restrict__ lbits, Sc1* __restrict__ sc,
    uint32_t* __restrict__ lb, int64_t* __restrict__ nu_out) {
  __shared__ uint32_t s_scan[32];
  __shared__ uint32_t s_tile, s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(&sc->tile_ctr[RS_MAX_PASSES], 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int i0 = (int)tile * SEG_TILE + (int)threadIdx.x * RS_ITEMS;
  uint32_t key[RS_ITEMS];
  uint32_t heads = 0;  // bit j: item j starts a run
  uint32_t prev = (i0 > 0 && i0 <= K) ? sk[i0 - 1] : 0u;
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    int i = i0 + j;
    key[j] = i < K ? sk[i] : 0u;
    bool h = i < K && (i == 0 || key[j] != prev);
    heads |= (uint32_t)h << j;
    prev = key[j];
  }
  uint32_t tot;
  uint32_t excl_t = block_excl_scan(__popc(heads), s_scan, &tot);
  if (threadIdx.x == 0) s_excl = lookback_one(lb, tile, tot);
  __syncthreads();
  uint32_t u_run = s_excl + excl_t;  // heads strictly before my first item
  bool bad = false;
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    int i = i0 + j;
    if (i < K) {
      if ((heads >> j) & 1u) {
        luniq[u_run] = key[j];
        lstart[u_run] = i;
        if (key[j] < vocab)
          atomicOr(lbits + (key[j] >> 5), 1u << (key[j] & 31u));
        else
          bad = true;
        ++u_run;
      }
      segidx[i] = (int32_t)u_run - 1;
      inverse[sv[i]] = (int32_t)u_run - 1;
      if (i == K - 1) {
        sc->u_local = u_run;
        lstart[u_run] = K;
        if (nu_out) *nu_out = u_run;
      }
    }
  }
  if (bad) atomicOr(&sc->err, 1u);
}

void launch_segments(const uint32_t* sk, const int32_t* sv, int K, uint32_t vocab,
                     uint32_t* luniq, int32_t* lstart, int32_t* segidx, int32_t* inverse,
                     uint32_t* lbits, Sc1* sc, uint32_t* lb, int64_t* nu_out, cudaStream_t s) {
  int tiles = (K + SEG_TILE - 1) / SEG_TILE;
  k_segments<<<tiles, RS_THREADS, 0, s>>>(sk, sv, K, vocab, luniq, lstart, segidx, inverse, lbits,
                                          sc, lb, nu_out);
}

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

// --------------------------------------------------------------------- S3

__global__ void k_gbits(const uint32_t* __restrict__ I, int64_t n, uint32_t vocab,
                        uint32_t* __restrict__ gbits, Sc3* __restrict__ sc) {
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    uint32_t id = I[q];
    if (id >= vocab) {
      bad = true;
      continue;
    }
    uint32_t* w = gbits + (id >> 5);
    uint32_t b = 1u << (id & 31u);
    if (!(__ldcg(w) & b)) atomicOr(w, b);
  }
  if (__any_sync(FULL, bad) && lane_id() == 0) atomicOr(&sc->err, 1u);
}

void launch_gbits(const uint32_t* I, int64_t n, uint32_t vocab, uint32_t* gbits, Sc3* sc,
                  cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  k_gbits<<<(int)blocks, 256, 0, s>>>(I, n, vocab, gbits, sc);
}

// Popcount scan of the presence bitmap: thread t of tile T owns words
// T*1024 + 4t .. 4t+3.  wrank[w] = number of set bits in words < w.
__global__ void __launch_bounds__(GS_THREADS) k_gscan(const uint32_t* __restrict__ gbits,
                                                      int64_t W, uint32_t* __restrict__ wrank,
                                                      uint32_t* __restrict__ ihat,
                                                      Sc3* __restrict__ sc,
                                                      uint32_t* __restrict__ lb) {
  __shared__ uint32_t s_scan[32];
  __shared__ uint32_t s_tile, s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(&sc->tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t w0 = (int64_t)tile * GS_TILE_WORDS + 4 * (int64_t)threadIdx.x;
  uint32_t wd[4];
  if (w0 + 3 < W) {
    uint4 v = __ldcg(reinterpret_cast<const uint4*>(gbits + w0));
    wd[0] = v.x; wd[1] = v.y; wd[2] = v.z; wd[3] = v.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) wd[j] = (w0 + j < W) ? __ldcg(gbits + w0 + j) : 0u;
  }
  uint32_t c = __popc(wd[0]) + __popc(wd[1]) + __popc(wd[2]) + __popc(wd[3]);
  uint32_t tot;
  uint32_t excl_t = block_excl_scan(c, s_scan, &tot);
  if (threadIdx.x == 0) s_excl = lookback_one(lb, tile, tot);
  __syncthreads();
  uint32_t r = s_excl + excl_t;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int64_t w = w0 + j;
    if (w < W) {
      wrank[w] = r;
      uint32_t bits = wd[j];
      while (bits) {
        int b = __ffs(bits) - 1;
        ihat[r++] = (uint32_t)(w * 32 + b);
        bits &= bits - 1;
      }
    }
  }
  const int64_t ntiles = (W + GS_TILE_WORDS - 1) / GS_TILE_WORDS;
  if ((int64_t)tile == ntiles - 1 && threadIdx.x == GS_THREADS - 1) sc->u_global = s_excl + tot;
}

void launch_gscan(const uint32_t* gbits, int64_t W, uint32_t* wrank, uint32_t* ihat, Sc3* sc,
                  uint32_t* lb, cudaStream_t s) {
  int64_t tiles = (W + GS_TILE_WORDS - 1) / GS_TILE_WORDS;
  k_gscan<<<(unsigned)tiles, GS_THREADS, 0, s>>>(gbits, W, wrank, ihat, sc, lb);
}

__global__ void k_l2g(const uint32_t* __restrict__ luniq, const Sc1* __restrict__ sc1, int K,
                      uint32_t vocab, const uint32_t* __restrict__ gbits,
                      const uint32_t* __restrict__ wrank, int32_t* __restrict__ l2g) {
  const int U = (int)sc1->u_local;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < U; u += gridDim.x * blockDim.x) {
    uint32_t w = luniq[u];
    int32_t slot = -1;
    if (w < vocab) {
      uint32_t below = __ldcg(gbits + (w >> 5)) & ((1u << (w & 31u)) - 1u);
      slot = (int32_t)(__ldcg(wrank + (w >> 5)) + __popc(below));
    }
    l2g[u] = slot;
  }
  (void)K;
}

void launch_l2g(const uint32_t* luniq, const Sc1* sc1, int K, uint32_t vocab,
                const uint32_t* gbits, const uint32_t* wrank, int32_t* l2g, cudaStream_t s) {
  int blocks = (K + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  k_l2g<<<blocks, 256, 0, s>>>(luniq, sc1, K, vocab, gbits, wrank, l2g);
}

}  // namespace lms
