// coop.cu -- S3, the global unique + remap of step 4, as ONE
// launch: a normal launch sized to co-residency, phases separated by an
// in-kernel grid barrier.  (S1 is in group.cu.)
//
// The step touches at most a few MB (ids, bitmaps), so it is bound by
// latency, not bandwidth: a chain of dependent launches or a serial
// decoupled look-back costs more than the data movement.
//
// S3: warp-aggregated test-then-set of a |V|-bit presence bitmap over the
//     gathered ids I (hot Zipf words cost one load per warp, not one atomic per
//     token) -- or, with the symmetric window, the OR of the G ranks' local
//     bitmaps read over NVLink -- then a popcount scan over the bitmap that
//     emits I^ in ascending order and the per-word rank table, U_g, and the
//     J^ -> I^ map l2g (each CTA maps the local words of its own word range,
//     found through S1's per-word local prefix lrank).  Peer mode: handshake
//     + 1 grid barrier; gathered ids: 3.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace lms {

namespace {

constexpr int CT = CO_THREADS;

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

}  // namespace

// --------------------------------------------------------------------- S3

__global__ void __launch_bounds__(CO_THREADS, 1) k_s3(S3Args a) {
  __shared__ uint32_t s_scan[32];
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t gtid = (int64_t)blockIdx.x * CT + tid;
  const int64_t gthreads = (int64_t)gridDim.x * CT;

  stamp(a.trace, 32);
  if (a.peer_mode == 2) {
    // emulation: every rank's S1 completed before this launch
    if (gtid == 0) {
      uint32_t err = 0u;
      for (int j = 0; j < a.world; ++j) err |= __ldcg(&a.peer_sc1[j]->err) & 1u;
      a.sc->err = err;
      a.sc->u_global = 0;
    }
    grid_barrier(a.bar);
  } else if (a.peer_mode) {
    // handshake: this rank's S1 (the previous kernel on this stream) is
    // complete; tell every peer, then wait until every peer has said so
    // (flag = 2 * epoch + this rank's id-error bit: every rank learns every
    // rank's error, so all of them report it and none enters a collective alone)
    if (gtid == 0) {
      const uint32_t e = *a.epoch + 1u;
      *a.epoch = e;
      const uint32_t f = 2u * e + (__ldcg(&a.sc1->err) & 1u);
      // one sys fence, then relaxed stores (the release pattern): a release
      // store per peer costs a fence each, 2-5 us apiece while S4 saturates
      // HBM beside this kernel
      __threadfence_system();
      stamp(a.trace, 42);
      for (int j = 0; j < a.world; ++j)
        st_relaxed_sys(reinterpret_cast<uint32_t*>(a.peer_base[j] + a.flags_off) + a.rank, f);
      stamp(a.trace, 43);
      const uint32_t* mine = reinterpret_cast<const uint32_t*>(a.peer_base[a.rank] + a.flags_off);
      uint32_t err = 0u;
      for (int j = 0; j < a.world; ++j) {
        uint32_t v;
        while ((int32_t)((v = ld_relaxed_sys(mine + j)) - 2u * e) < 0) __nanosleep(64);
        err |= v & 1u;
      }
      __threadfence_system();  // acquire pattern: the peers' bitmaps are read after this
      a.sc->err = err;
      a.sc->u_global = 0;
    }
    stamp(a.trace, 40);
    grid_barrier(a.bar);
    stamp(a.trace, 33);
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

  // phase B: popcounts of this CTA's word range (one word per thread per
  // round); in peer mode the range's words are formed here first (phase A':
  // the OR of the G local bitmaps read over NVLink), so no barrier between
  const int64_t per = (a.W + gridDim.x - 1) / gridDim.x;
  const int64_t w0 = (int64_t)blockIdx.x * per;
  const int64_t w1 = min(a.W, w0 + per);
  uint32_t cnt = 0;
  if (a.peer_mode) {
    for (int64_t w = w0 + tid; w < w1; w += CT) {
      uint32_t g = 0u;
#pragma unroll 8
      for (int j = 0; j < a.world; ++j)
        g |= __ldcv(reinterpret_cast<const uint32_t*>(a.peer_base[j] + a.lbits_off) + w);
      a.gbits[w] = g;
      cnt += __popc(g);
    }
  } else {
    for (int64_t w = w0 + tid; w < w1; w += CT) cnt += __popc(__ldcg(a.gbits + w));
  }
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
  __syncthreads();  // this CTA's wrank words are written

  // phase D: l2g[u] = slot of J^[u] in I^ for the local words of this CTA's
  // word range -- a contiguous block of u, [lrank[w0], lrank[w1]) (S1's
  // per-word local prefix) -- from this CTA's own wrank/gbits: no barrier
  // (the Zipf head puts thousands of local words in the first ranges: 8 per
  // thread per round, loads issued together)
  const int U = (int)a.sc1->u_local;
  if (w0 < w1) {
    const int u0 = (int)__ldcg(a.lrank + w0);
    const int u1 = w1 < a.W ? (int)__ldcg(a.lrank + w1) : U;
    constexpr int DB = 8;
    for (int ub = u0; ub < u1; ub += CT * DB) {
      uint32_t w[DB], bits[DB], base[DB];
#pragma unroll
      for (int q = 0; q < DB; ++q) {
        const int u = ub + q * CT + tid;
        w[q] = u < u1 ? __ldcg(a.luniq + u) : 0u;
      }
#pragma unroll
      for (int q = 0; q < DB; ++q) {
        bits[q] = __ldcg(a.gbits + (w[q] >> 5));
        base[q] = __ldcg(a.wrank + (w[q] >> 5));
      }
#pragma unroll
      for (int q = 0; q < DB; ++q) {
        const int u = ub + q * CT + tid;
        if (u < u1) {
          LMS_CHECK(w[q] < a.vocab && (int64_t)(w[q] >> 5) >= w0 && (int64_t)(w[q] >> 5) < w1);
          a.l2g[u] = (int32_t)(base[q] + __popc(bits[q] & ((1u << (w[q] & 31u)) - 1u)));
        }
      }
    }
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

// ------------------------------------------------- global counts (8(b) view)

struct PeerBases {
  const char* p[8];
};

// gcounts[r] = sum over ranks j holding word I^[r] of rank j's S1 count of it
// (read from rank j's window: presence bit, lrank + popcount -> local index).
__global__ void __launch_bounds__(256) k_gcounts_peer(int32_t* __restrict__ gcounts,
                                                      const uint32_t* __restrict__ ihat,
                                                      const Sc3* __restrict__ sc3, int world,
                                                      PeerBases pb, size_t lbits_off,
                                                      size_t lrank_off, size_t counts_off) {
  const int64_t ug = sc3->u_global;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < ug;
       r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t w = __ldg(ihat + r);
    int32_t c = 0;
    for (int j = 0; j < world; ++j) {
      const uint32_t bits = __ldcv(reinterpret_cast<const uint32_t*>(pb.p[j] + lbits_off) + (w >> 5));
      if ((bits >> (w & 31u)) & 1u) {
        const uint32_t idx = __ldcv(reinterpret_cast<const uint32_t*>(pb.p[j] + lrank_off) + (w >> 5)) +
                             __popc(bits & ((1u << (w & 31u)) - 1u));
        c += __ldcv(reinterpret_cast<const int32_t*>(pb.p[j] + counts_off) + idx);
      }
    }
    gcounts[r] = c;
  }
}

// gcounts[slot(I[q])] += 1 over the gathered ids (zeroed before).
__global__ void __launch_bounds__(256) k_gcounts_ids(int32_t* __restrict__ gcounts,
                                                     const uint32_t* __restrict__ I, int64_t n,
                                                     const uint32_t* __restrict__ gbits,
                                                     const uint32_t* __restrict__ wrank,
                                                     uint32_t vocab) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t id = __ldg(I + q);
    if (id >= vocab) continue;
    const uint32_t bits = __ldcg(gbits + (id >> 5));
    atomicAdd(gcounts + __ldcg(wrank + (id >> 5)) + __popc(bits & ((1u << (id & 31u)) - 1u)), 1);
  }
}

cudaError_t launch_gcounts(int32_t* gcounts, int64_t ucap, const uint32_t* ihat, const Sc3* sc3,
                           const uint32_t* I, int64_t n, const uint32_t* gbits,
                           const uint32_t* wrank, uint32_t vocab, int world,
                           char* const* peer_base, size_t lbits_off, size_t lrank_off,
                           size_t counts_off, int num_sms, cudaStream_t s) {
  if (peer_base) {
    PeerBases pb{};
    for (int j = 0; j < world && j < 8; ++j) pb.p[j] = peer_base[j];
    int64_t blocks = (ucap + 255) / 256;
    if (blocks > (int64_t)num_sms * 4) blocks = (int64_t)num_sms * 4;
    if (blocks < 1) blocks = 1;
    k_gcounts_peer<<<(unsigned)blocks, 256, 0, s>>>(gcounts, ihat, sc3, world, pb, lbits_off,
                                                    lrank_off, counts_off);
    return cudaGetLastError();
  }
  cudaError_t e = cudaMemsetAsync(gcounts, 0, 4 * (size_t)ucap, s);
  if (e != cudaSuccess) return e;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
  if (blocks < 1) blocks = 1;
  k_gcounts_ids<<<(unsigned)blocks, 256, 0, s>>>(gcounts, I, n, gbits, wrank, vocab);
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
  // Highest launch priority: at G > 1 S4 (no grid barrier) becomes ready on
  // the side stream at the same moment (both wait only on S1); S3's CTAs
  // must be dispatched first, or its grid barrier waits for S4's CTAs to
  // retire and make room (measured: +~15 us at 1b G = 2).
  static int prio = 1;
  if (prio > 0) {
    int least = 0, greatest = 0;
    prio = cudaDeviceGetStreamPriorityRange(&least, &greatest) == cudaSuccess ? greatest : 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(CO_THREADS);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributePriority;
  at[0].val.priority = prio;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_s3, a);
}

}  // namespace lms
