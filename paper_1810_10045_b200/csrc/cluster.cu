// cluster.cu -- S1 (local unique, step 1) inside ONE thread-block
// cluster for K <= 16 x 4096 tokens.
//
// The whole sort lives in distributed shared memory: CTA c of the cluster
// owns sorted positions [4096c, 4096c + 4096).  Each LSD pass (<= 10-bit
// digits) ranks the CTA's tile with warp multisplit (__match_any_sync),
// publishes per-digit tile totals in its own shared memory, and after a
// cluster barrier every CTA reads the other CTAs' totals over DSMEM to form its
// bases and scatters its keys straight into the destination CTAs' shared
// buffers.  No global round trips and no grid-wide barriers inside the sort:
// cluster barriers cost a fraction of a grid sync.  The run flags / J^ /
// inverse epilogue is the same as the cooperative kernel's.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace lms {

namespace {
__device__ __forceinline__ void cstamp(unsigned long long* tr, int i) {
  if (tr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[i] = t;
  }
}
constexpr int CT = CL_THREADS;
constexpr int NW = CL_THREADS / 32;
}  // namespace

// IT keys per thread: tile = 512 * IT keys per CTA (IT = 4 spreads K <= 32K
// over up to 16 SMs; the ranking is match_any-throughput-bound per SM).
template <int IT>
__global__ void __launch_bounds__(CL_THREADS, 1) k_s1_cluster(S1Args a) {
  constexpr int CL_TILE = CL_THREADS * IT;
  extern __shared__ uint32_t sm[];
  __shared__ uint32_t s_scan[32];
  // programmatic dependent launch: the next kernel on the stream (S4) may be
  // scheduled now; it waits in griddepcontrol.wait until this grid completes
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ uint32_t s_heads, s_rtot, s_roff;
  cg::cluster_group cl = cg::this_cluster();
  const int cr = (int)cl.block_rank();
  const int C = (int)cl.num_blocks();
  const int ndig = 1 << a.bits;
  // (key, val) pairs, ping-pong: one 8-byte DSMEM store per element
  uint2* kv[2] = {reinterpret_cast<uint2*>(sm), reinterpret_cast<uint2*>(sm + 2 * CL_MAX_TILE)};
  uint32_t* s_cnt = sm + 4 * CL_MAX_TILE;  // [NW][ndig]
  uint32_t* s_tot = s_cnt + NW * ndig;  // [ndig] this tile's digit totals
  uint32_t* s_base = s_tot + ndig;      // [ndig]  written remotely by the digit owners
  uint32_t* s_tmp = s_base + ndig;      // [ndig]  owner-side scratch (C x range)
  uint32_t* s_dex = s_tmp + ndig + 32;  // [ndig]  (nr * C <= ndig + C)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = a.K;
  const int t0 = cr * CL_TILE;  // first global sorted position of this CTA

  cstamp(a.trace, 0);
  // zero the local presence bitmap (ordered before the epilogue by cluster barriers)
  for (int64_t w = (int64_t)cr * CT + tid; w < a.W; w += (int64_t)C * CT) a.lbits[w] = 0u;
  if (cr == 0 && tid == 0) {
    a.sc->err = 0u;
    a.sc->u_local = 0;
    a.sc->fixcount = 0u;
    if (a.sc3) {
      a.sc3->err = 0u;
      a.sc3->u_global = 0;
    }
  }
  bool bad = false;
  int cur = 0;
  for (int p = 0; p < a.passes; ++p) {
    const int shift = p * a.bits;
    const uint32_t mask = (uint32_t)(ndig - 1);
    for (int i = tid; i < NW * ndig; i += CT) s_cnt[i] = 0;
    uint32_t key[IT], rank[IT], dig[IT];
    int32_t val[IT];
    const int lb = warp * (32 * IT);  // local base of this warp (striped layout)
#pragma unroll
    for (int j = 0; j < IT; ++j) {
      const int li = lb + j * 32 + lane;
      const int gi = t0 + li;
      if (gi < K) {
        if (p == 0) {
          key[j] = __ldcs(a.ids + gi);
          val[j] = gi;
          bad |= key[j] >= a.vocab;
        } else {
          const uint2 e = kv[cur][li];
          key[j] = e.x;
          val[j] = (int32_t)e.y;
        }
      } else {
        key[j] = 0;
        val[j] = -1;
      }
    }
    __syncthreads();
    uint32_t* wc = s_cnt + warp * ndig;
#pragma unroll
    for (int j = 0; j < IT; ++j) {
      const int gi = t0 + lb + j * 32 + lane;
      const uint32_t d = gi < K ? ((key[j] >> shift) & mask) : 0xffffffffu;
      dig[j] = d;
      const unsigned m = __match_any_sync(FULL, d);
      const uint32_t before = d != 0xffffffffu ? wc[d] : 0u;
      rank[j] = before + __popc(m & lanemask_lt());
      __syncwarp();
      if (d != 0xffffffffu && lane == (__ffs(m) - 1)) wc[d] = before + __popc(m);
      __syncwarp();
    }
    __syncthreads();
    for (int d = tid; d < ndig; d += CT) {
      uint32_t run = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const uint32_t c = s_cnt[w * ndig + d];
        s_cnt[w * ndig + d] = run;
        run += c;
      }
      s_tot[d] = run;
    }
    cstamp(a.trace, 1 + 4 * p);
    cl.sync();  // every CTA's digit totals are published
    cstamp(a.trace, 2 + 4 * p);
    {
      // CTA cr owns digits [r0, r1): it reads that range from every CTA once,
      // forms the per-CTA exclusive prefixes and the digit totals, and after
      // the range offsets are known writes every CTA's bases remotely.
      const int r0 = (int)((int64_t)ndig * cr / C), r1 = (int)((int64_t)ndig * (cr + 1) / C);
      const int nr = r1 - r0;
      for (int i = tid; i < nr * C; i += CT) {
        const int c = i / nr, dl = i % nr;
        s_tmp[c * nr + dl] = cl.map_shared_rank(s_tot, c)[r0 + dl];
      }
      __syncthreads();
      // each thread owns dpt consecutive digits of the range (nr <= 1024)
      const int dpt = (nr + CT - 1) / CT;
      const int dl0 = tid * dpt;
      uint32_t dt[2] = {0u, 0u}, mysum = 0;
      for (int k = 0; k < dpt; ++k) {
        const int dl = dl0 + k;
        if (dl < nr) {
          uint32_t run = 0;
          for (int c = 0; c < C; ++c) {
            const uint32_t v = s_tmp[c * nr + dl];
            s_tmp[c * nr + dl] = run;  // exclusive prefix over CTAs
            run += v;
          }
          dt[k] = run;
          mysum += run;
        }
      }
      uint32_t rtot;
      uint32_t dex = block_excl_scan(mysum, s_scan, &rtot);
      for (int k = 0; k < dpt; ++k) {
        const int dl = dl0 + k;
        if (dl < nr) {
          s_dex[dl] = dex;  // digit start within the range
          dex += dt[k];
        }
      }
      if (tid == 0) s_rtot = rtot;
      cl.sync();  // range totals published
      if (tid < 32) {
        uint32_t v = (tid < cr) ? *cl.map_shared_rank(&s_rtot, tid) : 0u;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if (tid == 0) s_roff = v;
      }
      __syncthreads();
      const uint32_t roff = s_roff;
      for (int i = tid; i < nr * C; i += CT) {
        const int c = i / nr, dl = i % nr;
        cl.map_shared_rank(s_base, c)[r0 + dl] = roff + s_dex[dl] + s_tmp[c * nr + dl];
      }
    }
    cl.sync();  // every CTA's bases are complete
    cstamp(a.trace, 3 + 4 * p);
    // scatter into the destination CTAs' shared buffers
    const int nxt = cur ^ 1;
#pragma unroll
    for (int j = 0; j < IT; ++j) {
      const uint32_t d = dig[j];
      if (d != 0xffffffffu) {
        const uint32_t pos = s_base[d] + s_cnt[warp * ndig + d] + rank[j];
        const int dst = (int)(pos / CL_TILE), off = (int)(pos % CL_TILE);
        cl.map_shared_rank(kv[nxt], dst)[off] = make_uint2(key[j], (uint32_t)val[j]);
      }
    }
    cl.sync();  // all keys landed; totals may be overwritten next pass
    cstamp(a.trace, 4 + 4 * p);
    cur = nxt;
  }
  if (bad) {
    atomicOr(&a.sc->err, 1u);
    if (a.sc3) atomicOr(&a.sc3->err, 1u);
  }

  // ---- run flags over this CTA's sorted slice (blocked: 8 per thread)
  const uint2* skv = kv[cur];
  const int li0 = tid * IT;
  uint32_t heads = 0;
  uint32_t prev = 0;
  if (li0 > 0)
    prev = skv[li0 - 1].x;
  else if (cr > 0)
    prev = cl.map_shared_rank(skv, cr - 1)[CL_TILE - 1].x;
  const uint32_t prev_first = prev;  // key before this thread's slice (word heads)
  uint32_t sk[IT];
  int32_t sv[IT];
#pragma unroll
  for (int j = 0; j < IT; ++j) {
    const uint2 e = skv[li0 + j];
    sk[j] = e.x;
    sv[j] = (int32_t)e.y;
    const int gi = t0 + li0 + j;
    const bool h = gi < K && (gi == 0 || sk[j] != prev);
    heads |= (uint32_t)h << j;
    prev = sk[j];
  }
  uint32_t tile_heads;
  const uint32_t excl_t = block_excl_scan(__popc(heads), s_scan, &tile_heads);
  if (tid == 0) s_heads = tile_heads;
  cstamp(a.trace, 20);
  cl.sync();  // head counts published
  cstamp(a.trace, 21);
  uint32_t tile_excl = 0;
  for (int c = 0; c < cr; ++c) tile_excl += *cl.map_shared_rank(&s_heads, c);
  uint32_t u_run = tile_excl + excl_t;
  bool bad2 = false;
#pragma unroll
  for (int j = 0; j < IT; ++j) {
    const int li = li0 + j;
    const int gi = t0 + li;
    if (gi < K) {
      const uint32_t key = sk[j];
      const int32_t pos = sv[j];
      a.va[gi] = pos;  // the stable permutation (sorted position -> token)
      if ((heads >> j) & 1u) {
        a.luniq[u_run] = key;
        a.lstart[u_run] = gi;
        if (a.ihat) {
          a.ihat[u_run] = key;
          a.l2g[u_run] = (int32_t)u_run;
        }
        if (key < a.vocab) {
          atomicOr(a.lbits + (key >> 5), 1u << (key & 31u));
          // first present id of its 32-id word: the word's local base index
          const uint32_t pkey = j == 0 ? prev_first : sk[j > 0 ? j - 1 : 0];
          if (a.lrank && (gi == 0 || (pkey >> 5) != (key >> 5))) a.lrank[key >> 5] = u_run;
        } else {
          bad2 = true;
        }
        ++u_run;
      }
      a.segidx[gi] = (int32_t)u_run - 1;
      a.inverse[pos] = (int32_t)u_run - 1;
      if (gi == K - 1) {
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
  cstamp(a.trace, 22);
  cl.sync();  // no CTA leaves while another may still read its shared memory
  if (a.trace && threadIdx.x == 0) {  // latest exit over all CTAs
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(a.trace + 62, t);
  }
}

SortPlan make_cluster_plan(uint64_t vocab) {
  int bits = 1;
  while (bits < 32 && (1ull << bits) < vocab) ++bits;
  SortPlan p;
  p.passes = (bits + CL_MAX_BITS - 1) / CL_MAX_BITS;
  p.bits = (bits + p.passes - 1) / p.passes;
  return p;
}

size_t cluster_smem_bytes(int bits) {
  return (size_t)(4 * CL_MAX_TILE + (NW + 4) * (1 << bits) + 32) * 4;
}

// keys per thread: the fewest that fit K into one cluster of <= CL_MAX_CTAS CTAs
// (K just above 32K -- e.g. the 32768 + 1024 ids of the seeded output
// exchange -- keeps 16 CTAs instead of dropping to 9 CTAs x 8 keys)
static int cluster_items(int K) {
  for (int it : {4, 5, 6})
    if (K <= CL_MAX_CTAS * CL_THREADS * it) return it;
  return 8;
}

bool cluster_s1_ok(int K) {
  static int ok = -1;
  if (ok < 0) {
    ok = 1;
    for (const void* f : {(const void*)k_s1_cluster<4>, (const void*)k_s1_cluster<5>,
                          (const void*)k_s1_cluster<6>, (const void*)k_s1_cluster<8>}) {
      ok &= cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                cudaSuccess &&
            cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)cluster_smem_bytes(CL_MAX_BITS)) == cudaSuccess;
      max_carveout(f);
    }
    if (!ok) cudaGetLastError();
  }
  return ok && K >= 1 && K <= CL_MAX_CTAS * CL_MAX_TILE;
}

cudaError_t launch_s1_cluster(const S1Args& a, cudaStream_t s) {
  const int it = cluster_items(a.K);
  const int tile = CL_THREADS * it;
  const int C = (a.K + tile - 1) / tile;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(CL_THREADS);
  cfg.dynamicSmemBytes = cluster_smem_bytes(a.bits);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  switch (it) {
    case 4: return cudaLaunchKernelEx(&cfg, k_s1_cluster<4>, a);
    case 5: return cudaLaunchKernelEx(&cfg, k_s1_cluster<5>, a);
    case 6: return cudaLaunchKernelEx(&cfg, k_s1_cluster<6>, a);
    default: return cudaLaunchKernelEx(&cfg, k_s1_cluster<8>, a);
  }
}

}  // namespace lms
