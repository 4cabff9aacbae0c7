// lmscale.cu -- host side of the C ABI declared in include/lmscale.h:
// context, workspace, stream/event choreography of S1-S6 and NCCL.
//
// Step choreography of lmscale_sync_embedding_grad (one rank):
//
//   caller stream s  : [zero S3] -> ncclAllGather(J -> I) -> gbits(I) -> gscan -> l2g* -> scatter -> fixup -> ncclAllReduce(M)
//   side stream      :  S1: [zero S1] -> radix hist -> radix passes -> segments --------^ (*waits)
//   copy stream      :                                     D2H {U_g, err} after gscan
//
// The host blocks only on the 16-byte {U_g, err} copy, which lands while the
// scatter kernel (already enqueued) runs; then it enqueues the all-reduce
// with count U_g * D.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/lmscale.h"
#include "common.cuh"
#include "kernels.cuh"

using namespace lms;

namespace {

enum Ev {
  EV_FORK = 0,
  EV_S1_BEGIN,
  EV_S1_END,
  EV_GATHER_END,
  EV_S3_END,
  EV_JOIN,
  EV_SCATTER_END,
  EV_FIXUP_END,
  EV_AR_END,
  EV_UPD_BEGIN,
  EV_UPD_END,
  EV_COUNT
};

// pieces of the dense baseline's all-gather (each scattered on arrival)
constexpr int DENSE_CHUNKS = 4;

// which kernels the last step ran (for lmscale_get_stats' byte accounting)
enum PathKind {
  PATH_NONE = 0,
  PATH_W1_FOLD,    // world 1: S1 + S4 with S6 folded in
  PATH_W1_UPDATE,  // world 1: S1 + S4 + k_update
  PATH_W1_SYNC,    // world 1: S1 + S4 (M returned)
  PATH_NCCL,       // G > 1: S3 + S4 + ncclAllReduce (+ k_update)
  PATH_P2P,        // G > 1: fused S5+S6 over NVLink P2P (present rows)
  PATH_P2P_COMP,   // G > 1: compressed fused S5+S6 (binary16 / bfloat16)
  PATH_NVLS        // G > 1: fused S5+S6 over NVLS multicast
};

}  // namespace

struct lmscale_ctx {
  lmscale_config cfg;
  int num_sms = 0;
  int64_t K = 0, W = 0, NI = 0, ucap = 0, nr_max = 0;
  cudaStream_t s_side = nullptr, s_copy = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_s1 = nullptr, ev_s3 = nullptr, ev_copy = nullptr;
  cudaEvent_t ev_s4 = nullptr;
  cudaEvent_t tev[EV_COUNT] = {};
  bool timing_valid = false, update_timed = false;
  ncclComm_t comm = nullptr;
  // device workspace
  void* base = nullptr;
  size_t ws_bytes = 0;
  uint32_t *luniq, *lbits, *gbits, *wrank, *I, *ihat, *ctot, *ctot1, *wcount, *tick;
  int32_t *perm, *runfirst, *inverse, *lstart, *counts, *l2g, *gcounts;
  bool s1_fold = false;  // the S4 range geometry the last S1 cut (seg_plan's fold)
  float* part = nullptr;       // S4 partial rows of cut runs (2 nr_max x D)
  float* part2 = nullptr;      // S4 group sums of partial rows (2 nr_max x D)
  uint32_t* pcnt = nullptr;    // S4 last-arriver counters
  bool lbits_clean = true;     // the presence bitmap is all zero (S1 may skip clearing it)
  float* M = nullptr;
  bool m_nccl = false;
  void* m_reg = nullptr;
  NvlsState* nvls = nullptr;   // fused S5+S6 available
  size_t lbits_off = 0;        // byte offset of lbits inside the M window
  size_t mhat_off = 0;         // byte offset of the compressed M^ rows inside the M window
  size_t flags_off = 0;        // byte offset of the S3 handshake flags inside the M window
  size_t lrank_off = 0;        // byte offset of lrank (per-word local base index) in the window
  size_t counts_off = 0;       // byte offset of S1's counts in the window
  uint32_t* lrank = nullptr;   // S1: index in J^ of the first present id of each 32-id word
  char* peer_base[8] = {};     // LSA base of every rank's M window
  bool peer_s3 = false;        // S3 ORs the peers' local bitmaps (no ID all-gather)
  uint32_t* s3_epoch = nullptr;
  void* ck_dev = nullptr;      // FLAG_CHECK scratch: (U_g, checksum) x (1 + world)
  float cF = 0.f;              // compression scale (0: off), lmscale_set_compression
  int cbf = 0;                 // codec: 0 binary16, 1 bfloat16 (lmscale_set_codec)
  GridBar* bars = nullptr;     // in-kernel grid barriers: [1] S1, [2] S3
  float* table_ptr = nullptr;  // lmscale_alloc_table
  size_t table_bytes = 0;
  bool table_nccl = false;
  ncclWindow_t table_win = nullptr;  // symmetric window of the table (NVLS direct update)
  char nvls_why[256] = {0};    // why not, when it is not
  Sc1* sc1;
  Sc3* sc3;
  // lazily allocated
  float* grad_all = nullptr;
  cudaEvent_t ev_dense[DENSE_CHUNKS] = {};
  uint32_t* stage_ids = nullptr;
  float* stage_grad = nullptr;
  // pinned host mirror of {Sc3, Sc1}
  Sc3* h_sc3 = nullptr;
  Sc1* h_sc1 = nullptr;
  // call state
  int64_t last_k = -1, last_n = -1;
  bool have_s1 = false, have_s3 = false;
  int64_t last_ug = 0;
  bool m_consumed = false;       // the last step consumed M (S6 folded / fused S5+S6)
  bool gcounts_valid = false;    // gcounts hold the global counts of the last collective sync
  bool have_pending_ug = false;  // last step did not read U_g back to the host
  int fused_last = 0;  // last step used the fused NVLS S5+S6 kernel (2: direct into E windows)
  int last_path = PATH_NONE;
  bool last_path_local = false;  // local-slot M layout (U_i rows written by S4)
  bool last_peer_s3 = false;     // ids exchanged as presence bitmaps
  bool last_table = false;       // the last step updated a table
  cudaStream_t last_stream = nullptr;
  // CUDA graph of lmscale_step (LMSCALE_FLAG_GRAPH)
  bool capturing = false;
  cudaStream_t s_cap = nullptr;
  cudaEvent_t ev_cap = nullptr;
  cudaGraphExec_t gexec = nullptr;
  struct {
    const void *ids, *grad, *table;
    int64_t k;
    float lr;
    int kernels;
    int fused;
    int path;
    float cF;
    int cbf;
    bool clean_in;   // the graph's S1 assumes a zero presence bitmap on entry
    bool clean_out;  // ... and leaves it zero
  } gkey{};
  lmscale_stats stats{};
  int kernels_call = 0;
  int64_t kernels_total = 0;
  char err[512] = {0};
  int tmode = 0;                        // timing mode, see rec()
  unsigned long long* trace = nullptr;  // LMSCALE_PHASE_TRACE diagnostics (64 stamps)
};

namespace {

lmscale_status fail(lmscale_ctx* c, lmscale_status st, const char* fmt, ...) {
  if (c) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(c->err, sizeof(c->err), fmt, ap);
    va_end(ap);
  }
  return st;
}

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(ctx, LMSCALE_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,      \
                  cudaGetErrorString(e_));                                               \
  } while (0)

#define NK(call)                                                                         \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess)                                                               \
      return fail(ctx, LMSCALE_ERR_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call,      \
                  ncclGetErrorString(r_));                                               \
  } while (0)

#define LAUNCHED(n)                                                                      \
  do {                                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess)                                                               \
      return fail(ctx, LMSCALE_ERR_CUDA, "%s:%d launch: %s", __FILE__, __LINE__,         \
                  cudaGetErrorString(e_));                                               \
    ctx->kernels_call += (n);                                                            \
  } while (0)

inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

bool comm_enabled(const lmscale_ctx* c) {
  return c->cfg.world > 1 && !(c->cfg.flags & LMSCALE_FLAG_NO_COMM);
}
bool timing(const lmscale_ctx* c) { return c->tmode != 0; }

// Timing modes (lmscale_set_timing): 0 none, 1 only the two events that
// bracket the S4 kernel, 2 every phase.  Each event is a GPU-side
// serialisation point (~3 us measured), so mode 1 is the one to time steps in.
void rec(lmscale_ctx* c, int ev, cudaStream_t s) {
  if (c->tmode == 0) return;
  if (c->tmode == 1 && ev != EV_S3_END && ev != EV_SCATTER_END) return;
  if (c->tmode == 3 && ev != EV_FIXUP_END && ev != EV_AR_END) return;
  if (c->capturing)  // a timing node inside the CUDA graph
    cudaEventRecordWithFlags(c->tev[ev], s, cudaEventRecordExternal);
  else
    cudaEventRecord(c->tev[ev], s);
}

void begin_call(lmscale_ctx* c) {
  c->kernels_call = 0;
  c->err[0] = 0;
}
void end_call(lmscale_ctx* c) {
  c->kernels_total += c->kernels_call;
  c->stats.kernels_last_call = c->kernels_call;
  c->stats.kernels_total_lo = (int32_t)(c->kernels_total & 0x7fffffff);
}

// S1 on stream s: one launch (counting-sort grouping over the
// vocabulary, group.cu).  world1: I = J, so it also writes I^, l2g and U_g.
// fold: the S4 that follows folds S6 in (world-1 step): S1 cuts the S4
// ranges for that kernel's launch geometry (seg_plan).
lmscale_status run_s1(lmscale_ctx* ctx, const uint32_t* ids, int64_t k, int64_t* nu_out,
                      cudaStream_t s, bool world1 = false, bool fold = false) {
  G1Args a;
  a.ids = ids;
  a.K = (int)k;
  a.vocab = (uint32_t)ctx->cfg.vocab;
  a.wcount = ctx->wcount;
  a.tick = ctx->tick;
  a.lbits = ctx->lbits;
  a.lrank = ctx->lrank;
  a.W = ctx->W;
  a.ctot = ctx->ctot1;
  a.luniq = ctx->luniq;
  a.counts = ctx->counts;
  a.lstart = ctx->lstart;
  a.perm = ctx->perm;
  a.inverse = ctx->inverse;
  a.runfirst = ctx->runfirst;
  a.nr = seg_ranges(k, ctx->cfg.dim, ctx->num_sms, fold, &a.seg_len);
  ctx->s1_fold = fold;
  a.sc = ctx->sc1;
  a.nu_out = nu_out;
  a.zero_bits = ctx->lbits_clean ? 0 : 1;
  a.trace = ctx->trace;
  a.ihat = world1 ? ctx->ihat : nullptr;
  a.l2g = world1 ? ctx->l2g : nullptr;
  a.sc3 = world1 ? ctx->sc3 : nullptr;
  a.bar = ctx->bars + 1;
  CK(launch_group(a, ctx->num_sms, s));
  LAUNCHED(1);
  ctx->lbits_clean = false;
  ctx->last_k = k;
  ctx->have_s1 = true;
  ctx->have_s3 = world1;
  ctx->gcounts_valid = false;
  if (world1) ctx->last_n = k;
  return LMSCALE_OK;
}

// S3 on stream s: one launch (bitmap, scan, I^, U_g,
// and the l2g map of the last S1, which must be complete on `s`).
// emu (lmscale_emulate_step): the world's contexts on this GPU; the peers'
// bitmaps are read from their windows after every rank's S1 (no handshake).
lmscale_status run_s3(lmscale_ctx* ctx, const uint32_t* I, int64_t n, cudaStream_t s,
                      bool peer = false, lmscale_ctx* const* emu = nullptr) {
  S3Args a;
  a.peer_mode = emu ? 2 : peer ? 1 : 0;
  a.world = ctx->cfg.world;
  a.rank = ctx->cfg.rank;
  for (int j = 0; j < 8; ++j) {
    a.peer_base[j] = emu ? (j < a.world ? (char*)emu[j]->M : nullptr) : ctx->peer_base[j];
    a.peer_sc1[j] = emu && j < a.world ? emu[j]->sc1 : nullptr;
  }
  a.lbits_off = ctx->lbits_off;
  a.flags_off = ctx->flags_off;
  a.epoch = ctx->s3_epoch;
  a.I = I;
  a.n = n;
  a.vocab = (uint32_t)ctx->cfg.vocab;
  a.gbits = ctx->gbits;
  a.W = ctx->W;
  a.wrank = ctx->wrank;
  a.ihat = ctx->ihat;
  a.ctot = ctx->ctot;
  a.sc = ctx->sc3;
  a.luniq = ctx->luniq;
  a.lrank = ctx->lrank;
  a.sc1 = ctx->sc1;
  a.l2g = ctx->l2g;
  a.trace = ctx->trace;
  a.bar = ctx->bars + 2;
  CK(launch_s3(a, ctx->num_sms, s));
  LAUNCHED(1);
  ctx->last_n = (peer || emu) ? (int64_t)ctx->cfg.world * ctx->last_k : n;  // I has G*k ids either way
  ctx->have_s3 = true;
  return LMSCALE_OK;
}

void print_trace(lmscale_ctx* ctx, cudaStream_t s) {
  if (!ctx->trace || ctx->capturing) return;
  cudaStreamSynchronize(s);
  unsigned long long t[64];
  cudaMemcpy(t, ctx->trace, sizeof(t), cudaMemcpyDeviceToHost);
  fprintf(stderr, "[lmscale trace] S1:");
  for (int i = 1; i <= 13; ++i)
    if (t[i] && t[i - 1]) fprintf(stderr, " %d:%.2f", i, (t[i] - t[0]) * 1e-3);
  if (t[16] > t[0])
    fprintf(stderr, " | last CTA: PA end %.2f (cta %llu) PC end %.2f (cta %llu) PD end %.2f (cta %llu)",
            (t[16] - t[0]) * 1e-3, t[19], (t[17] - t[0]) * 1e-3, t[20], (t[18] - t[0]) * 1e-3,
            t[21]);
  fprintf(stderr, " | S3:");
  for (int i = 33; i <= 43; ++i)
    if (t[i] && t[32]) fprintf(stderr, " %d:%.2f", i, (t[i] - t[32]) * 1e-3);
  if (t[32] > t[0]) fprintf(stderr, " | S1start->S3start %.2f us", (t[32] - t[0]) * 1e-3);
  if (t[54] && t[58]) {
    const unsigned long long s0 = ~t[54];
    fprintf(stderr,
            " | S4 (from first CTA start): last CTA start %.2f, last prologue end %.2f,"
            " first consumer end %.2f, last consumer end %.2f; S1 stamp0 -> S4 first start %.2f",
            (t[55] - s0) * 1e-3, (t[56] - s0) * 1e-3, ((~t[57]) - s0) * 1e-3, (t[58] - s0) * 1e-3,
            ((long long)s0 - (long long)t[0]) * 1e-3);
  }
  fprintf(stderr, "\n");
}

// S4 (+ the world-1 S6 when apply): one launch (segsum.cu).  Output slots:
// local (slot = u: world 1, or the local-slot layout) or global (l2g, with
// the absent slots zero-filled when fill_absent).
lmscale_status run_s4(lmscale_ctx* ctx, const float* grad, cudaStream_t s,
                      float* table = nullptr, float lr = 0.f, bool fill_absent = true,
                      float m16_F = 0.f, bool apply = false, bool local_slots = false,
                      bool pdl = false) {
  const bool world1 = ctx->cfg.world == 1;
  SegArgs a{};
  a.grad = grad;
  a.perm = ctx->perm;
  a.runfirst = ctx->runfirst;
  a.lstart = ctx->lstart;
  a.word = ctx->ihat;  // world 1: I^ = J^
  a.l2g = (world1 || local_slots) ? nullptr : ctx->l2g;
  a.sc1 = ctx->sc1;
  a.table = table;
  a.lr = lr;
  a.apply = apply ? 1 : 0;
  a.M = ctx->M;
  a.m16 = m16_F > 0.f ? 1 : 0;
  a.cF = m16_F;
  a.cbf = ctx->cbf;
  a.part = ctx->part;
  a.part2 = ctx->part2;
  a.cnt = ctx->pcnt;
  a.cnt2 = ctx->pcnt + 2 * (size_t)ctx->nr_max * ((ctx->cfg.dim + 511) / 512);
  a.lbits = ctx->lbits;
  a.W = ctx->W;
  a.clear_bits = world1 ? 1 : 0;  // nothing reads the bitmap after S1 at world 1
  static const bool no_pdl = getenv("LMSCALE_NO_PDL") != nullptr;
  a.pdl = (pdl && !no_pdl) ? 1 : 0;
  a.K = (int)ctx->last_k;
  a.D = (int)ctx->cfg.dim;
  a.num_sms = ctx->num_sms;
  a.trace = ctx->trace;
  a.vocab = (uint32_t)ctx->cfg.vocab;
  a.mrows = ctx->ucap;
  a.part_rows = 2 * ctx->nr_max;
  a.fold = ctx->s1_fold ? 1 : 0;  // the ranges S1 cut
  CK(launch_seg(a, s));
  LAUNCHED(1);
  if (world1) ctx->lbits_clean = true;
  if (!world1 && !local_slots && fill_absent && !a.m16) {
    CK(launch_zero_absent(ctx->M, (int)ctx->cfg.dim, ctx->ihat, ctx->lbits, ctx->sc3, ctx->sc1,
                          std::min<int64_t>(ctx->last_n, ctx->cfg.vocab), ctx->num_sms, s));
    LAUNCHED(1);
  }
  rec(ctx, EV_SCATTER_END, s);
  return LMSCALE_OK;
}

lmscale_status check_ids_args(lmscale_ctx* ctx, const void* ids, int64_t k) {
  if (!ctx) return LMSCALE_ERR_INVALID_ARG;
  if (!ids) return fail(ctx, LMSCALE_ERR_INVALID_ARG, "ids is NULL");
  if (k < 1 || k > ctx->K)
    return fail(ctx, LMSCALE_ERR_INVALID_ARG, "k=%lld outside [1, max_tokens=%lld]",
                (long long)k, (long long)ctx->K);
  return LMSCALE_OK;
}

float ev_ms(const lmscale_ctx* c, int a, int b) {
  float ms = -1.f;
  if (cudaEventElapsedTime(&ms, c->tev[a], c->tev[b]) != cudaSuccess) return -1.f;
  return ms;
}

}  // namespace

extern "C" {

const char* lmscale_version(void) {
#ifdef LMSCALE_DEVICE_CHECKS
  return "lmscale 0.2 sm_100a +device-checks";
#else
  return "lmscale 0.2 sm_100a";
#endif
}

const char* lmscale_status_string(lmscale_status s) {
  switch (s) {
    case LMSCALE_OK: return "ok";
    case LMSCALE_ERR_INVALID_ARG: return "invalid argument";
    case LMSCALE_ERR_ID_RANGE: return "token id >= vocab";
    case LMSCALE_ERR_CUDA: return "CUDA error";
    case LMSCALE_ERR_NCCL: return "NCCL error";
    case LMSCALE_ERR_OOM: return "out of device memory";
    case LMSCALE_ERR_UNSUPPORTED: return "unsupported on this context";
    case LMSCALE_ERR_CONSISTENCY: return "U_g or I^ differs across ranks";
  }
  return "unknown status";
}

const char* lmscale_last_error(const lmscale_ctx* ctx) { return ctx ? ctx->err : "null context"; }

lmscale_status lmscale_alloc_table(lmscale_ctx* ctx, float** table_out, int64_t* bytes_out) {
  if (!ctx || !table_out) return LMSCALE_ERR_INVALID_ARG;
  if (ctx->table_ptr) return fail(ctx, LMSCALE_ERR_INVALID_ARG, "table already allocated");
  const size_t bytes = 4 * (size_t)ctx->cfg.vocab * ctx->cfg.dim;
  if (ctx->nvls) {
    const size_t al = ((bytes + (1 << 21) - 1) >> 21) << 21;
    void* p = nullptr;
    if (ncclMemAlloc(&p, al) != ncclSuccess)
      return fail(ctx, LMSCALE_ERR_OOM, "ncclMemAlloc(table, %zu)", al);
    ctx->table_ptr = (float*)p;
    ctx->table_nccl = true;
    ctx->table_bytes = al;
    char why[256] = {0};
    ctx->table_win = nvls_register_table(ctx->comm, p, al, why, sizeof(why));
    if (!ctx->table_win) snprintf(ctx->nvls_why, sizeof(ctx->nvls_why), "%s", why);
  } else {
    if (cudaMalloc((void**)&ctx->table_ptr, bytes) != cudaSuccess) {
      cudaGetLastError();
      ctx->table_ptr = nullptr;
      return fail(ctx, LMSCALE_ERR_OOM, "cudaMalloc(table, %zu)", bytes);
    }
    ctx->table_bytes = bytes;
  }
  *table_out = ctx->table_ptr;
  if (bytes_out) *bytes_out = (int64_t)bytes;
  return LMSCALE_OK;
}

lmscale_status lmscale_set_codec(lmscale_ctx* ctx, int32_t codec) {
  if (!ctx) return LMSCALE_ERR_INVALID_ARG;
  if (codec != LMSCALE_CODEC_FP16 && codec != LMSCALE_CODEC_BF16)
    return fail(ctx, LMSCALE_ERR_INVALID_ARG, "unknown codec %d", codec);
  if (ctx->gexec) {  // a captured step carries the old codec
    cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
  }
  ctx->cbf = codec == LMSCALE_CODEC_BF16 ? 1 : 0;
  return LMSCALE_OK;
}

lmscale_status lmscale_set_compression(lmscale_ctx* ctx, float F) {
  if (!ctx) return LMSCALE_ERR_INVALID_ARG;
  if (!(F >= 0.f) || std::isinf(F))
    return fail(ctx, LMSCALE_ERR_INVALID_ARG, "compression scale F=%g must be >= 0 and finite", F);
  if (F > 0.f && comm_enabled(ctx) && !ctx->nvls)
    return fail(ctx, LMSCALE_ERR_UNSUPPORTED, "compression needs the symmetric window: %s",
                ctx->nvls_why);
  if (F > 0.f && ctx->cfg.world > 8)
    return fail(ctx, LMSCALE_ERR_UNSUPPORTED,
                "the compressed exchange addresses at most 8 peers (world %d)", ctx->cfg.world);
  if (F != ctx->cF && ctx->gexec) {  // a captured step carries the old F
    cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
  }
  ctx->cF = F;
  return LMSCALE_OK;
}

static lmscale_status codec_call(lmscale_ctx* ctx, bool down, const void* in, int64_t n, float F,
                                 void* out, void* stream) {
  if (!ctx) return LMSCALE_ERR_INVALID_ARG;
  if (n < 0 || !(F > 0.f) || std::isinf(F))
    return fail(ctx, LMSCALE_ERR_INVALID_ARG, "codec: n=%lld F=%g", (long long)n, F);
  if (n == 0) return LMSCALE_OK;
  if (!in || !out) return fail(ctx, LMSCALE_ERR_INVALID_ARG, "codec: NULL pointer");
  cudaSetDevice(ctx->cfg.device);
  begin_call(ctx);
  CK(launch_codec(down, in, n, F, ctx->cbf, out, ctx->num_sms, S(stream)));
  LAUNCHED(1);
  end_call(ctx);
  return LMSCALE_OK;
}

lmscale_status lmscale_compress(lmscale_ctx* ctx, const float* x, int64_t n, float F, uint16_t* q,
                                void* stream) {
  return codec_call(ctx, true, x, n, F, q, stream);
}

lmscale_status lmscale_decompress(lmscale_ctx* ctx, const uint16_t* q, int64_t n, float F, float* x,
                                  void* stream) {
  return codec_call(ctx, false, q, n, F, x, stream);
}

lmscale_status lmscale_plan_seeds(int32_t world, int32_t policy, double alpha,
                                  uint64_t master_seed, uint64_t* seeds_out,
                                  int32_t* groups_out) {
  if (world < 1 || !seeds_out) return LMSCALE_ERR_INVALID_ARG;
  const int n = plan_seed_groups(world, policy, alpha, master_seed, seeds_out);
  if (n < 1) return LMSCALE_ERR_INVALID_ARG;
  if (groups_out) *groups_out = n;
  return LMSCALE_OK;
}

lmscale_status lmscale_draw_samples(lmscale_ctx* ctx, uint64_t seed, uint64_t step, int64_t n,
                                    uint32_t* out, void* stream) {
  if (!ctx) return LMSCALE_ERR_INVALID_ARG;
  if (!out || n < 1 || n > ctx->cfg.vocab || n > DRAW_MAX_S)
    return fail(ctx, LMSCALE_ERR_INVALID_ARG, "draw_samples: S=%lld (vocab %lld, max %d)",
                (long long)n, (long long)ctx->cfg.vocab, DRAW_MAX_S);
  cudaSetDevice(ctx->cfg.device);
  begin_call(ctx);
  CK(launch_draw_samples(seed, step, (int)n, (uint64_t)ctx->cfg.vocab, out, S(stream)));
  LAUNCHED(1);
  end_call(ctx);
  return LMSCALE_OK;
}

lmscale_status lmscale_lookup(lmscale_ctx* ctx, const uint32_t* ids, int64_t k,
                              const float* table, float* out, void* stream) {
  if (!ctx) return LMSCALE_ERR_INVALID_ARG;
  if (k < 0 || (k > 0 && (!ids || !table || !out)))
    return fail(ctx, LMSCALE_ERR_INVALID_ARG, "lookup: k=%lld or NULL pointer", (long long)k);
  cudaSetDevice(ctx->cfg.device);
  begin_call(ctx);
  CK(launch_lookup(table, (int)ctx->cfg.dim, ids, k, (uint32_t)ctx->cfg.vocab, out,
                   ctx->num_sms, S(stream)));
  if (k > 0) LAUNCHED(1);
  end_call(ctx);
  return LMSCALE_OK;
}

lmscale_status lmscale_set_timing(lmscale_ctx* ctx, int mode) {
  if (!ctx || mode < 0 || mode > 3) return LMSCALE_ERR_INVALID_ARG;
  if (mode != ctx->tmode && ctx->gexec) {  // the captured graph carries the old events
    cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
  }
  ctx->tmode = mode;
  ctx->timing_valid = false;
  return LMSCALE_OK;
}

lmscale_status lmscale_get_nccl_id(uint8_t out_id[128]) {
  if (!out_id) return LMSCALE_ERR_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return LMSCALE_ERR_NCCL;
  static_assert(sizeof(id) == 128, "NCCL unique id is 128 bytes");
  memcpy(out_id, &id, 128);
  return LMSCALE_OK;
}

lmscale_status lmscale_init(const lmscale_config* cfg, const uint8_t* nccl_id,
                            lmscale_ctx** out) {
  if (!out) return LMSCALE_ERR_INVALID_ARG;
  *out = nullptr;
  if (!cfg || cfg->vocab < 1 || cfg->vocab > 0xffffffffll || cfg->max_tokens < 1 ||
      cfg->dim < 1 || cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world ||
      cfg->max_tokens > (1ll << 29) || (int64_t)cfg->world * cfg->max_tokens > (1ll << 30) ||
      cfg->dim > (1ll << 20))
    return LMSCALE_ERR_INVALID_ARG;
  lmscale_ctx* ctx = new (std::nothrow) lmscale_ctx();
  if (!ctx) return LMSCALE_ERR_OOM;
  ctx->cfg = *cfg;
  lmscale_status st = [&]() -> lmscale_status {
    CK(cudaSetDevice(cfg->device));
    CK(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, cfg->device));
    ctx->K = cfg->max_tokens;
    ctx->W = (cfg->vocab + 31) / 32;
    ctx->NI = (int64_t)cfg->world * cfg->max_tokens;
    ctx->ucap = std::min<int64_t>(ctx->NI, cfg->vocab);
    ctx->nr_max = seg_max_ranges(ctx->K, ctx->num_sms);

    const int64_t K = ctx->K, D = cfg->dim;
    // ---- workspace layout (one allocation, 256-byte aligned sub-buffers)
    size_t off = 0;
    auto take = [&](size_t bytes) {
      size_t o = off;
      off = align_up(off + bytes);
      return o;
    };
    size_t o_perm = take(4 * K), o_tick = take(4 * K),
           o_inverse = take(4 * K), o_luniq = take(4 * K), o_lstart = take(4 * (K + 1)),
           o_counts = take(4 * K), o_l2g = take(4 * K), o_wrank = take(4 * ctx->W),
           o_I = take(4 * ctx->NI), o_ihat = take(4 * ctx->ucap),
           o_gcounts = take(4 * ctx->ucap), o_bars = take(sizeof(GridBar) * 8),
           o_wcount = take(4 * 32 * (size_t)ctx->W), o_lrank = take(4 * ctx->W);
    size_t o_sc3 = take(sizeof(Sc3) + sizeof(Sc1)), o_sc1 = o_sc3 + sizeof(Sc3),
           o_ctot = take(4 * 4096), o_ctot1 = take(4 * 2 * (size_t)G1_STRIPES * G1_MAX_GRID),
           o_lbits = take(4 * ctx->W), o_gbits = take(4 * ctx->W), o_epoch = take(64),
           o_ck = take(16 * (size_t)(cfg->world + 1));
    // M lives in its own allocation: with a communicator it comes from
    // ncclMemAlloc and is registered with NCCL (zero-copy NVLS / symmetric use).
    // (+256: room to align the compressed M^ region at byte 2*ucap*D)
    const size_t m_bytes = align_up(4 * (size_t)ctx->ucap * D + 256, 1 << 21);
    size_t m_bytes_used = m_bytes;
    ctx->mhat_off = align_up(2 * (size_t)ctx->ucap * D, 256);
    size_t o_part = take(4 * (size_t)2 * ctx->nr_max * D);
    size_t o_part2 = take(4 * (size_t)2 * ctx->nr_max * D);
    size_t o_pcnt = take(4 * (size_t)3 * ctx->nr_max * ((D + 511) / 512));
    size_t o_runfirst = take(4 * ((size_t)ctx->nr_max + 1));
    ctx->ws_bytes = off;
    if (cudaMalloc(&ctx->base, off) != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, LMSCALE_ERR_OOM, "cudaMalloc(%zu) failed", off);
    }
    char* b = (char*)ctx->base;
    ctx->perm = (int32_t*)(b + o_perm);
    ctx->tick = (uint32_t*)(b + o_tick);
    ctx->inverse = (int32_t*)(b + o_inverse);
    ctx->luniq = (uint32_t*)(b + o_luniq);
    ctx->lstart = (int32_t*)(b + o_lstart);
    ctx->counts = (int32_t*)(b + o_counts);
    ctx->l2g = (int32_t*)(b + o_l2g);
    ctx->wrank = (uint32_t*)(b + o_wrank);
    ctx->I = (uint32_t*)(b + o_I);
    ctx->ihat = (uint32_t*)(b + o_ihat);
    ctx->gcounts = (int32_t*)(b + o_gcounts);
    ctx->bars = (GridBar*)(b + o_bars);
    ctx->wcount = (uint32_t*)(b + o_wcount);
    ctx->lrank = (uint32_t*)(b + o_lrank);  // moves into the window when there is one
    ctx->sc1 = (Sc1*)(b + o_sc1);
    ctx->sc3 = (Sc3*)(b + o_sc3);
    ctx->ctot = (uint32_t*)(b + o_ctot);
    ctx->ctot1 = (uint32_t*)(b + o_ctot1);
    ctx->lbits = (uint32_t*)(b + o_lbits);
    ctx->gbits = (uint32_t*)(b + o_gbits);
    ctx->s3_epoch = (uint32_t*)(b + o_epoch);
    ctx->ck_dev = (void*)(b + o_ck);
    ctx->part = (float*)(b + o_part);
    ctx->pcnt = (uint32_t*)(b + o_pcnt);
    ctx->part2 = (float*)(b + o_part2);
    ctx->runfirst = (int32_t*)(b + o_runfirst);
    CK(cudaMemset(ctx->base, 0, off));
    CK(cudaHostAlloc((void**)&ctx->h_sc3, sizeof(Sc3) + sizeof(Sc1), cudaHostAllocDefault));
    ctx->h_sc1 = (Sc1*)((char*)ctx->h_sc3 + sizeof(Sc3));
    CK(cudaStreamCreateWithFlags(&ctx->s_side, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ctx->s_copy, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_s1, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_s3, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_s4, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_copy, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&ctx->s_cap, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_cap, cudaEventDisableTiming));
    for (int i = 0; i < EV_COUNT; ++i) CK(cudaEventCreate(&ctx->tev[i]));
    ctx->tmode = (cfg->flags & LMSCALE_FLAG_TIMING) ? 2 : 0;
    // M and this rank's local presence bitmap, per-word prefix and counts
    // share one window: the fused kernel reads the peers' bitmaps to load only
    // present rows
    const size_t lb_off = m_bytes;
    const size_t lr_off = align_up(m_bytes + 4 * (size_t)ctx->W, 256);
    const size_t ct_off = align_up(lr_off + 4 * (size_t)ctx->W, 256);
    const size_t fl_off = align_up(ct_off + 4 * (size_t)K, 256);
    const size_t win_bytes = align_up(fl_off + 4 * 64, 1 << 21);
    if (comm_enabled(ctx)) {
      if (!nccl_id) return fail(ctx, LMSCALE_ERR_INVALID_ARG, "world > 1 needs an NCCL id");
      ncclUniqueId id;
      memcpy(&id, nccl_id, sizeof(id));
      NK(ncclCommInitRank(&ctx->comm, cfg->world, id, cfg->rank));
      void* m = nullptr;
      if (ncclMemAlloc(&m, win_bytes) != ncclSuccess)
        return fail(ctx, LMSCALE_ERR_OOM, "ncclMemAlloc(%zu) failed", win_bytes);
      ctx->M = (float*)m;
      ctx->m_nccl = true;
      m_bytes_used = win_bytes;
      // Fused S5+S6 needs a symmetric window (LSA peer pointers, multicast);
      // without it, M is registered for NCCL's zero-copy all-reduce.
      char why[256] = {0};
      if (!getenv("LMSCALE_NO_NVLS"))
        ctx->nvls = nvls_create(ctx->comm, ctx->M, win_bytes, ctx->num_sms, why, sizeof(why));
      else
        snprintf(why, sizeof(why), "LMSCALE_NO_NVLS set");
      if (ctx->nvls) {
        ctx->lbits = (uint32_t*)((char*)m + lb_off);
        ctx->lbits_off = lb_off;
        ctx->flags_off = fl_off;
        ctx->lrank_off = lr_off;
        ctx->lrank = (uint32_t*)((char*)m + lr_off);
        ctx->counts_off = ct_off;
        ctx->counts = (int32_t*)((char*)m + ct_off);
        ctx->peer_s3 = !getenv("LMSCALE_NO_PEER_S3") && cfg->world <= 8 &&
                       nvls_peer_bases(ctx->nvls, cfg->world, (void**)ctx->peer_base);
      } else {
        snprintf(ctx->nvls_why, sizeof(ctx->nvls_why), "%s", why);
        NK(ncclCommRegister(ctx->comm, ctx->M, win_bytes, &ctx->m_reg));
      }
      CK(cudaMemset(m, 0, win_bytes));
    } else if (cfg->world > 1) {
      // NO_COMM at world > 1 (staged calls, lmscale_emulate_step): the same
      // window layout in device memory, so G contexts on one GPU can stand in
      // for each other's windows
      if (cudaMalloc((void**)&ctx->M, win_bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, LMSCALE_ERR_OOM, "cudaMalloc(%zu) failed", win_bytes);
      }
      char* m = (char*)ctx->M;
      ctx->lbits = (uint32_t*)(m + lb_off);
      ctx->lbits_off = lb_off;
      ctx->flags_off = fl_off;
      ctx->lrank_off = lr_off;
      ctx->lrank = (uint32_t*)(m + lr_off);
      ctx->counts_off = ct_off;
      ctx->counts = (int32_t*)(m + ct_off);
      CK(cudaMemset(m, 0, win_bytes));
      m_bytes_used = win_bytes;
    } else {
      if (cudaMalloc((void**)&ctx->M, m_bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, LMSCALE_ERR_OOM, "cudaMalloc(%zu) failed", m_bytes);
      }
      CK(cudaMemset(ctx->M, 0, m_bytes));
    }
    off += m_bytes_used;
    if (getenv("LMSCALE_PHASE_TRACE")) {
      CK(cudaMalloc(&ctx->trace, 64 * sizeof(unsigned long long)));
      CK(cudaMemset(ctx->trace, 0, 64 * sizeof(unsigned long long)));
    }
    ctx->stats.workspace_bytes = (int64_t)off;
    ctx->stats.us_dedup = ctx->stats.us_gather = ctx->stats.us_merge = ctx->stats.us_scatter =
        ctx->stats.us_allreduce = ctx->stats.us_update = ctx->stats.us_total = -1.0;
    return LMSCALE_OK;
  }();
  if (st != LMSCALE_OK) {
    fprintf(stderr, "lmscale_init: %s\n", ctx->err);
    lmscale_destroy(ctx);
    return st;
  }
  *out = ctx;
  return LMSCALE_OK;
}

void lmscale_destroy(lmscale_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->cfg.device);
  cudaDeviceSynchronize();
  if (ctx->table_ptr) {
    if (ctx->table_win) nvls_deregister_table(ctx->comm, ctx->table_win);
    if (ctx->table_nccl)
      ncclMemFree(ctx->table_ptr);
    else
      cudaFree(ctx->table_ptr);
  }
  if (ctx->nvls) nvls_destroy(ctx->comm, ctx->nvls);
  if (ctx->m_reg) ncclCommDeregister(ctx->comm, ctx->m_reg);
  if (ctx->M) {
    if (ctx->m_nccl)
      ncclMemFree(ctx->M);
    else
      cudaFree(ctx->M);
  }
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  for (int i = 0; i < EV_COUNT; ++i)
    if (ctx->tev[i]) cudaEventDestroy(ctx->tev[i]);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_s1) cudaEventDestroy(ctx->ev_s1);
  if (ctx->ev_s3) cudaEventDestroy(ctx->ev_s3);
  if (ctx->ev_s4) cudaEventDestroy(ctx->ev_s4);
  if (ctx->ev_copy) cudaEventDestroy(ctx->ev_copy);
  if (ctx->s_side) cudaStreamDestroy(ctx->s_side);
  if (ctx->s_copy) cudaStreamDestroy(ctx->s_copy);
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  if (ctx->s_cap) cudaStreamDestroy(ctx->s_cap);
  if (ctx->ev_cap) cudaEventDestroy(ctx->ev_cap);
  if (ctx->h_sc3) cudaFreeHost(ctx->h_sc3);
  if (ctx->base) cudaFree(ctx->base);
  if (ctx->trace) cudaFree(ctx->trace);
  if (ctx->grad_all) cudaFree(ctx->grad_all);
  for (int c = 0; c < DENSE_CHUNKS; ++c)
    if (ctx->ev_dense[c]) cudaEventDestroy(ctx->ev_dense[c]);
  if (ctx->stage_ids) cudaFree(ctx->stage_ids);
  if (ctx->stage_grad) cudaFree(ctx->stage_grad);
  delete ctx;
}

// ------------------------------------------------------------- staged calls

lmscale_status lmscale_unique(lmscale_ctx* ctx, const uint32_t* ids, int64_t k,
                              uint32_t* uniq_out, int32_t* counts_out, int32_t* inverse_out,
                              int64_t* num_unique_out, void* stream) {
  lmscale_status st = check_ids_args(ctx, ids, k);
  if (st) return st;
  begin_call(ctx);
  cudaStream_t s = S(stream);
  ctx->last_path = PATH_NONE;
  ctx->m_consumed = false;
  st = run_s1(ctx, ids, k, num_unique_out, s);
  if (st) return st;
  if (uniq_out || counts_out || inverse_out) {
    launch_counts_export(ctx->lstart, ctx->luniq, ctx->inverse, ctx->sc1, (int)k, ctx->counts,
                         uniq_out, counts_out, inverse_out, s);
    LAUNCHED(1);
  }
  end_call(ctx);
  return LMSCALE_OK;
}

lmscale_status lmscale_global_unique(lmscale_ctx* ctx, const uint32_t* gathered, int64_t n,
                                     void* stream) {
  if (!ctx) return LMSCALE_ERR_INVALID_ARG;
  if (!gathered || n < 1 || n > ctx->NI)
    return fail(ctx, LMSCALE_ERR_INVALID_ARG, "gathered/n invalid (n=%lld, cap %lld)",
                (long long)n, (long long)ctx->NI);
  if (!ctx->have_s1) return fail(ctx, LMSCALE_ERR_INVALID_ARG, "call lmscale_unique first");
  begin_call(ctx);
  cudaStream_t s = S(stream);
  lmscale_status st = run_s3(ctx, gathered, n, s);
  if (st) return st;
  end_call(ctx);
  return LMSCALE_OK;
}

lmscale_status lmscale_scatter_expand(lmscale_ctx* ctx, const float* grad, int64_t k,
                                      void* stream) {
  if (!ctx) return LMSCALE_ERR_INVALID_ARG;
  if (!grad) return fail(ctx, LMSCALE_ERR_INVALID_ARG, "grad is NULL");
  if (!ctx->have_s3 || k != ctx->last_k)
    return fail(ctx, LMSCALE_ERR_INVALID_ARG,
                "call lmscale_unique and lmscale_global_unique first (same k)");
  begin_call(ctx);
  lmscale_status st = run_s4(ctx, grad, S(stream));
  if (st) return st;
  end_call(ctx);
  return LMSCALE_OK;
}

lmscale_status lmscale_get_sparse_grad(lmscale_ctx* ctx, lmscale_sparse_grad* out,
                                       void* stream) {
  if (!ctx || !out) return LMSCALE_ERR_INVALID_ARG;
  if (!ctx->have_s3) return fail(ctx, LMSCALE_ERR_INVALID_ARG, "no exchange computed yet");
  CK(cudaStreamSynchronize(S(stream)));
  CK(cudaMemcpy(ctx->h_sc3, ctx->sc3, sizeof(Sc3), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ctx->h_sc1, ctx->sc1, sizeof(Sc1), cudaMemcpyDeviceToHost));
  out->ids = ctx->ihat;
  out->counts = ctx->gcounts_valid ? (ctx->cfg.world == 1 ? ctx->counts : ctx->gcounts) : nullptr;
  out->rows = ctx->m_consumed ? nullptr : ctx->M;  // S6 folded / fused S5+S6 consumed M
  out->num_unique = ctx->h_sc3->u_global;
  ctx->have_pending_ug = false;
  ctx->stats.u_global = ctx->h_sc3->u_global;
  ctx->stats.u_local = ctx->h_sc1->u_local;
  if ((ctx->h_sc3->err | ctx->h_sc1->err) & 1u)
    return fail(ctx, LMSCALE_ERR_ID_RANGE, "a token id >= vocab (%lld)",
                (long long)ctx->cfg.vocab);
  return LMSCALE_OK;
}

lmscale_status lmscale_get_local_maps(lmscale_ctx* ctx, const uint32_t** uniq,
                                      const int32_t** counts, const int32_t** inverse,
                                      const int32_t** l2g, int64_t* num_unique_local,
                                      void* stream) {
  if (!ctx) return LMSCALE_ERR_INVALID_ARG;
  if (!ctx->have_s1) return fail(ctx, LMSCALE_ERR_INVALID_ARG, "no S1 computed yet");
  cudaStream_t s = S(stream);
  CK(cudaStreamSynchronize(s));
  CK(cudaMemcpy(ctx->h_sc1, ctx->sc1, sizeof(Sc1), cudaMemcpyDeviceToHost));
  if (uniq) *uniq = ctx->luniq;
  if (counts) *counts = ctx->counts;
  if (inverse) *inverse = ctx->inverse;
  if (l2g) *l2g = ctx->have_s3 ? ctx->l2g : nullptr;
  if (num_unique_local) *num_unique_local = ctx->h_sc1->u_local;
  return LMSCALE_OK;
}

// ----------------------------------------------------------- collective path

}  // extern "C"

namespace {
// S1-S5 (+ S6 when table != nullptr).  With G == 1 and table != nullptr the
// host never waits: S6 reads U_g on the device.  need_host_ug forces the
// {U_g, err, U_i} readback (always done for G > 1: NCCL's count is a host value).
lmscale_status step_impl(lmscale_ctx* ctx, const uint32_t* ids, const float* grad, int64_t k,
                         float* table, float lr, bool need_host_ug, lmscale_sparse_grad* out,
                         void* stream) {
  lmscale_status st = check_ids_args(ctx, ids, k);
  if (st) return st;
  if (!grad) return fail(ctx, LMSCALE_ERR_INVALID_ARG, "grad is NULL");
  if ((ctx->cfg.flags & LMSCALE_FLAG_NO_COMM) && ctx->cfg.world > 1)
    return fail(ctx, LMSCALE_ERR_UNSUPPORTED, "collective call on a NO_COMM context");
  if (ctx->cF > 0.f && ctx->cfg.world > 1 && !table)
    return fail(ctx, LMSCALE_ERR_UNSUPPORTED,
                "compression is on: the compressed exchange runs in lmscale_step (with a table)");
  begin_call(ctx);
  cudaStream_t s = S(stream);
  const int G = ctx->cfg.world;
  const int64_t D = ctx->cfg.dim;
  ctx->timing_valid = false;
  ctx->update_timed = false;
  rec(ctx, EV_FORK, s);
  if (ctx->trace && !ctx->capturing) cudaMemsetAsync(ctx->trace, 0, 64 * sizeof(unsigned long long), s);
  const uint32_t* I = ids;
  int64_t n = k;
  const bool peer_s3 = G > 1 && ctx->peer_s3;
  // S4 at world 1 with a table: S6 folded in (finished rows go straight into
  // the table; M is not written and not re-read).  LMSCALE_NO_INLINE_S6:
  // separate k_update.
  static const bool no_inline = getenv("LMSCALE_NO_INLINE_S6") != nullptr;
  const bool inline_s6 = G == 1 && table && !no_inline;
  // compressed exchange (R15): S4 writes binary16 rows, present rows only
  const bool comp = G > 1 && ctx->cF > 0.f;
  // the peer-to-peer fused kernels load only present rows: no zero-fill of M
  const bool p2p = G > 1 && table && ctx->nvls &&
                   (comp || (table == ctx->table_ptr && ctx->table_win && nvls_use_p2p(G)));
  // local-slot layout (peer S3, P2P): S4 writes row u of M_g for the u-th
  // local word (no l2g needed), so it runs on the side stream while S3 runs
  // (S4 has no grid barrier).  The fused kernel finds word w's row on rank j
  // as lrank_j[w/32] + popc(bits below w).
  static const bool no_local = getenv("LMSCALE_NO_S4_OVERLAP") != nullptr;
  const bool local_m = peer_s3 && p2p && !no_local;
  const bool overlap = local_m && ctx->tmode == 0;  // timed passes measure S4 alone
  ctx->m_consumed = false;
  ctx->gcounts_valid = false;
  if (peer_s3) {
    // J^-set exchange: no ID all-gather; S3 ORs the G
    // local presence bitmaps over NVLink after S1 (same I^, U_g and l2g).
    rec(ctx, EV_S1_BEGIN, s);
    st = run_s1(ctx, ids, k, nullptr, s);
    if (st) return st;
    rec(ctx, EV_S1_END, s);
    rec(ctx, EV_GATHER_END, s);
    if (overlap) {
      CK(cudaEventRecord(ctx->ev_s1, s));
      CK(cudaStreamWaitEvent(ctx->s_side, ctx->ev_s1, 0));
      st = run_s4(ctx, grad, ctx->s_side, nullptr, lr, false, comp ? ctx->cF : 0.f, false, true);
      if (st) return st;
      CK(cudaEventRecord(ctx->ev_s4, ctx->s_side));
    }
  } else if (G > 1) {
    // S1 on the side stream, concurrent with the S2 ID all-gather.
    CK(cudaEventRecord(ctx->ev_fork, s));
    CK(cudaStreamWaitEvent(ctx->s_side, ctx->ev_fork, 0));
    rec(ctx, EV_S1_BEGIN, ctx->s_side);
    st = run_s1(ctx, ids, k, nullptr, ctx->s_side);
    if (st) return st;
    rec(ctx, EV_S1_END, ctx->s_side);
    CK(cudaEventRecord(ctx->ev_s1, ctx->s_side));
    NK(ncclAllGather(ids, ctx->I, (size_t)k, ncclUint32, ctx->comm, s));
    I = ctx->I;
    n = (int64_t)G * k;
    rec(ctx, EV_GATHER_END, s);
    CK(cudaStreamWaitEvent(s, ctx->ev_s1, 0));
  } else {
    // world 1: I = J, so S3's I^, U_g and l2g come out of S1 (one launch).
    rec(ctx, EV_S1_BEGIN, s);
    st = run_s1(ctx, ids, k, nullptr, s, /*world1=*/true, /*fold=*/inline_s6);
    if (st) return st;
    rec(ctx, EV_S1_END, s);
    rec(ctx, EV_GATHER_END, s);
  }
  rec(ctx, EV_JOIN, s);
  // S3: I^, U_g, l2g; {U_g, err, U_i} to the host on the copy stream.
  if (G > 1) {
    st = peer_s3 ? run_s3(ctx, nullptr, 0, s, true) : run_s3(ctx, I, n, s);
    if (st) return st;
  }
  rec(ctx, EV_S3_END, s);
  if ((ctx->cfg.flags & LMSCALE_FLAG_CHECK) && G > 1 && !ctx->capturing) {
    // debug: every rank must hold the same U_g and I^
    unsigned long long* d = reinterpret_cast<unsigned long long*>(ctx->ck_dev);
    CK(launch_checksum(ctx->ihat, ctx->sc3, d, s));
    LAUNCHED(1);
    NK(ncclAllGather(d, d + 2, 2, ncclUint64, ctx->comm, s));
    std::vector<unsigned long long> h(2 * (size_t)(G + 1));
    CK(cudaMemcpyAsync(h.data(), d, h.size() * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int j = 0; j < G; ++j)
      if (h[2 + 2 * j] != h[0] || h[3 + 2 * j] != h[1]) {
        end_call(ctx);
        return fail(ctx, LMSCALE_ERR_CONSISTENCY,
                    "rank %d: U_g %llu checksum %llx, rank %d: U_g %llu checksum %llx",
                    ctx->cfg.rank, h[0], h[1], j, h[2 + 2 * j], h[3 + 2 * j]);
      }
  }
  // The host reads {U_g, err, U_i} only when it must: for NCCL's element count
  // (G > 1 without the fused NVLS kernel) or when the caller asks for U_g.
  const bool host_reads = need_host_ug || !(table && (G == 1 || ctx->nvls));
  if (host_reads) {
    CK(cudaEventRecord(ctx->ev_s3, s));
    CK(cudaStreamWaitEvent(ctx->s_copy, ctx->ev_s3, 0));
    CK(cudaMemcpyAsync(ctx->h_sc3, ctx->sc3, sizeof(Sc3) + sizeof(Sc1), cudaMemcpyDeviceToHost,
                       ctx->s_copy));
    CK(cudaEventRecord(ctx->ev_copy, ctx->s_copy));
  }
  // global counts of I^ for the borrowed view of lmscale_sync_embedding_grad
  // (world 1: S1's counts are already the global ones)
  const bool want_counts = out && !table;
  if (want_counts && G > 1) {
    CK(launch_gcounts(ctx->gcounts, ctx->ucap, ctx->ihat, ctx->sc3, peer_s3 ? nullptr : I, n,
                      ctx->gbits, ctx->wrank, (uint32_t)ctx->cfg.vocab, G,
                      peer_s3 ? ctx->peer_base : nullptr, ctx->lbits_off, ctx->lrank_off,
                      ctx->counts_off, ctx->num_sms, s));
    LAUNCHED(1);
    ctx->gcounts_valid = true;
  }
  // S4: segmented scatter-add into M; world 1: S6
  // folded in (inline_s6 above).
  if (overlap) {
    CK(cudaStreamWaitEvent(s, ctx->ev_s4, 0));  // S4 ran beside S3
  } else {
    st = run_s4(ctx, grad, s, inline_s6 ? table : nullptr, lr, /*fill_absent=*/G > 1 && !p2p,
                comp ? ctx->cF : 0.f, inline_s6, local_m, /*pdl=*/G == 1);
    if (st) return st;
  }
  rec(ctx, EV_FIXUP_END, s);
  ctx->last_path = G == 1 ? (inline_s6 ? PATH_W1_FOLD : (table ? PATH_W1_UPDATE : PATH_W1_SYNC))
                          : PATH_NCCL;
  ctx->last_path_local = local_m;
  ctx->last_peer_s3 = peer_s3;
  ctx->last_table = table != nullptr;
  ctx->last_stream = s;
  if (G > 1 && table && ctx->nvls) {
    // S5+S6 fused over NVLS: no host round trip, U_g is read on the device.
    launch_nvls_update(ctx->nvls, ctx->ihat, ctx->sc3, table, ctx->M, (int)D, lr,
                       ctx->cfg.rank, G, ctx->trace,
                       table == ctx->table_ptr ? ctx->table_win : nullptr, ctx->lbits_off,
                       comp ? ctx->cF : 0.f, ctx->cbf, ctx->mhat_off, ctx->lrank_off,
                       local_m ? 1 : 0, ctx->ucap, (uint32_t)ctx->cfg.vocab, s);
    LAUNCHED(1);
    rec(ctx, EV_AR_END, s);  // us_allreduce = the fused S5+S6 kernel
    if (ctx->trace && !ctx->capturing) {
      print_trace(ctx, s);
      unsigned long long t[64];
      cudaMemcpy(t, ctx->trace, sizeof(t), cudaMemcpyDeviceToHost);
      fprintf(stderr,
              "[lmscale trace rank %d] S5+S6: barrier1 %.2f  exchange+update %.2f  barrier2 %.2f"
              "  tail %.2f us | setup %.2f presence(CTA0) %.2f | S3 start -> S5+S6 start %.2f us | presence table done (last CTA)"
              " %.2f, exchange done (last CTA) %.2f us after barrier1\n",
              ctx->cfg.rank, (t[49] - t[48]) * 1e-3, (t[50] - t[49]) * 1e-3,
              (t[51] - t[50]) * 1e-3, (t[52] - t[51]) * 1e-3,
              t[44] ? (t[44] - t[48]) * 1e-3 : 0.0, t[45] ? (t[45] - t[44]) * 1e-3 : 0.0,
              (t[48] - t[32]) * 1e-3,
              t[47] ? ((long long)t[47] - (long long)t[49]) * 1e-3 : 0.0,
              t[53] ? ((long long)t[53] - (long long)t[49]) * 1e-3 : 0.0);
    }
    rec(ctx, EV_UPD_BEGIN, s);
    rec(ctx, EV_UPD_END, s);
    ctx->update_timed = timing(ctx);
    ctx->timing_valid = timing(ctx);
    ctx->fused_last = comp ? 3 : (table == ctx->table_ptr && ctx->table_win) ? 2 : 1;
    ctx->last_path = comp ? PATH_P2P_COMP : ctx->fused_last == 2 ? PATH_P2P : PATH_NVLS;
    ctx->m_consumed = true;
    ctx->have_pending_ug = true;
    int64_t ug = -1;
    if (need_host_ug) {
      CK(cudaEventSynchronize(ctx->ev_copy));
      ctx->have_pending_ug = false;
      ug = ctx->h_sc3->u_global;
      ctx->stats.u_global = ug;
      ctx->stats.u_local = ctx->h_sc1->u_local;
      if (ctx->h_sc3->err & 1u) {
        end_call(ctx);
        return fail(ctx, LMSCALE_ERR_ID_RANGE, "a token id >= vocab (%lld)",
                    (long long)ctx->cfg.vocab);
      }
    }
    if (out) {
      out->ids = ctx->ihat;
      out->counts = nullptr;
      out->rows = nullptr;  // M was consumed by the fused update
      out->num_unique = ug;
    }
    end_call(ctx);
    return LMSCALE_OK;
  }
  ctx->fused_last = 0;
  if (G == 1 && table && !need_host_ug) {
    // S6 straight away with the device-side count: no host round trip.
    rec(ctx, EV_AR_END, s);
    rec(ctx, EV_UPD_BEGIN, s);
    if (!inline_s6) {
      launch_update(table, (int)D, ctx->ihat, ctx->M, ctx->ucap, ctx->sc3, lr, ctx->num_sms, s);
      LAUNCHED(1);
    }
    rec(ctx, EV_UPD_END, s);
    ctx->update_timed = timing(ctx);
    ctx->timing_valid = timing(ctx);
    ctx->have_pending_ug = true;
    ctx->m_consumed = inline_s6;
    print_trace(ctx, s);
    if (out) {
      out->ids = ctx->ihat;
      out->counts = nullptr;
      out->rows = inline_s6 ? nullptr : ctx->M;  // folded S6 consumed the rows
      out->num_unique = -1;
    }
    end_call(ctx);
    return LMSCALE_OK;
  }
  // host learns U_g (hidden behind the scatter kernel)
  CK(cudaEventSynchronize(ctx->ev_copy));
  ctx->have_pending_ug = false;
  const int64_t ug = ctx->h_sc3->u_global;
  ctx->last_ug = ug;
  ctx->stats.u_global = ug;
  ctx->stats.u_local = ctx->h_sc1->u_local;
  if (ctx->h_sc3->err & 1u) {
    end_call(ctx);
    return fail(ctx, LMSCALE_ERR_ID_RANGE, "a token id >= vocab (%lld)",
                (long long)ctx->cfg.vocab);
  }
  // S5: all-reduce of M.
  if (G > 1 && ug > 0) NK(ncclAllReduce(ctx->M, ctx->M, (size_t)(ug * D), ncclFloat, ncclSum,
                                        ctx->comm, s));
  rec(ctx, EV_AR_END, s);
  if (table) {
    rec(ctx, EV_UPD_BEGIN, s);
    if (!inline_s6) {
      launch_update(table, (int)D, ctx->ihat, ctx->M, ug, nullptr, lr, ctx->num_sms, s);
      if (ug > 0) LAUNCHED(1);
    }
    rec(ctx, EV_UPD_END, s);
    ctx->update_timed = timing(ctx);
  }
  ctx->m_consumed = inline_s6;
  print_trace(ctx, s);

  if (out) {
    out->ids = ctx->ihat;
    out->counts = want_counts ? (G == 1 ? ctx->counts : ctx->gcounts) : nullptr;
    out->rows = inline_s6 ? nullptr : ctx->M;
    out->num_unique = ug;
  }
  if (want_counts && G == 1) ctx->gcounts_valid = true;
  ctx->timing_valid = timing(ctx);
  end_call(ctx);
  return LMSCALE_OK;
}

}  // namespace

extern "C" {

lmscale_status lmscale_sync_embedding_grad(lmscale_ctx* ctx, const uint32_t* ids,
                                           const float* grad, int64_t k,
                                           lmscale_sparse_grad* out, void* stream) {
  if (ctx && !out) return fail(ctx, LMSCALE_ERR_INVALID_ARG, "out is NULL");
  return step_impl(ctx, ids, grad, k, nullptr, 0.f, true, out, stream);
}

lmscale_status lmscale_emulate_step(lmscale_ctx* const* ctxs, int world,
                                    const uint32_t* const* ids, const float* const* grads,
                                    int64_t k, float* const* tables, float lr, void* stream) {
  if (!ctxs || !ids || !grads || !tables || world < 2 || world > 8) return LMSCALE_ERR_INVALID_ARG;
  for (int r = 0; r < world; ++r) {
    lmscale_ctx* c = ctxs[r];
    if (!c) return LMSCALE_ERR_INVALID_ARG;
    if (c->cfg.world != world || c->cfg.rank != r || !(c->cfg.flags & LMSCALE_FLAG_NO_COMM) ||
        c->cfg.vocab != ctxs[0]->cfg.vocab || c->cfg.dim != ctxs[0]->cfg.dim ||
        c->cfg.device != ctxs[0]->cfg.device || c->K != ctxs[0]->K || c->cF != ctxs[0]->cF ||
        c->cbf != ctxs[0]->cbf)
      return fail(c, LMSCALE_ERR_INVALID_ARG,
                  "emulate_step: context %d must be a NO_COMM context of rank %d of world %d "
                  "with the same vocab, dim, max_tokens, device and compression as context 0",
                  r, r, world);
    if (!grads[r] || !tables[r])
      return fail(c, LMSCALE_ERR_INVALID_ARG, "emulate_step: grad / table of rank %d is NULL", r);
    lmscale_status st0 = check_ids_args(c, ids[r], k);
    if (st0) return st0;
  }
  lmscale_ctx* ctx = ctxs[0];  // errors of the launches are reported on context 0
  cudaStream_t s = S(stream);
  const float cF = ctx->cF;
  const int D = (int)ctx->cfg.dim;
  for (int r = 0; r < world; ++r) {
    begin_call(ctxs[r]);
    ctxs[r]->timing_valid = false;
  }
  lmscale_status st = LMSCALE_OK;
  // S1 on every rank, then S3 (J^-set exchange) and S4 (local-slot layout)
  for (int r = 0; r < world && !st; ++r) st = run_s1(ctxs[r], ids[r], k, nullptr, s);
  for (int r = 0; r < world && !st; ++r) st = run_s3(ctxs[r], nullptr, 0, s, true, ctxs);
  for (int r = 0; r < world && !st; ++r)
    st = run_s4(ctxs[r], grads[r], s, nullptr, lr, false, cF, false, /*local_slots=*/true);
  if (st) return st;
  char* bases[8];
  for (int j = 0; j < world; ++j) bases[j] = (char*)ctxs[j]->M;
  // the global counts of I^ (the sparse-grad view's `counts`), from every
  // rank's S1 counts in its window, as lmscale_sync does at world > 1
  for (int r = 0; r < world; ++r) {
    lmscale_ctx* c = ctxs[r];
    CK(launch_gcounts(c->gcounts, c->ucap, c->ihat, c->sc3, nullptr, 0, c->gbits, c->wrank,
                      (uint32_t)c->cfg.vocab, world, bases, c->lbits_off, c->lrank_off,
                      c->counts_off, c->num_sms, s));
    c->kernels_call += 1;
  }
  // S5+S6: every rank's fused kernel (compressed: every phase 1, then every phase 2)
  for (int ph = 1; ph <= (cF > 0.f ? 2 : 1); ++ph)
    for (int r = 0; r < world; ++r) {
      lmscale_ctx* c = ctxs[r];
      CK(launch_p2p_emulated(bases, tables, world, r, c->ihat, c->sc3, c->M, D, lr, c->lbits_off,
                             c->lrank_off, c->mhat_off, cF, c->cbf, ph, c->ucap,
                             (uint32_t)c->cfg.vocab, c->num_sms, s));
      c->kernels_call += 1;
    }
  for (int r = 0; r < world; ++r) {
    lmscale_ctx* c = ctxs[r];
    c->have_s3 = true;
    c->m_consumed = true;
    c->gcounts_valid = true;
    c->lbits_clean = false;
    end_call(c);
  }
  CK(cudaMemcpyAsync(ctx->h_sc3, ctx->sc3, sizeof(Sc3) + sizeof(Sc1), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (ctx->h_sc3->err & 1u)
    return fail(ctx, LMSCALE_ERR_ID_RANGE, "a token id >= vocab on some rank");
  return LMSCALE_OK;
}

lmscale_status lmscale_step(lmscale_ctx* ctx, const uint32_t* ids, const float* grad, int64_t k,
                            float* table, float lr, int64_t* num_unique_out, void* stream) {
  if (ctx && !table) return fail(ctx, LMSCALE_ERR_INVALID_ARG, "table is NULL");
  // CUDA-graph replay: the step has no host round trip when world == 1, or
  // when world > 1 runs the peer-bitmap S3 and a fused S5+S6 kernel (no NCCL
  // host calls at all), so it is captured once per argument tuple and
  // replayed (one launch instead of 3-4 kernels + events).
  if (ctx && (ctx->cfg.flags & LMSCALE_FLAG_GRAPH) && !(ctx->cfg.flags & LMSCALE_FLAG_CHECK) &&
      !num_unique_out &&
      (ctx->cfg.world == 1 || (ctx->peer_s3 && ctx->nvls))) {
    lmscale_status st0 = check_ids_args(ctx, ids, k);
    if (st0) return st0;
    cudaStream_t s = S(stream);
    const bool hit = ctx->gexec && ctx->gkey.ids == ids && ctx->gkey.grad == grad &&
                     ctx->gkey.table == table && ctx->gkey.k == k && ctx->gkey.lr == lr &&
                     ctx->gkey.cF == ctx->cF && ctx->gkey.cbf == ctx->cbf;
    if (!hit) {
      if (ctx->gexec) {
        cudaGraphExecDestroy(ctx->gexec);
        ctx->gexec = nullptr;
      }
      // capture on the library's own stream (the caller's may be the legacy
      // default stream, which cannot be captured)
      if (ctx->cfg.world == 1 && !ctx->lbits_clean) {
        // world 1 leaves the bitmap clean: capture the S1 that relies on it
        CK(cudaMemsetAsync(ctx->lbits, 0, 4 * (size_t)ctx->W, s));
        ctx->lbits_clean = true;
      }
      const bool clean_in = ctx->lbits_clean;
      CK(cudaStreamBeginCapture(ctx->s_cap, cudaStreamCaptureModeThreadLocal));
      ctx->capturing = true;
      lmscale_sparse_grad sg;
      lmscale_status st = step_impl(ctx, ids, grad, k, table, lr, false, &sg, ctx->s_cap);
      ctx->capturing = false;
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(ctx->s_cap, &g);
      const bool clean_out = ctx->lbits_clean;
      ctx->lbits_clean = clean_in;  // nothing ran yet
      if (st) {
        if (g) cudaGraphDestroy(g);
        return st;
      }
      if (e != cudaSuccess)
        return fail(ctx, LMSCALE_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
      e = cudaGraphInstantiate(&ctx->gexec, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) {
        ctx->gexec = nullptr;
        return fail(ctx, LMSCALE_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
      }
      ctx->gkey.ids = ids;
      ctx->gkey.grad = grad;
      ctx->gkey.table = table;
      ctx->gkey.k = k;
      ctx->gkey.lr = lr;
      ctx->gkey.cF = ctx->cF;
      ctx->gkey.cbf = ctx->cbf;
      ctx->gkey.kernels = ctx->kernels_call;
      ctx->gkey.fused = ctx->fused_last;
      ctx->gkey.path = ctx->last_path;
      ctx->gkey.clean_in = clean_in;
      ctx->gkey.clean_out = clean_out;
      ctx->kernels_total -= ctx->kernels_call;  // captured, not launched yet
    }
    // the graph's S1 skips clearing the presence bitmap when it was captured
    // with a clean one: restore that precondition if a staged call dirtied it
    if (ctx->gkey.clean_in && !ctx->lbits_clean)
      CK(cudaMemsetAsync(ctx->lbits, 0, 4 * (size_t)ctx->W, s));
    begin_call(ctx);
    if (ctx->trace) CK(cudaMemsetAsync(ctx->trace, 0, 64 * sizeof(unsigned long long), s));
    CK(cudaGraphLaunch(ctx->gexec, s));
    print_trace(ctx, s);
    ctx->kernels_call = ctx->gkey.kernels;
    ctx->fused_last = ctx->gkey.fused;
    ctx->last_path = ctx->gkey.path;
    ctx->lbits_clean = ctx->gkey.clean_out;
    ctx->last_stream = s;
    ctx->have_pending_ug = true;
    ctx->m_consumed = ctx->fused_last != 0 || ctx->last_path == PATH_W1_FOLD;
    ctx->gcounts_valid = false;
    ctx->timing_valid = timing(ctx);
    ctx->update_timed = timing(ctx);
    ctx->have_s1 = ctx->have_s3 = true;
    ctx->last_k = k;
    end_call(ctx);
    return LMSCALE_OK;
  }
  lmscale_sparse_grad sg;
  lmscale_status st =
      step_impl(ctx, ids, grad, k, table, lr, num_unique_out != nullptr, &sg, stream);
  if (st == LMSCALE_OK && num_unique_out) *num_unique_out = sg.num_unique;
  return st;
}

lmscale_status lmscale_apply_sparse_update(lmscale_ctx* ctx, float* table,
                                           const lmscale_sparse_grad* sg, float lr,
                                           void* stream) {
  if (!ctx) return LMSCALE_ERR_INVALID_ARG;
  if (!table || !sg || (sg->num_unique > 0 && (!sg->ids || !sg->rows)) || sg->num_unique < 0 ||
      sg->num_unique > ctx->cfg.vocab)
    return fail(ctx, LMSCALE_ERR_INVALID_ARG, "table/sg invalid");
  begin_call(ctx);
  cudaStream_t s = S(stream);
  rec(ctx, EV_UPD_BEGIN, s);
  launch_update(table, (int)ctx->cfg.dim, sg->ids, sg->rows, sg->num_unique, nullptr, lr,
                ctx->num_sms, s);
  if (sg->num_unique > 0) LAUNCHED(1);
  rec(ctx, EV_UPD_END, s);
  ctx->update_timed = timing(ctx);
  end_call(ctx);
  return LMSCALE_OK;
}

lmscale_status lmscale_dense_apply(lmscale_ctx* ctx, const uint32_t* ids, const float* grad,
                                   int64_t n, float* table, float lr, void* stream) {
  if (!ctx) return LMSCALE_ERR_INVALID_ARG;
  if (!ids || !grad || !table || n < 1 || n > ctx->NI)
    return fail(ctx, LMSCALE_ERR_INVALID_ARG, "dense_apply args invalid");
  begin_call(ctx);
  launch_dense(table, (int)ctx->cfg.dim, ids, grad, n, lr, (uint32_t)ctx->cfg.vocab,
               ctx->num_sms, S(stream));
  LAUNCHED(1);
  end_call(ctx);
  return LMSCALE_OK;
}

lmscale_status lmscale_sync_dense_baseline(lmscale_ctx* ctx, const uint32_t* ids,
                                           const float* grad, int64_t k, float* table,
                                           float lr, void* stream) {
  lmscale_status st = check_ids_args(ctx, ids, k);
  if (st) return st;
  if (!grad || !table) return fail(ctx, LMSCALE_ERR_INVALID_ARG, "grad/table is NULL");
  if ((ctx->cfg.flags & LMSCALE_FLAG_NO_COMM) && ctx->cfg.world > 1)
    return fail(ctx, LMSCALE_ERR_UNSUPPORTED, "collective call on a NO_COMM context");
  begin_call(ctx);
  cudaStream_t s = S(stream);
  const int G = ctx->cfg.world;
  const int64_t D = ctx->cfg.dim;
  const uint32_t* I = ids;
  const float* A = grad;
  if (G > 1) {
    if (!ctx->grad_all) {
      if (cudaMalloc(&ctx->grad_all, 4 * (size_t)ctx->NI * D) != cudaSuccess) {
        cudaGetLastError();
        ctx->grad_all = nullptr;
        return fail(ctx, LMSCALE_ERR_OOM, "dense gather buffer (%lld bytes)",
                    (long long)(4 * ctx->NI * D));
      }
      for (int c = 0; c < DENSE_CHUNKS; ++c)
        CK(cudaEventCreateWithFlags(&ctx->ev_dense[c], cudaEventDisableTiming));
    }
    // The Theta(G K D) all-gather in DENSE_CHUNKS pieces on `s`; each piece's
    // atomic scatter runs on the side stream as soon as the piece has arrived,
    // overlapping the gather of the next one.
    const int64_t kc = (k + DENSE_CHUNKS - 1) / DENSE_CHUNKS;
    CK(cudaEventRecord(ctx->ev_fork, s));
    CK(cudaStreamWaitEvent(ctx->s_side, ctx->ev_fork, 0));
    int nlaunch = 0;
    for (int c = 0; c < DENSE_CHUNKS; ++c) {
      const int64_t r0 = c * kc, n = std::min<int64_t>(kc, k - r0);
      if (n <= 0) break;
      uint32_t* Ic = ctx->I + (size_t)G * r0;
      float* Ac = ctx->grad_all + (size_t)G * r0 * D;
      NK(ncclGroupStart());
      NK(ncclAllGather(ids + r0, Ic, (size_t)n, ncclUint32, ctx->comm, s));
      NK(ncclAllGather(grad + r0 * D, Ac, (size_t)(n * D), ncclFloat, ctx->comm, s));
      NK(ncclGroupEnd());
      CK(cudaEventRecord(ctx->ev_dense[c], s));
      CK(cudaStreamWaitEvent(ctx->s_side, ctx->ev_dense[c], 0));
      launch_dense(table, (int)D, Ic, Ac, (int64_t)G * n, lr, (uint32_t)ctx->cfg.vocab,
                   ctx->num_sms, ctx->s_side);
      ++nlaunch;
    }
    CK(cudaEventRecord(ctx->ev_s4, ctx->s_side));
    CK(cudaStreamWaitEvent(s, ctx->ev_s4, 0));
    LAUNCHED(nlaunch);
    end_call(ctx);
    return LMSCALE_OK;
  }
  launch_dense(table, (int)D, I, A, (int64_t)G * k, lr, (uint32_t)ctx->cfg.vocab, ctx->num_sms,
               s);
  LAUNCHED(1);
  end_call(ctx);
  return LMSCALE_OK;
}

lmscale_status lmscale_train_step_host(lmscale_ctx* ctx, const uint32_t* ids_host,
                                       const float* grad_host, int64_t k, float* table, float lr,
                                       uint32_t* ids_out_host, int64_t* num_unique_out,
                                       void* stream) {
  lmscale_status st = check_ids_args(ctx, ids_host, k);
  if (st) return st;
  if (!grad_host || !table) return fail(ctx, LMSCALE_ERR_INVALID_ARG, "grad/table is NULL");
  const int64_t D = ctx->cfg.dim;
  if (!ctx->stage_ids) {
    if (cudaMalloc(&ctx->stage_ids, 4 * (size_t)ctx->K) != cudaSuccess ||
        cudaMalloc(&ctx->stage_grad, 4 * (size_t)ctx->K * D) != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, LMSCALE_ERR_OOM, "host-step staging buffers");
    }
  }
  cudaStream_t s = S(stream);
  CK(cudaMemcpyAsync(ctx->stage_ids, ids_host, 4 * (size_t)k, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(ctx->stage_grad, grad_host, 4 * (size_t)k * D, cudaMemcpyHostToDevice, s));
  lmscale_sparse_grad sg;
  st = step_impl(ctx, ctx->stage_ids, ctx->stage_grad, k, table, lr, true, &sg, stream);
  if (st) return st;
  if (ids_out_host && sg.num_unique > 0)
    CK(cudaMemcpyAsync(ids_out_host, sg.ids, 4 * (size_t)sg.num_unique, cudaMemcpyDeviceToHost,
                       s));
  if (num_unique_out) *num_unique_out = sg.num_unique;
  CK(cudaStreamSynchronize(s));
  return LMSCALE_OK;
}

lmscale_status lmscale_get_stats(const lmscale_ctx* cctx, lmscale_stats* out) {
  if (!cctx || !out) return LMSCALE_ERR_INVALID_ARG;
  lmscale_ctx* ctx = const_cast<lmscale_ctx*>(cctx);
  lmscale_stats& st = ctx->stats;
  st.us_dedup = st.us_gather = st.us_merge = st.us_scatter = st.us_allreduce = st.us_update =
      st.us_total = -1.0;
  if (ctx->timing_valid && ctx->tmode == 1) {
    CK(cudaEventSynchronize(ctx->tev[EV_SCATTER_END]));
    st.us_scatter = 1e3 * ev_ms(ctx, EV_S3_END, EV_SCATTER_END);
  } else if (ctx->timing_valid && ctx->tmode == 3) {
    CK(cudaEventSynchronize(ctx->tev[EV_AR_END]));
    st.us_allreduce = 1e3 * ev_ms(ctx, EV_FIXUP_END, EV_AR_END);
  } else if (ctx->timing_valid && ctx->tmode == 2) {
    CK(cudaEventSynchronize(ctx->tev[EV_AR_END]));
    if (ctx->update_timed) CK(cudaEventSynchronize(ctx->tev[EV_UPD_END]));
    st.us_dedup = 1e3 * ev_ms(ctx, EV_S1_BEGIN, EV_S1_END);
    st.us_gather = 1e3 * ev_ms(ctx, EV_FORK, EV_GATHER_END);
    st.us_merge = 1e3 * ev_ms(ctx, EV_JOIN, EV_S3_END);
    st.us_scatter = 1e3 * ev_ms(ctx, EV_S3_END, EV_SCATTER_END);
    st.us_allreduce = 1e3 * ev_ms(ctx, EV_FIXUP_END, EV_AR_END);
    st.us_update = ctx->update_timed ? 1e3 * ev_ms(ctx, EV_UPD_BEGIN, EV_UPD_END) : -1.0;
    st.us_total = 1e3 * ev_ms(ctx, EV_FORK, ctx->update_timed ? EV_UPD_END : EV_AR_END);
  }
  // byte accounting of the last step (SURVEY 8(d) algorithmic bytes, per rank),
  // for the kernels that actually ran; U_g / U_i read back if the step kept
  // them on the device
  if (ctx->last_path != PATH_NONE) {
    if (ctx->have_pending_ug && !ctx->capturing) {
      CK(cudaStreamSynchronize(ctx->last_stream));
      CK(cudaMemcpy(ctx->h_sc3, ctx->sc3, sizeof(Sc3) + sizeof(Sc1), cudaMemcpyDeviceToHost));
      ctx->have_pending_ug = false;
      st.u_global = ctx->h_sc3->u_global;
      st.u_local = ctx->h_sc1->u_local;
    }
    const int64_t G = ctx->cfg.world, D = ctx->cfg.dim, k = ctx->last_k;
    const int64_t ug = st.u_global, ui = st.u_local;
    const int p = ctx->last_path;
    const int64_t esz = p == PATH_P2P_COMP ? 2 : 4;
    st.bytes_ids_gathered = G == 1 ? 0 : ctx->last_peer_s3 ? 4 * ctx->W * (G - 1) : 4 * (G - 1) * k;
    st.bytes_grad_allreduce = G == 1 ? 0 : esz * ug * D;
    st.bytes_scatter = 4 * k * D + (p == PATH_W1_FOLD ? 8 * ug * D
                                    : ctx->last_path_local ? esz * ui * D : esz * ug * D);
    st.bytes_update =
        (p == PATH_W1_UPDATE || (p == PATH_NCCL && ctx->last_table)) ? 12 * ug * D : 0;
  }
  st.fused_s5_s6 = ctx->fused_last;
  st.nvls_available = ctx->nvls ? 1 : 0;
  *out = st;
  return LMSCALE_OK;
}

}  // extern "C"
