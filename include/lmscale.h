/*
 * lmscale.h -- C ABI of the B200-native uniqueness embedding-gradient
 * exchange (Patwary et al., "Language Modeling at Scale", arXiv 1810.10045,
 * Sec. 3.1).
 *
 * Problem statement: G data-parallel GPUs; GPU g
 * holds K token word-indices J_g (uint32) and their K x D fp32 embedding
 * gradient rows Delta_g; every GPU holds the same |V| x D fp32 embedding table
 * E.  The exchange replaces the Theta(G K D) all-gather of (J, Delta) pairs
 * with
 *   S1  local unique  J -> J^ (+ counts, inverse)                (step 1)
 *   S2  all-gather of J -> I (G K ids)                            (step 3)
 *   S3  global unique I -> I^ (ascending), U_g, J^ -> I^ map     (step 4)
 *   S4  segmented scatter-add Delta -> M_g (U_g x D, zero rows)  (steps 2+5)
 *   S5  all-reduce M_g -> M^                                      (step 6)
 *   S6  duplicate-free row update E[I^[r]] -= lr * M^[r]          (step 7)
 *
 * Conventions (all functions):
 *  - Pointers are DEVICE pointers on the context's device unless a parameter
 *    says "host".  `stream` is a cudaStream_t passed as void* (NULL = the
 *    legacy default stream); every call is stream-ordered on it.
 *  - The caller owns ids / grad / table.  The context owns all scratch, sized
 *    at init from (vocab, max_tokens, dim, world); no call allocates except
 *    the first lmscale_sync_dense_baseline / lmscale_train_step_host (their
 *    staging buffers).
 *  - Ids are uint32 word indices; an id >= vocab is an error
 *    (LMSCALE_ERR_ID_RANGE), detected on the device and reported at the next
 *    host synchronisation point of the call that reports it (below).  Kernels
 *    never access memory out of bounds for such ids; outputs of a call that
 *    returned an error are unspecified.
 *  - Row-major layouts: grad is k x dim, table is vocab x dim, rows are
 *    contiguous with stride dim floats.  dim % 4 == 0 with 16-byte aligned
 *    pointers takes the 128-bit vector path; any dim >= 1 is accepted.
 *  - Collective calls (lmscale_sync_embedding_grad, lmscale_sync_dense_baseline,
 *    lmscale_train_step_host with world > 1) must be made by every rank in the
 *    same order with the same k (the ID all-gather is fixed-size).  world == 1
 *    makes no NCCL call.
 *  - Errors are status codes; nothing is thrown across the ABI.  One context
 *    per (process, GPU); a context is not thread-safe.
 *  - Numerics: lr multiplies the raw sum (plain SGD, reading R3);
 *    pass lr / G for averaging.  Accumulation is fp32.
 */
#ifndef LMSCALE_H
#define LMSCALE_H

#include <stdint.h>

#if defined(__GNUC__)
#define LMSCALE_API __attribute__((visibility("default")))
#else
#define LMSCALE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lmscale_ctx lmscale_ctx; /* opaque, one per rank */

typedef enum {
  LMSCALE_OK = 0,
  LMSCALE_ERR_INVALID_ARG = 1, /* null / misaligned pointer, k < 1 or k > max_tokens, bad config, wrong call order */
  LMSCALE_ERR_ID_RANGE = 2,    /* some id >= vocab */
  LMSCALE_ERR_CUDA = 3,        /* CUDA runtime error (message: lmscale_last_error) */
  LMSCALE_ERR_NCCL = 4,        /* NCCL error or asynchronous communicator error */
  LMSCALE_ERR_OOM = 5,         /* workspace allocation failed */
  LMSCALE_ERR_UNSUPPORTED = 6, /* e.g. a collective call on a LMSCALE_FLAG_NO_COMM context */
  LMSCALE_ERR_CONSISTENCY = 7  /* LMSCALE_FLAG_CHECK: U_g or the I^ checksum differs across ranks
                                  (S:268); every rank returns it */
} lmscale_status;

/* Context flags. */
#define LMSCALE_FLAG_NO_COMM 1u /* no NCCL communicator: staged calls only (test emulation of G ranks) */
#define LMSCALE_FLAG_TIMING 2u  /* record CUDA events around each phase; lmscale_get_stats reports them */
#define LMSCALE_FLAG_CHECK 8u   /* debug: after S3 of every collective call, all-gather (U_g, a
                                   checksum of I^) and compare across ranks: one host
                                   sync per call; disables graph capture */
#define LMSCALE_FLAG_GRAPH 4u   /* lmscale_step captures the whole step into a CUDA graph (once per
                                   (ids, grad, table, k, lr) tuple) and replays it; applies with
                                   num_unique_out == NULL (no host round trip) and either
                                   world == 1 or a world > 1 context with the symmetric window
                                   (peer-bitmap S3 + fused S5+S6: no NCCL host calls) */

typedef struct {
  int64_t vocab;      /* |V| >= 1 */
  int64_t max_tokens; /* K capacity per rank, >= 1 */
  int64_t dim;        /* D >= 1 */
  int32_t world;      /* G >= 1 */
  int32_t rank;       /* 0 <= rank < world */
  int32_t device;     /* CUDA device ordinal of this rank */
  uint32_t flags;     /* LMSCALE_FLAG_* */
} lmscale_config;

/* The synchronised sparse gradient: a borrowed view into the
 * context's workspace, valid until the next call on the same context that
 * runs S1-S5. */
typedef struct {
  const uint32_t* ids;   /* device, I^ ascending, num_unique entries */
  const int32_t* counts; /* device, num_unique entries: tokens of word I^[r] over all ranks
                            (the global counts of step 4) after lmscale_sync_embedding_grad
                            (and lmscale_get_sparse_grad after it); NULL after the staged
                            calls and after lmscale_step, which do not compute them */
  float* rows;           /* device, num_unique x dim row-major: M^ after a collective sync,
                            this rank's M_g after lmscale_scatter_expand;
                            NULL after an lmscale_step that consumed the rows (S6 folded
                            into S4 at world 1, or the fused S5+S6 kernel), also from
                            lmscale_get_sparse_grad */
  int64_t num_unique;    /* host value U_g (-1 when the step kept it on the device) */
} lmscale_sparse_grad;

typedef struct {
  int64_t u_local;  /* U_i of the last S1 */
  int64_t u_global; /* U_g of the last S3 */
  /* per-phase device time of the last collective sync, microseconds (FLAG_TIMING; else -1) */
  double us_dedup, us_gather, us_merge, us_scatter, us_allreduce, us_update, us_total;
  /* per-rank byte accounting of the last lmscale_step / sync / host step, for
     the kernels that ran (SURVEY Sec. 8(d) algorithmic bytes; filled on every
     path, U_g read back from the device if the step kept it there): */
  int64_t bytes_ids_gathered;  /* S2 ingress: 4 (G-1) K ids, or 4 ceil(V/32) (G-1) bitmap words */
  int64_t bytes_grad_allreduce;/* S5 payload: 4 U_g D (2 U_g D compressed); 0 at world 1 */
  int64_t bytes_scatter;       /* S4: 4 K D read + rows written (4 U_g D; local-slot layout
                                  4 U_i D; world-1 fold: 8 U_g D, each E row read + written) */
  int64_t bytes_update;        /* separate S6 launch: 12 U_g D; 0 when folded or fused */
  int64_t workspace_bytes;     /* device bytes owned by the context */
  int32_t kernels_last_call;   /* kernels this library launched in the last call */
  int32_t kernels_total_lo;    /* running count of launched kernels (low 31 bits) */
  int32_t fused_s5_s6;         /* 1: the last step ran S5+S6 as one multicast (NVLS) kernel
                                  with a caller-owned table (us_allreduce then times that
                                  kernel, us_update ~ 0);
                                  2: same with the context's table window (peer-to-peer
                                  kernel for world <= 8: stores into every replica);
                                  3: the compressed (binary16) exchange of
                                  lmscale_set_compression */
  int32_t nvls_available;      /* 1: the context has the multicast window (world > 1) */
} lmscale_stats;

/* ------------------------------------------------------------------ setup */

/* Rank 0 creates the NCCL unique id (128 host bytes) that every rank passes
 * to lmscale_init; the caller distributes it (e.g. a torch.distributed
 * broadcast).  Not needed when world == 1 or FLAG_NO_COMM. */
LMSCALE_API lmscale_status lmscale_get_nccl_id(uint8_t out_id[128] /* host */);

/* Create a context: cudaSetDevice(cfg->device), ncclCommInitRank when
 * world > 1 and !FLAG_NO_COMM, and allocate the workspace (about
 * 4*world*max_tokens + 4*min(world*max_tokens, vocab)*dim + 40*max_tokens +
 * vocab/2 bytes).  *out receives the context, or NULL on error. */
LMSCALE_API lmscale_status lmscale_init(const lmscale_config* cfg /* host */,
                            const uint8_t* nccl_id /* host, 128 bytes, or NULL */,
                            lmscale_ctx** out /* host */);

/* Free the workspace and the communicator (after a device synchronise). */
LMSCALE_API void lmscale_destroy(lmscale_ctx* ctx);

/* ------------------------------------------------------- staged operations
 * These are the per-rank steps of P:402-422 with no communication.  They are
 * what the collective call below runs between its two NCCL calls, and they let
 * a test emulate G ranks with G NO_COMM contexts on one GPU. */

/* S1, step 1: J^ = sorted distinct ids (ascending, reading R2),
 * counts[u] = #{p : ids[p] = J^[u]}, inverse[p] = index of ids[p] in J^.
 * uniq_out / counts_out need capacity k, inverse_out k entries; each may be
 * NULL (results stay in the workspace).  *num_unique_out (device int64, may be
 * NULL) receives U_i.  Errors: INVALID_ARG; ID_RANGE is reported by the next
 * lmscale_get_sparse_grad / collective call. */
LMSCALE_API lmscale_status lmscale_unique(lmscale_ctx* ctx, const uint32_t* ids, int64_t k,
                              uint32_t* uniq_out, int32_t* counts_out,
                              int32_t* inverse_out, int64_t* num_unique_out,
                              void* stream);

/* S3, step 4 over a caller-provided gathered id vector I (n ids,
 * n <= world * max_tokens): I^ = sorted distinct(I), U_g = |I^|, and the map
 * l2g[u] = position of J^[u] in I^ for the J^ of the last lmscale_unique on
 * this context. */
LMSCALE_API lmscale_status lmscale_global_unique(lmscale_ctx* ctx, const uint32_t* gathered,
                                     int64_t n, void* stream);

/* S4, steps 2+5: M_g[l2g[u]] = sum of grad rows of J^[u]
 * (segmented fp32 sum, deterministic order), every other of the U_g rows is
 * exactly 0.  grad is the k x dim gradient belonging to the ids of the last
 * lmscale_unique (same k).  Requires lmscale_unique then lmscale_global_unique. */
LMSCALE_API lmscale_status lmscale_scatter_expand(lmscale_ctx* ctx, const float* grad, int64_t k,
                                      void* stream);

/* Synchronise `stream` and return the view of I^ / M and U_g.  Returns
 * ID_RANGE if any id seen since the last S1 was >= vocab. */
LMSCALE_API lmscale_status lmscale_get_sparse_grad(lmscale_ctx* ctx, lmscale_sparse_grad* out /* host */,
                                       void* stream);

/* Debug/parity views of the last S1/S3 maps (device pointers into the
 * workspace; synchronises `stream`).  Any out pointer may be NULL. */
LMSCALE_API lmscale_status lmscale_get_local_maps(lmscale_ctx* ctx, const uint32_t** uniq,
                                      const int32_t** counts, const int32_t** inverse,
                                      const int32_t** l2g, int64_t* num_unique_local /* host */,
                                      void* stream);

/* ------------------------------------------------------ collective path */

/* S1-S5: the whole uniqueness exchange of one step.  ids: k
 * uint32, grad: k x dim fp32.  On return out->ids / out->rows hold I^ and the
 * all-reduced M^ (identical on every rank) and out->num_unique = U_g (host).
 * The call blocks the host until U_g is known (one 16-byte device->host read,
 * hidden behind S4), because NCCL takes its element count from the host.
 * world == 1: no NCCL, out->rows = M_0.  Errors: INVALID_ARG, ID_RANGE (all
 * ranks see it: I is identical everywhere; no all-reduce is issued), CUDA,
 * NCCL, UNSUPPORTED (NO_COMM context). */
LMSCALE_API lmscale_status lmscale_sync_embedding_grad(lmscale_ctx* ctx, const uint32_t* ids,
                                           const float* grad, int64_t k,
                                           lmscale_sparse_grad* out /* host */,
                                           void* stream);

/* S6, step 7 (no duplicates P:433-435): for r < sg->num_unique,
 * table[sg->ids[r], :] = table[sg->ids[r], :] - lr * sg->rows[r, :]
 * (one fused multiply-add per element, rows disjoint, no atomics).  sg is a
 * view returned by this context (or any device I^/rows pair with the
 * documented layout).  table: vocab x dim, in place. */
LMSCALE_API lmscale_status lmscale_apply_sparse_update(lmscale_ctx* ctx, float* table,
                                           const lmscale_sparse_grad* sg /* host */,
                                           float lr, void* stream);

/* One whole training-step exchange, S1-S6: the collective sync
 * of lmscale_sync_embedding_grad followed by the row update of
 * lmscale_apply_sparse_update on `table` (vocab x dim, in place), in one call.
 * With world == 1 and num_unique_out == NULL the host never waits: S6 reads
 * U_g on the device, so the call returns as soon as the kernels are enqueued.
 * num_unique_out (host, may be NULL) receives U_g (forces a host sync point).
 * Collective when world > 1; errors as lmscale_sync_embedding_grad (with
 * world == 1 and no host sync, ID_RANGE surfaces at the next
 * lmscale_get_sparse_grad). */
LMSCALE_API lmscale_status lmscale_step(lmscale_ctx* ctx, const uint32_t* ids, const float* grad,
                                        int64_t k, float* table, float lr,
                                        int64_t* num_unique_out /* host, or NULL */, void* stream);

/* The world-G step of lmscale_step on ONE GPU, for validating
 * the G > 1 kernels without G GPUs: ctxs[r] (host array, r < world, 2 <=
 * world <= 8) are NO_COMM contexts of rank r of `world` on the same device,
 * with equal vocab, dim, max_tokens and compression setting; ids[r] (k
 * uint32), grads[r] (k x dim fp32) and tables[r] (rank r's replica of E,
 * vocab x dim, updated in place) are device pointers in host arrays.  Runs
 * the kernels of lmscale_step's P2P path -- S1 on every rank; S3 as the
 * J^-set exchange (each rank ORs the G presence bitmaps, reading the other
 * contexts' windows); S4 in the local-slot layout; the fused S5+S6 kernel of
 * every rank (compressed, Sec. 3.3: both phases of the codec exchange),
 * reading the peers' M rows and storing each updated row into every replica
 * -- with the NCCL window replaced by the contexts' buffers and the
 * cross-rank barriers by launch order (every S1 before any S3, every S4
 * before any exchange, every compressed phase 1 before any phase 2).
 * Synchronises `stream`.  Errors: INVALID_ARG (mismatched contexts, NULL
 * pointers, k out of range), ID_RANGE (an id >= vocab on any rank: no
 * replica is touched), CUDA. */
LMSCALE_API lmscale_status lmscale_emulate_step(lmscale_ctx* const* ctxs /* host */, int world,
                                                const uint32_t* const* ids /* host array */,
                                                const float* const* grads /* host array */,
                                                int64_t k, float* const* tables /* host array */,
                                                float lr, void* stream);

/* S0, the comparison path: all-gather ids and the k x dim grad
 * rows of every rank (Theta(G K D) bytes), then apply all G*k row updates
 * table[I[q]] -= lr * Delta_all[q] with 128-bit vector atomics (the paper's
 * "rows under update are locked").  Collective.  First call allocates the
 * 4*world*max_tokens*dim byte gather buffer. */
LMSCALE_API lmscale_status lmscale_sync_dense_baseline(lmscale_ctx* ctx, const uint32_t* ids,
                                           const float* grad, int64_t k, float* table,
                                           float lr, void* stream);

/* The dense atomic scatter alone (staged dense path): table[ids[q]] -= lr *
 * grad[q] for q < n.  n <= world * max_tokens. */
LMSCALE_API lmscale_status lmscale_dense_apply(lmscale_ctx* ctx, const uint32_t* ids, const float* grad,
                                   int64_t n, float* table, float lr, void* stream);

/* One end-to-end step from HOST buffers: copy ids (k uint32) and grad (k x dim
 * fp32) host->device (pinned memory recommended), run S1-S6 on `table`
 * (device), copy I^ back to ids_out (host, capacity world*k) and U_g to
 * *num_unique_out (host).  Synchronises `stream` before returning.
 * Collective when world > 1. */
LMSCALE_API lmscale_status lmscale_train_step_host(lmscale_ctx* ctx, const uint32_t* ids_host,
                                       const float* grad_host, int64_t k, float* table,
                                       float lr, uint32_t* ids_out_host,
                                       int64_t* num_unique_out, void* stream);

/* ---------------------------------------------------------------- misc */

/* Allocate the vocab x dim fp32 embedding table E on this context's device
 * (owned by the context, freed by lmscale_destroy).  Collective when world > 1
 * and the context has the symmetric window: the table is then allocated with
 * ncclMemAlloc and registered as a symmetric window, and lmscale_step's fused
 * S5+S6 kernel stores each updated row straight into every replica of E over
 * NVLink (peer-to-peer for world <= 8, multicast above; no local copy phase).
 * Any caller-owned table keeps working; this one is faster.
 * *bytes_out (host, may be NULL) receives vocab * dim * 4. */
LMSCALE_API lmscale_status lmscale_alloc_table(lmscale_ctx* ctx, float** table_out /* host */,
                                               int64_t* bytes_out /* host */);

/* Timing mode of subsequent calls: 0 none, 1 only the two events bracketing
 * the S4 kernel (us_scatter), 2 every phase (all us_* fields; each event is a
 * GPU-side serialisation point of a few microseconds, so mode 2 inflates the
 * step it measures), 3 only the two events bracketing the S5 (+ S6) phase
 * (us_allreduce: the fused S5+S6 kernel at world > 1).  FLAG_TIMING at init
 * selects mode 2.  INVALID_ARG outside 0..3. */
LMSCALE_API lmscale_status lmscale_set_timing(lmscale_ctx* ctx, int mode);

/* Compression (Sec. 3.3; reading R15).  F > 0 makes
 * every later collective lmscale_step / lmscale_train_step_host (world > 1)
 * exchange binary16 payloads instead of fp32 rows:
 *   - S4 stores each row of M_g as RNE(fp32(F * x)), saturated to +-65504;
 *   - the owner of row r (r mod world == rank) up-casts the copies of the ranks
 *     holding word I^[r], divides each by F, sums them in fp32 in rank order
 *     and sends the compressed sum to every rank;
 *   - every rank up-casts M^ (one fp32 division by F) and applies S6 to its
 *     own table: E[I^[r]] = fma(-lr, M^[r], E[I^[r]]).
 * Half the NVLink bytes of the fp32 exchange; replicas stay bit-identical.
 * F == 0 turns compression off.  F < 0 or non-finite: INVALID_ARG.  world > 1
 * needs the symmetric window (stats.nvls_available == 1), else UNSUPPORTED
 * (NO_COMM contexts accept F: it applies to lmscale_emulate_step).
 * world == 1 has no communication and is unaffected.  While compression is
 * on, lmscale_sync_embedding_grad (fp32 M^ rows through NCCL) returns
 * UNSUPPORTED. */
LMSCALE_API lmscale_status lmscale_set_compression(lmscale_ctx* ctx, float F);

/* The 16-bit format of the compressed exchange and of lmscale_compress /
 * lmscale_decompress ("fp16 (and bf16)"; R15):
 * LMSCALE_CODEC_FP16 (binary16, the paper's, default; saturates at +-65504)
 * or LMSCALE_CODEC_BF16 (bfloat16: same RNE of fp32(F * x), saturates at
 * +-0x7F7F = +-3.3895e38).  INVALID_ARG for any other value. */
#define LMSCALE_CODEC_FP16 0
#define LMSCALE_CODEC_BF16 1
LMSCALE_API lmscale_status lmscale_set_codec(lmscale_ctx* ctx, int32_t codec);

/* The codec alone, device pointers, stream-ordered, i < n, in the
 * context's 16-bit format (lmscale_set_codec; binary16 by default):
 * compress:   q[i] = bits of RNE(fp32(F * x[i])), saturated (binary16: +-65504);
 * decompress: x[i] = fp32(q[i]) / F (exact widening, one fp32 division).
 * F > 0 and finite, n >= 0 (n == 0 launches nothing), else INVALID_ARG. */
LMSCALE_API lmscale_status lmscale_compress(lmscale_ctx* ctx, const float* x, int64_t n, float F,
                                            uint16_t* q, void* stream);
LMSCALE_API lmscale_status lmscale_decompress(lmscale_ctx* ctx, const uint16_t* q, int64_t n,
                                              float F, float* x, void* stream);

/* Seeding (Sec. 3.2; reading R16).  Sampled softmax
 * picks S candidate words per GPU (1024 in the paper); GPUs that share
 * a seed draw the same words, so the output-embedding exchange over
 * [K targets || S samples] keeps a small global unique set.  Policies: */
#define LMSCALE_SEED_DISTINCT 0 /* every GPU its own seed (G groups) */
#define LMSCALE_SEED_SAME 1     /* one seed for all (1 group) */
#define LMSCALE_SEED_LOG2 2     /* max(1, round(log2 G)) groups */
#define LMSCALE_SEED_LOGE 3     /* max(1, round(ln G)) groups */
#define LMSCALE_SEED_LOG10 4    /* max(1, round(log10 G)) groups */
#define LMSCALE_SEED_POWER 5    /* max(1, ceil(G^alpha)) groups, 0 < alpha <= 1 (0.64) */

/* Host only (no GPU, no context): seeds_out[r] (host, world entries) = the
 * seed of rank r.  Ranks form contiguous near-equal blocks, group(r) =
 * floor(r * n / world); seed of group q = SplitMix64 output of master + q.
 * *groups_out (host, may be NULL) = n.  INVALID_ARG: world < 1, unknown
 * policy, alpha outside (0, 1] for POWER, NULL seeds_out. */
LMSCALE_API lmscale_status lmscale_plan_seeds(int32_t world, int32_t policy, double alpha,
                                              uint64_t master_seed, uint64_t* seeds_out,
                                              int32_t* groups_out);

/* Draw S candidate ids (device, S uint32 written to out) uniformly without
 * replacement from [0, vocab): the first S distinct values of the stream
 * x_i = floor(u_i * vocab / 2^64), u_i = mix64(A + i), A = mix64(seed ^
 * mix64(step)) (R16), in stream order.  Deterministic per (seed, step, S,
 * vocab); ranks with the same seed and step get the same ids.  One CTA,
 * stream-ordered.  INVALID_ARG: S < 1, S > vocab, S > 8192, out NULL. */
LMSCALE_API lmscale_status lmscale_draw_samples(lmscale_ctx* ctx, uint64_t seed, uint64_t step,
                                                int64_t S, uint32_t* out, void* stream);

/* Forward lookup: out[p, :] = table[ids[p], :]
 * for p < k -- the K x dim input activations the gradient rows of the
 * exchange belong to.  ids: k uint32 (device), table: vocab x dim, out: k x dim
 * (device, caller-owned).  An id >= vocab yields a zero row (no error is
 * raised here; lmscale_unique / the step report ID_RANGE).  Stream-ordered,
 * no communication.  INVALID_ARG: NULL pointers, k < 0. */
LMSCALE_API lmscale_status lmscale_lookup(lmscale_ctx* ctx, const uint32_t* ids, int64_t k,
                                          const float* table, float* out, void* stream);

LMSCALE_API lmscale_status lmscale_get_stats(const lmscale_ctx* ctx, lmscale_stats* out /* host */);
LMSCALE_API const char* lmscale_status_string(lmscale_status s);
/* Last detailed error message of this context (static storage inside ctx). */
LMSCALE_API const char* lmscale_last_error(const lmscale_ctx* ctx);
/* Library version string, e.g. "lmscale 0.2 sm_100a" ("+device-checks" for the checked build). */
LMSCALE_API const char* lmscale_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LMSCALE_H */
