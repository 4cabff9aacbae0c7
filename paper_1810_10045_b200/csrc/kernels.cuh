// kernels.cuh -- internal launch interface of the lmscale CUDA kernels.
// Not part of the public ABI (include/lmscale.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <nccl.h>

namespace lms {

struct GridBar;

// Scatter-add chunk: sorted positions per warp work item.
constexpr int SC_CHUNK = 32;
// Fix-up: partial rows summed per CTA work item.
constexpr int FX_PART = 128;
// Runs of <= FX_SHORT tokens are summed whole by the chunk holding their start
// (<= SC_CHUNK: the read-on past a chunk edge stays within one more chunk).
constexpr int FX_SHORT = 32;
// Zero-row group: slots per warp work item.
constexpr int SC_ZGROUP = 32;

// Per-step device scalars of S1 (zeroed at the start of S1).
struct Sc1 {
  int64_t u_local;
  uint32_t err;        // bit 0: an id >= vocab seen by S1; bit 1: S4 split a run into fix-up parts
  uint32_t fixcount;   // S4: runs cut by chunk boundaries (zeroed by S1)
};
// Per-step device scalars of S3 (zeroed at the start of S3).
struct Sc3 {
  int64_t u_global;
  uint32_t err;        // bit 0: an id >= vocab in I
  uint32_t pad;
};

struct SortPlan {
  int passes;
  int bits;  // digit width per pass
};

// ---- cooperative S1 / S3 (coop.cu) -----------------------------------------
constexpr int CO_THREADS = 512;
constexpr int CO_ITEMS = 8;
constexpr int CO_TILE = CO_THREADS * CO_ITEMS;  // 4096 keys per tile
constexpr int CO_MAX_BITS = 11;                 // <= 2048 digits per pass
constexpr int CO_HOTW = 2048;                   // shared-memory bitmap words in S3

struct S1Args {
  const uint32_t* ids;
  int K;
  uint32_t vocab;
  int passes, bits;
  uint32_t *ka, *kb;
  int32_t *va, *vb;
  uint32_t* cT;  // [passes][1 << bits][ntp] digit-major per-tile counts
  uint32_t* bT;  // [ntiles][1 << bits] tile-major bases (one pass at a time)
  uint32_t* rtot;  // [grid] digit-range totals
  int ntiles, ntp;
  uint32_t* luniq;
  int32_t* lstart;
  int32_t* segidx;
  int32_t* inverse;
  uint32_t* lbits;
  uint32_t* lrank;  // optional: lrank[w] = local index of the first present id of word w
  int64_t W;
  uint32_t* heads;  // [ntiles]
  Sc1* sc;
  int64_t* nu_out;
  unsigned long long* trace;  // optional phase timestamps (LMSCALE_PHASE_TRACE)
  // world == 1 shortcut (I = J, so I^ = J^, U_g = U_i, l2g = identity): when
  // non-null, S1 also writes I^, l2g and the S3 scalars and S3 is skipped.
  uint32_t* ihat;
  int32_t* l2g;
  Sc3* sc3;
  GridBar* bar;  // in-kernel grid barrier (cooperative-size grid, normal launch)
};
struct S3Args {
  const uint32_t* I;
  int64_t n;
  uint32_t vocab;
  uint32_t* gbits;
  int64_t W;
  uint32_t* wrank;
  uint32_t* ihat;
  uint32_t* ctot;  // [grid]
  Sc3* sc;
  const uint32_t* luniq;  // nullptr: skip the l2g phase
  const Sc1* sc1;
  int32_t* l2g;
  unsigned long long* trace;
  GridBar* bar;
  // peer mode (the J^-set exchange): instead of building
  // the bitmap from a gathered I, OR the G local presence bitmaps (S1's lbits)
  // read from the peers' symmetric windows after a flag handshake
  int peer_mode;
  int world, rank;
  char* peer_base[8];   // LSA base of each rank's M window
  size_t lbits_off;     // byte offset of lbits in the window
  size_t flags_off;     // byte offset of the per-rank arrival flags (world words)
  uint32_t* epoch;      // local step counter of the handshake (device)
};
SortPlan make_coop_plan(uint64_t vocab);

// ---- cluster S1 (cluster.cu): K <= CL_MAX_CTAS * CL_MAX_TILE, one cluster --
constexpr int CL_THREADS = 512;
constexpr int CL_MAX_TILE = 4096;  // keys per CTA (512 threads x 8)
constexpr int CL_MAX_BITS = 10;
constexpr int CL_MAX_CTAS = 16;
SortPlan make_cluster_plan(uint64_t vocab);
size_t cluster_smem_bytes(int bits);
bool cluster_s1_ok(int K);
// Writes the stable permutation to a.va (a.ka/a.kb/a.vb unused).
cudaError_t launch_s1_cluster(const S1Args& a, cudaStream_t s);
size_t s1_smem_bytes(int bits);
cudaError_t launch_s1(const S1Args& a, int num_sms, cudaStream_t s);
cudaError_t launch_s3(const S3Args& a, int num_sms, cudaStream_t s);

void launch_counts_export(const int32_t* lstart, const uint32_t* luniq, const int32_t* inverse,
                          const Sc1* sc, int K, int32_t* counts, uint32_t* uniq_out,
                          int32_t* counts_out, int32_t* inverse_out, cudaStream_t s);

// ---- S4 -------------------------------------------------------------------
struct ScatterArgs {
  const float* grad;      // K x D
  const int32_t* perm;    // sorted position -> token position
  const int32_t* segidx;  // sorted position -> local unique index u
  const int32_t* l2g;     // u -> global slot
  const int32_t* lstart;  // u -> first sorted position (U_i + 1 entries)
  const uint32_t* ihat;   // slot -> word id
  const uint32_t* lbits;  // local presence bitmap
  const Sc3* sc3;         // U_g
  const Sc1* sc1;         // U_i
  Sc1* sc1w;              // fixup list counter
  int2* fixent;           // fix-up entries: (owner chunk, part | nparts << 16)
  float* part2;           // level-2 partial rows, one per entry (fix_cap x D)
  int fix_cap;
  int fx_last;            // 1: last-arriver fix-up (no grid barrier); 0: listed fix-up phase
  int fxp;                // last-arriver fix-up: partials per part
  int pdl;                // launched as a programmatic dependent of the S1 kernel before it
  uint32_t* fxcnt;        // last-arriver counters: parts [fx_stride], runs [fx_stride]
  int64_t fx_stride;      // nchunks x column blocks
  int zero_rows;          // 0: every slot is present locally (world 1): slot = local index
  int fill_absent;        // zero the M rows of slots absent on this rank (world > 1)
  int m16;                // M rows are stored compressed (binary16 of cF * x, R15)
  int apply;              // world 1: S6 folded in -- finished rows update `table`, no M
  float cF;               // compression scale F
  int cbf;                // codec: 0 binary16, 1 bfloat16
  int short_runs;         // finish runs <= FX_SHORT in their starting chunk (large K)
  float* table;           // non-null: world-1 fused S6 (E[I^[r]] -= lr * M[r])
  float lr;
  unsigned long long* trace;
  GridBar* bar;           // in-kernel grid barrier state (zeroed at init)
  float* M;               // U_g x D
  float* partial;         // 2 * nchunks x D
  int K;
  int D;
  int64_t ug_cap;         // capacity bound on U_g (sizes the grid)
  int num_sms;
};
// One launch: scatter, cut-run fix-up, and (a.apply) the world-1 S6.
cudaError_t launch_scatter(const ScatterArgs& a, cudaStream_t s);
// debug consistency check: out[0] = U_g, out[1] = checksum of I^
cudaError_t launch_checksum(const uint32_t* ihat, const Sc3* sc3, unsigned long long* out,
                            cudaStream_t s);
// forward lookup: out[p] = E[ids[p]] (zero row for an id >= vocab)
cudaError_t launch_lookup(const float* table, int D, const uint32_t* ids, int64_t n,
                          uint32_t vocab, float* out, int num_sms, cudaStream_t s);
// seeding (Sec. 3.2, R16): the first S distinct draws of the (seed, step) stream
constexpr int DRAW_MAX_S = 8192;
cudaError_t launch_draw_samples(uint64_t seed, uint64_t step, int S, uint64_t V, uint32_t* out,
                                cudaStream_t s);
// seed-group plan; returns the number of groups, -1 on a bad policy / alpha
int plan_seed_groups(int world, int policy, double alpha, uint64_t master, uint64_t* seeds);
// compression codec (R15): down = compress (fp32 -> binary16 bits), else decompress
cudaError_t launch_codec(bool down, const void* in, int64_t n, float F, int bf, void* out,
                         int num_sms, cudaStream_t s);

// ---- S6 / S0 --------------------------------------------------------------
// n_dev != nullptr: the row count is read on the device (min(n, *n_dev)); n
// is then the capacity that sizes the grid.
void launch_update(float* table, int D, const uint32_t* ids, const float* rows, int64_t n,
                   const Sc3* n_dev, float lr, int num_sms, cudaStream_t s);
void launch_dense(float* table, int D, const uint32_t* ids, const float* grad, int64_t n,
                  float lr, uint32_t vocab, int num_sms, cudaStream_t s);

// ---- S5+S6 fused over NVLS multicast (nvls.cu) ------------------------------
struct NvlsState;
// Collective (every rank, same order): window-register M and create a device
// communicator with a multimem mapping.  nullptr (+ err) if unsupported.
NvlsState* nvls_create(ncclComm_t comm, void* M, size_t bytes, int num_sms, char* err,
                       size_t errlen);
void nvls_destroy(ncclComm_t comm, NvlsState* st);
// twin != nullptr: `table` is the symmetric-window table registered as twin.
void launch_nvls_update(NvlsState* st, const uint32_t* ihat, const Sc3* sc3, float* table,
                        const float* M, int D, float lr, int rank, int world,
                        unsigned long long* trace, ncclWindow_t twin, size_t lbits_off,
                        float cF, int cbf, size_t mhat_off, size_t lrank_off, int local_m,
                        cudaStream_t s);
// true: the peer-to-peer fused kernel (presence-aware) is used for this G
bool nvls_use_p2p(int world);
// LSA base of every rank's M window (world entries written to out_host)
bool nvls_peer_bases(NvlsState* st, int world, void** out_host);
ncclWindow_t nvls_register_table(ncclComm_t comm, void* table, size_t bytes, char* err,
                                 size_t errlen);
void nvls_deregister_table(ncclComm_t comm, ncclWindow_t w);

}  // namespace lms
