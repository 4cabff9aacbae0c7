// kernels.cuh -- internal launch interface of the lmscale CUDA kernels.
// Not part of the public ABI (include/lmscale.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <nccl.h>

namespace lms {

struct GridBar;

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

// ---- S3 (coop.cu) ----------------------------------------------------------
constexpr int CO_THREADS = 512;
constexpr int CO_HOTW = 2048;  // shared-memory bitmap words in S3

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
  const uint32_t* lrank;  // S1's per-word local prefix (index in J^ of word w's first id)
  const Sc1* sc1;
  int32_t* l2g;
  unsigned long long* trace;
  GridBar* bar;
  // peer mode (the J^-set exchange): instead of building
  // the bitmap from a gathered I, OR the G local presence bitmaps (S1's lbits)
  // read from the peers' symmetric windows after a flag handshake
  int peer_mode;         // 1: flag handshake; 2: emulation (lmscale_emulate_step:
                         // every rank's S1 ran before, errors from peer_sc1)
  int world, rank;
  char* peer_base[8];   // LSA base of each rank's M window
  const Sc1* peer_sc1[8];  // peer_mode 2: each rank's S1 scalars
  size_t lbits_off;     // byte offset of lbits in the window
  size_t flags_off;     // byte offset of the per-rank arrival flags (world words)
  uint32_t* epoch;      // local step counter of the handshake (device)
};

cudaError_t launch_s3(const S3Args& a, int num_sms, cudaStream_t s);
// Global counts of I^ (gcounts[r] = tokens of word I^[r] over all ranks):
// peer_base != nullptr: from every rank's S1 counts in its window (lbits,
// lrank, counts at the given offsets); else from the gathered ids I (n).
cudaError_t launch_gcounts(int32_t* gcounts, int64_t ucap, const uint32_t* ihat, const Sc3* sc3,
                           const uint32_t* I, int64_t n, const uint32_t* gbits,
                           const uint32_t* wrank, uint32_t vocab, int world,
                           char* const* peer_base, size_t lbits_off, size_t lrank_off,
                           size_t counts_off, int num_sms, cudaStream_t s);

// ---- S1 grouping (group.cu): one launch, three grid barriers ----------------
constexpr int G1_THREADS = 512;
constexpr int G1_MAX_GRID = 1024;
constexpr int G1_STRIPES = 16;
struct G1Args {
  const uint32_t* ids;
  int K;
  uint32_t vocab;
  uint32_t* wcount;   // [32 W] tokens per id (transposed layout); all zero between launches
  uint32_t* tick;     // [K] rank of the token among equal ids (arrival order)
  uint32_t* lbits;    // [W] presence bitmap; zero on entry unless zero_bits
  uint32_t* lrank;    // [W] index in J^ of the first present id of each 32-id word
  int64_t W;
  uint32_t* ctot;     // [G1_STRIPES][2 * grid] per-range (ids, tokens); zero between launches
  uint32_t* luniq;    // J^ (U_i)
  int32_t* counts;    // tokens per word of J^
  int32_t* lstart;    // first grouped position of each run (U_i + 1)
  int32_t* perm;      // grouped position -> token position
  int32_t* inverse;   // token position -> u (-1 for an id >= vocab)
  int32_t* runfirst;  // [nr + 1] run holding the first position of each S4 range; [nr] = U_i
  int nr;             // S4 ranges: [r seg_len, min(K, (r + 1) seg_len))
  uint32_t seg_len;
  Sc1* sc;
  int64_t* nu_out;
  int zero_bits;
  unsigned long long* trace;
  // world 1 (I = J): I^ = J^, l2g = identity, U_g = U_i; S3 is skipped
  uint32_t* ihat;
  int32_t* l2g;
  Sc3* sc3;
  GridBar* bar;     // in-kernel grid barrier (zeroed at init)
};
cudaError_t launch_group(const G1Args& a, int num_sms, cudaStream_t s);

void launch_counts_export(const int32_t* lstart, const uint32_t* luniq, const int32_t* inverse,
                          const Sc1* sc, int K, int32_t* counts, uint32_t* uniq_out,
                          int32_t* counts_out, int32_t* inverse_out, cudaStream_t s);

// ---- S4 (segsum.cu): bulk-copy-staged segmented sum over equal ranges -------
constexpr int SEG_MAX_SLOTS = 16;   // mbarrier ring slots (gradient groups, E rows)
constexpr int SEG_MAX_L = 4096;     // grouped positions per CTA range
constexpr int SEG_MAX_OCC = 4;      // CTAs per SM
constexpr int SEG_FXP = 8;          // partial rows of a cut run summed per group
constexpr int SEG_MAX_THREADS = 544;
struct SegArgs {
  const float* grad;      // K x D
  const int32_t* perm;    // grouped position -> token position
  const int32_t* runfirst;  // [nr + 1] run holding each range's first position (S1)
  const int32_t* lstart;  // u -> first grouped position (U_i + 1 entries)
  const uint32_t* word;   // u -> word id (world-1 apply: J^ = I^)
  const int32_t* l2g;     // u -> slot of M (global layout), nullptr: slot = u
  const Sc1* sc1;         // err
  float* table;           // apply: E, vocab x D
  float lr;
  int apply;              // world 1: S6 folded in (E rows updated, no M)
  float* M;               // slots x D (fp32, or binary16 when m16)
  int m16;
  float cF;
  int cbf;
  float* part;            // [2 nR] x D partial rows of cut runs
  float* part2;           // [2 nR] x D group sums of the partial rows
  uint32_t* cnt;          // [2 nR x ncb] group counters (zero between launches)
  uint32_t* cnt2;         // [nR x ncb] run counters (zero between launches)
  uint32_t* lbits;        // clear_bits: zeroed here (world 1)
  int64_t W;
  int clear_bits;
  int pdl;                // launched as a programmatic dependent of S1
  unsigned long long* trace;  // LMSCALE_PHASE_TRACE stamps (or nullptr)
  int K, D, num_sms;
  uint32_t seg_len;       // set by launch_seg: grouped positions per range
  int fold;               // range geometry of the S1 that ran before (seg_plan)
  uint32_t vocab;         // bounds of the checked build (LMS_CHECK)
  int64_t mrows, part_rows;
  int cbw, nct, gr, nslot, neslot, lmax;
};
struct SegPlan {
  bool tma;
  int cbw, nct, threads, ncb, gr, nslot, neslot, occ, nr, lmax;
  size_t smem;
};
// fold: the launch geometry of the world-1 kernel with S6 folded in (else the
// M-row geometry); S1 cuts the ranges for the S4 that follows, so both use it
SegPlan seg_plan(int64_t K, int64_t D, bool vec, bool apply, bool fold, int num_sms);
// the S4 ranges for (K, D): nr ranges of seg_len grouped positions (the last
// one shorter); S1 writes runfirst for them
int seg_ranges(int64_t K, int64_t D, int num_sms, bool fold, uint32_t* seg_len);
int64_t seg_max_ranges(int64_t K, int num_sms);
cudaError_t launch_seg(const SegArgs& a, cudaStream_t s);
cudaError_t launch_zero_absent(float* M, int D, const uint32_t* ihat, const uint32_t* lbits,
                               const Sc3* sc3, const Sc1* sc1, int64_t ug_cap, int num_sms,
                               cudaStream_t s);
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
                        int64_t mcap, uint32_t vocab, cudaStream_t s);
// true: the peer-to-peer fused kernel (presence-aware) is used for this G
bool nvls_use_p2p(int world);
// LSA base of every rank's M window (world entries written to out_host)
bool nvls_peer_bases(NvlsState* st, int world, void** out_host);
// lmscale_emulate_step: rank `rank`'s P2P fused kernel with the peers'
// M-window bases / tables given directly (G contexts on one GPU, no
// barriers: launch order).  Compressed (cF > 0): phase 1 or 2.
cudaError_t launch_p2p_emulated(char* const* m_bases, float* const* tables, int world, int rank,
                                const uint32_t* ihat, const Sc3* sc3, const float* M, int D,
                                float lr, size_t lbits_off, size_t lrank_off, size_t mhat_off,
                                float cF, int cbf, int phase, int64_t mcap, uint32_t vocab,
                                int num_sms, cudaStream_t s);
ncclWindow_t nvls_register_table(ncclComm_t comm, void* table, size_t bytes, char* err,
                                 size_t errlen);
void nvls_deregister_table(ncclComm_t comm, ncclWindow_t w);

}  // namespace lms
