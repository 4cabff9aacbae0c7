// kernels.cuh -- internal launch interface of the lmscale CUDA kernels.
// Not part of the public ABI (include/lmscale.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lms {

// Radix sort tile: 256 threads x 16 keys.
constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 4096
constexpr int RS_MAX_PASSES = 4;

// Segment kernel tile (same shape).
constexpr int SEG_TILE = RS_TILE;

// Bitmap scan tile: 256 threads x 4 words.
constexpr int GS_THREADS = 256;
constexpr int GS_TILE_WORDS = GS_THREADS * 4;

// Scatter-add chunk: sorted positions per warp work item.
constexpr int SC_CHUNK = 32;
// Zero-row group: slots per warp work item.
constexpr int SC_ZGROUP = 32;

// Per-step device scalars of S1 (zeroed at the start of S1).
struct Sc1 {
  int64_t u_local;
  uint32_t err;        // bit 0: an id >= vocab seen by S1
  uint32_t tile_ctr[RS_MAX_PASSES + 1];  // radix passes, segments
  uint32_t pad;
};
// Per-step device scalars of S3 (zeroed at the start of S3).
struct Sc3 {
  int64_t u_global;
  uint32_t err;        // bit 0: an id >= vocab in I
  uint32_t tile_ctr;   // bitmap scan
};

struct SortPlan {
  int passes;
  int bits;  // digit width per pass
};
SortPlan make_sort_plan(uint64_t vocab);

// ---- S1 -------------------------------------------------------------------
void launch_radix_hist(const uint32_t* keys, int K, SortPlan plan, uint32_t* hist, Sc1* sc,
                       uint32_t vocab, cudaStream_t s);
void launch_radix_pass(int pass, const uint32_t* kin, const int32_t* vin, uint32_t* kout,
                       int32_t* vout, int K, SortPlan plan, const uint32_t* hist, uint32_t* lb,
                       Sc1* sc, cudaStream_t s);
void launch_segments(const uint32_t* sk, const int32_t* sv, int K, uint32_t vocab,
                     uint32_t* luniq, int32_t* lstart, int32_t* segidx, int32_t* inverse,
                     uint32_t* lbits, Sc1* sc, uint32_t* lb, int64_t* nu_out, cudaStream_t s);
void launch_counts_export(const int32_t* lstart, const uint32_t* luniq, const int32_t* inverse,
                          const Sc1* sc, int K, int32_t* counts, uint32_t* uniq_out,
                          int32_t* counts_out, int32_t* inverse_out, cudaStream_t s);

// ---- S3 -------------------------------------------------------------------
void launch_gbits(const uint32_t* I, int64_t n, uint32_t vocab, uint32_t* gbits, Sc3* sc,
                  cudaStream_t s);
void launch_gscan(const uint32_t* gbits, int64_t W, uint32_t* wrank, uint32_t* ihat, Sc3* sc,
                  uint32_t* lb, cudaStream_t s);
void launch_l2g(const uint32_t* luniq, const Sc1* sc1, int K, uint32_t vocab,
                const uint32_t* gbits, const uint32_t* wrank, int32_t* l2g, cudaStream_t s);

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
  float* M;               // U_g x D
  float* partial;         // 2 * nchunks x D
  int K;
  int D;
  int64_t ug_cap;         // capacity bound on U_g (sizes the grid)
  int num_sms;
};
void launch_scatter(const ScatterArgs& a, cudaStream_t s);
void launch_fixup(const ScatterArgs& a, cudaStream_t s);

// ---- S6 / S0 --------------------------------------------------------------
void launch_update(float* table, int D, const uint32_t* ids, const float* rows, int64_t n,
                   float lr, int num_sms, cudaStream_t s);
void launch_dense(float* table, int D, const uint32_t* ids, const float* grad, int64_t n,
                  float lr, uint32_t vocab, int num_sms, cudaStream_t s);

}  // namespace lms
