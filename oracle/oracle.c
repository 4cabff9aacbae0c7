/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the uniqueness
 * embedding-gradient exchange of Patwary et al., "Language Modeling at Scale"
 * (arXiv 1810.10045), Sec. 3.1.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1810_10045_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant with the CUDA path.
 *
 * Citations: "P:n" = PAPER.md line n (Sec. 3.1 enumerate);
 * "S:n" = SPEC.md line n.  Every floating-point accumulation is fp64; the
 * single rounding to fp32 happens where the function says so (DESIGN.md
 * reading R5).  No blocking, fusion or reordering beyond the paper's steps.
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * (goldens, library cross-checks, brute force, invariants); see the
 * "Pins" table in DESIGN.md.  No function is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* qsort comparator: a library primitive serves as the sort of step 1/4. */
static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

/* lower_bound: first index i in sorted a[0..n) with a[i] >= key. */
static int64_t lower_bound_u32(const uint32_t* a, int64_t n, uint32_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/*
 * Step 1: "compute the vector J^, which holds the word indices of
 * only unique words in its input sequence" -- J^ = sorted(set(J)) (ascending,
 * DESIGN.md reading R2), counts[u] = #{p : J[p] = J^[u]},
 * inverse[p] = lower_bound(J^, J[p]) ("mapping from an entry in J to ...").
 * uniq/counts need capacity K; inverse has K entries.  Returns U_i.
 */
int64_t oracle_unique_local(const uint32_t* J, int64_t K, uint32_t* uniq,
                            int32_t* counts, int32_t* inverse) {
  if (K <= 0) return 0;
  uint32_t* tmp = (uint32_t*)malloc((size_t)K * sizeof(uint32_t));
  memcpy(tmp, J, (size_t)K * sizeof(uint32_t));
  qsort(tmp, (size_t)K, sizeof(uint32_t), cmp_u32);
  int64_t U = 0;
  for (int64_t i = 0; i < K; ++i)
    if (i == 0 || tmp[i] != tmp[i - 1]) uniq[U++] = tmp[i];
  free(tmp);
  for (int64_t u = 0; u < U; ++u) counts[u] = 0;
  for (int64_t p = 0; p < K; ++p) {
    int64_t u = lower_bound_u32(uniq, U, J[p]);
    inverse[p] = (int32_t)u;
    counts[u] += 1;
  }
  return U;
}

/*
 * Step 2: "a local reduction of the gradient vectors, so that the
 * gradient vectors corresponding to the same words are accumulated into a
 * single vector" -- dhat[u,:] = sum_{p : inverse[p] = u} delta[p,:], fp64,
 * ascending p.  dhat is U x D, overwritten.
 */
void oracle_reduce_local(const float* delta, int64_t K, int64_t D,
                         const int32_t* inverse, int64_t U, double* dhat) {
  for (int64_t i = 0; i < U * D; ++i) dhat[i] = 0.0;
  for (int64_t p = 0; p < K; ++p) {
    double* row = dhat + (int64_t)inverse[p] * D;
    const float* src = delta + p * D;
    for (int64_t d = 0; d < D; ++d) row[d] += (double)src[d];
  }
}

/*
 * Step 2 restricted to the columns [c0, c1) of every row: the same loop (same
 * per-element summation order, ascending p), so any split of the columns
 * gives bit-identical results.  Used only by the all-cores timing variant of
 * bench.py's cpu_baseline (one thread per column block).
 */
void oracle_reduce_local_cols(const float* delta, int64_t K, int64_t D,
                              const int32_t* inverse, int64_t U, double* dhat, int64_t c0,
                              int64_t c1) {
  for (int64_t r = 0; r < U; ++r)
    for (int64_t d = c0; d < c1; ++d) dhat[r * D + d] = 0.0;
  for (int64_t p = 0; p < K; ++p) {
    double* row = dhat + (int64_t)inverse[p] * D;
    const float* src = delta + p * D;
    for (int64_t d = c0; d < c1; ++d) row[d] += (double)src[d];
  }
}

/*
 * Step 3: AllGather over the J vectors of all G GPUs; I is their
 * rank-ordered concatenation (reading R1: the text's J, not J^).
 * Simulated here by copying rank g's K_g ids to offset sum_{h<g} K_h.
 */
void oracle_allgather_ids(const uint32_t* const* J, const int64_t* K, int G,
                          uint32_t* I) {
  int64_t off = 0;
  for (int g = 0; g < G; ++g) {
    memcpy(I + off, J[g], (size_t)K[g] * sizeof(uint32_t));
    off += K[g];
  }
}

/*
 * Step 4: "a local filter operation over the G x K indices
 * (vector I) to extract all unique word indices to produce vector I^", "totally
 * ordered" -> ascending (R2).  gcounts[r] = #{q : I[q] = I^[r]} (global type
 * counts).  Returns U_g.  Ihat/gcounts need capacity n.
 */
int64_t oracle_unique_global(const uint32_t* I, int64_t n, uint32_t* Ihat,
                             int32_t* gcounts) {
  if (n <= 0) return 0;
  uint32_t* tmp = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  memcpy(tmp, I, (size_t)n * sizeof(uint32_t));
  qsort(tmp, (size_t)n, sizeof(uint32_t), cmp_u32);
  int64_t U = 0;
  for (int64_t i = 0; i < n; ++i)
    if (i == 0 || tmp[i] != tmp[i - 1]) Ihat[U++] = tmp[i];
  free(tmp);
  if (gcounts) {
    for (int64_t r = 0; r < U; ++r) gcounts[r] = 0;
    for (int64_t q = 0; q < n; ++q) gcounts[lower_bound_u32(Ihat, U, I[q])] += 1;
  }
  return U;
}

/*
 * Step 4, the maps: "a mapping from an entry in J to the corresponding
 * entry in I^ and transitively from J^ to I^".
 *   l2g[u]  = lower_bound(I^, J^[u])            (J^ -> I^)
 *   slot[p] = l2g[inverse[p]]                   (J  -> I^, transitively)
 */
void oracle_remap(const uint32_t* Jhat, int64_t Ui, const uint32_t* Ihat,
                  int64_t Ug, const int32_t* inverse, int64_t K, int32_t* l2g,
                  int32_t* slot) {
  for (int64_t u = 0; u < Ui; ++u) l2g[u] = (int32_t)lower_bound_u32(Ihat, Ug, Jhat[u]);
  if (slot)
    for (int64_t p = 0; p < K; ++p) slot[p] = l2g[inverse[p]];
}

/*
 * Step 5: "expand the Delta^_i matrix ... from a U_i x D matrix
 * into a U_g x D matrix via a local scatter operation.  The non existing
 * entries are filled with zeros" -- M[l2g[u],:] = dhat[u,:], every other row
 * exactly 0 (R4).  M is Ug x D fp64, overwritten.
 */
void oracle_scatter_expand(const double* dhat, int64_t Ui, int64_t D,
                           const int32_t* l2g, int64_t Ug, double* M) {
  for (int64_t i = 0; i < Ug * D; ++i) M[i] = 0.0;
  for (int64_t u = 0; u < Ui; ++u)
    memcpy(M + (int64_t)l2g[u] * D, dhat + u * D, (size_t)D * sizeof(double));
}

/*
 * Step 6: AllReduce over all M_i -> M^ = sum_i M_i, summed in rank
 * order, fp64.  Mhat has n entries, overwritten.
 */
void oracle_allreduce_sum(const double* const* M, int G, int64_t n, double* Mhat) {
  for (int64_t i = 0; i < n; ++i) Mhat[i] = 0.0;
  for (int g = 0; g < G; ++g)
    for (int64_t i = 0; i < n; ++i) Mhat[i] += M[g][i];
}

/*
 * Step 7 (no duplicates P:433-435): "Update the local embedding matrix
 * with the values in M^ using I^ to map index in M^ with row in E" -- plain
 * SGD on the raw sum (R3): E[I^[r],:] = round32(E[I^[r],:] - lr * M^[r,:]),
 * evaluated in fp64 and rounded once (R5).  E is V x D fp32, in place.
 */
void oracle_update_rows(float* E, int64_t D, const uint32_t* Ihat, int64_t Ug,
                        const double* Mhat, double lr) {
  for (int64_t r = 0; r < Ug; ++r) {
    float* row = E + (int64_t)Ihat[r] * D;
    for (int64_t d = 0; d < D; ++d)
      row[d] = (float)((double)row[d] - lr * Mhat[r * D + d]);
  }
}

/*
 * Baseline dense exchange: AllGather all (J, Delta)
 * pairs and apply every one of the G*K row updates in rank-then-position
 * order: E64 = E0; E64[J_g[p],:] -= lr * Delta_g[p,:] (fp64); E = round32(E64)
 * (an untouched row is E0 exactly, so rounding it back is the identity).
 * E64 is a caller-provided V x D fp64 scratch.  E is V x D fp32, in place.
 */
void oracle_sync_dense(float* E, double* E64, int64_t V, int64_t D, int G,
                       const uint32_t* const* J, const float* const* delta,
                       const int64_t* K, double lr) {
  for (int64_t i = 0; i < V * D; ++i) E64[i] = (double)E[i];
  for (int g = 0; g < G; ++g)
    for (int64_t p = 0; p < K[g]; ++p) {
      double* row = E64 + (int64_t)J[g][p] * D;
      const float* src = delta[g] + p * D;
      for (int64_t d = 0; d < D; ++d) row[d] -= lr * (double)src[d];
    }
  for (int64_t i = 0; i < V * D; ++i) E[i] = (float)E64[i];
}

/*
 * Per-type conservation, by definition ("the rows corresponding to the
 * same word accumulate"): out[:] = sum over all ranks g and positions p with
 * J_g[p] == w of Delta_g[p,:], fp64, rank-then-position order.  This is one
 * row of M^ computed from first principles; the full-size GPU parity test
 * samples rows with it.  Returns the number of contributing tokens.  absout
 * (optional) receives sum |Delta_g[p,:]| (the summation-error scale A).
 */
int64_t oracle_type_gradient(const uint32_t* const* J, const float* const* delta,
                             const int64_t* K, int G, int64_t D, uint32_t w,
                             double* out, double* absout) {
  int64_t n = 0;
  for (int64_t d = 0; d < D; ++d) { out[d] = 0.0; if (absout) absout[d] = 0.0; }
  for (int g = 0; g < G; ++g)
    for (int64_t p = 0; p < K[g]; ++p)
      if (J[g][p] == w) {
        const float* src = delta[g] + p * D;
        for (int64_t d = 0; d < D; ++d) {
          out[d] += (double)src[d];
          if (absout) absout[d] += src[d] < 0 ? -(double)src[d] : (double)src[d];
        }
        ++n;
      }
  return n;
}

/*
 * Compression (Sec. 3.3): "multiply the FP32 tensor by a scaling
 * factor, F before down-casting" to FP16.  Reading R15: the product F*x is an
 * fp32 product (the tensor is FP32), the down-cast is IEEE binary16
 * round-to-nearest-even (through subnormals to +-0), and values beyond the
 * largest finite half saturate to +-65504.  q holds the binary16 bits.
 * The conversion is the compiler's _Float16 cast (IEEE RNE): a primitive.
 */
void oracle_compress(const float* x, int64_t n, float F, uint16_t* q) {
  for (int64_t i = 0; i < n; ++i) {
    float p = F * x[i];
    _Float16 h;
    if (p > 65504.0f)
      h = (_Float16)65504.0f;
    else if (p < -65504.0f)
      h = (_Float16)-65504.0f;
    else
      h = (_Float16)p;
    memcpy(q + i, &h, sizeof(h));
  }
}

/*
 * "up-cast the FP16 tensor to FP32 at the receiving end" and "divide again by
 * F after up-casting": x = fp32(half) / F, one fp32 division.
 */
void oracle_decompress(const uint16_t* q, int64_t n, float F, float* x) {
  for (int64_t i = 0; i < n; ++i) {
    _Float16 h;
    memcpy(&h, q + i, sizeof(h));
    x[i] = (float)h / F;
  }
}

/*
 * The receiving end's reduction with compression on (R15): the up-cast
 * tensors are FP32, so the sum over ranks is an fp32 sum, in rank
 * order.  out has n entries, overwritten.
 */
void oracle_sum_f32(const float* const* a, int G, int64_t n, float* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = 0.0f;
  for (int g = 0; g < G; ++g)
    for (int64_t i = 0; i < n; ++i) out[i] += a[g][i];
}

/*
 * Seeding (Sec. 3.2; reading R16).  The sampled-softmax
 * candidates of a GPU are S words drawn "randomly" (P:263-264, 1024 per GPU at
 * P:605); GPUs of one seed group share the seed and so draw the same words.
 * R16 fixes the draw: uniform without replacement = the first S distinct
 * values of the stream x_i = floor(u_i * V / 2^64), i = 0, 1, 2, ..., with
 * u_i = mix64(A + i) and A = mix64(seed ^ mix64(step)), where mix64 is the
 * SplitMix64 output function (state + golden gamma, two xor-shift-multiplies).
 */
uint64_t oracle_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* x_i of the stream above (one draw). */
uint32_t oracle_draw_one(uint64_t seed, uint64_t step, uint64_t i, uint64_t V) {
  uint64_t A = oracle_mix64(seed ^ oracle_mix64(step));
  uint64_t u = oracle_mix64(A + i);
  return (uint32_t)(((unsigned __int128)u * V) >> 64);
}

/* The first S distinct values of the stream, in stream order (plain linear
 * membership test).  Requires S <= V.  Returns the number of draws used. */
int64_t oracle_draw_samples(uint64_t seed, uint64_t step, int64_t S, uint64_t V, uint32_t* out) {
  int64_t n = 0, i = 0;
  while (n < S) {
    uint32_t x = oracle_draw_one(seed, step, (uint64_t)i, V);
    ++i;
    int seen = 0;
    for (int64_t j = 0; j < n; ++j)
      if (out[j] == x) { seen = 1; break; }
    if (!seen) out[n++] = x;
  }
  return i;
}

/*
 * Forward lookup ("A |V| x D embedding matrix projects the input K
 * token sequence into a dense K x D matrix"): out[p,:] = E[J[p],:]; an id >=
 * V (outside the matrix) gives a zero row.
 */
void oracle_lookup(const float* E, int64_t V, int64_t D, const uint32_t* J, int64_t K,
                   float* out) {
  for (int64_t p = 0; p < K; ++p)
    for (int64_t d = 0; d < D; ++d)
      out[p * D + d] = (int64_t)J[p] < V ? E[(int64_t)J[p] * D + d] : 0.0f;
}

/*
 * bfloat16 variant of the codec ("fp16 (and bf16)";
 * reading R15): down-cast = round-to-nearest-even of fp32(F * x) to the upper
 * 16 bits (8-bit exponent, 7-bit mantissa), saturating to +-(largest finite
 * bfloat16) = +-0x7F7F; up-cast = the 16 bits as the top of an fp32, then one
 * fp32 division by F.  Inputs are finite.
 */
void oracle_compress_bf16(const float* x, int64_t n, float F, uint16_t* q) {
  const float maxbf = 3.3895313892515355e38f; /* bits 0x7F7F0000 */
  for (int64_t i = 0; i < n; ++i) {
    float p = F * x[i];
    if (p > maxbf) p = maxbf;
    if (p < -maxbf) p = -maxbf;
    uint32_t u;
    memcpy(&u, &p, sizeof(u));
    uint32_t r = u + 0x7FFFu + ((u >> 16) & 1u); /* ties to even on the dropped half */
    q[i] = (uint16_t)(r >> 16);
  }
}

void oracle_decompress_bf16(const uint16_t* q, int64_t n, float F, float* x) {
  for (int64_t i = 0; i < n; ++i) {
    uint32_t u = (uint32_t)q[i] << 16;
    float v;
    memcpy(&v, &u, sizeof(v));
    x[i] = v / F;
  }
}
