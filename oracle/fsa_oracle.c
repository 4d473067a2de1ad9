/*
 * fsa_oracle.c — CPU restatement of the reference FuseSampleAgg algorithm.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU baseline timer:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * load it.  The product path (paper_2511_13645_b200) never links or calls it.
 *
 * Parity is pinned: tests/test_oracle_golden.py checks every function here against golden
 * vectors produced by the reference itself (tests/golden/make_golden.py imports
 * /root/reference/pkg/src/fsa and runs its numba kernels), and against the live reference
 * when /root/reference is present.
 *
 * Every function cites the reference code it restates (paths relative to /root/reference):
 *   derive / splitmix / xorshift      pkg/src/fsa/rng.py:38-52,95-104; kernels.py:26-49
 *   reservoir (Vitter Algorithm R)    pkg/src/fsa/kernels.py:52-68
 *   sample_1hop / sample_2hop         pkg/src/fsa/kernels.py:87-120
 *   fused_1hop / fused_2hop           pkg/src/fsa/kernels.py:127-198
 *   backward (invert_targets +        pkg/src/fsa/kernels.py:296-338,
 *     scatter_from_grad, denominators) pkg/src/fsa/fused.py:191-255,290-299
 *
 * Floating point: sums start at +0.0 and run in slot order, divisions are IEEE; compiled with
 * -O2 -ffp-contract=off and without -ffast-math, matching numba's strict float semantics.
 * Parallelism: OpenMP over seeds / touched rows, exactly where the reference uses prange; the
 * per-row work is sequential, so results do not depend on the thread count
 * (kernels.py:1-5, parallel.py:3-7).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GOLDEN 0x9E3779B97F4A7C15ull
#define MIX1 0xBF58476D1CE4E5B9ull
#define MIX2 0x94D049BB133111EBull
#define ROOT_MULT 0xBF58476D1CE4E5B9ull
#define HOP_MULT 0x94D049BB133111EBull
#define INDEX_MULT 0xD6E8FEB86659FD93ull

/* rng.py:38-43 */
static inline uint64_t splitmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * MIX1;
  z = (z ^ (z >> 27)) * MIX2;
  return z ^ (z >> 31);
}

/* rng.py:46-52 */
static inline uint64_t xorshift64(uint64_t x) {
  x ^= x << 13;
  x ^= x >> 7;
  x ^= x << 17;
  return x;
}

/* rng.py:95-104 with the zero escape of rng.py:64-68 / kernels.py:41-49 */
uint64_t oracle_derive(uint64_t base, uint64_t root, uint64_t hop, uint64_t index) {
  uint64_t z = base + GOLDEN * (1ull + root * ROOT_MULT + hop * HOP_MULT + index * INDEX_MULT);
  uint64_t s = splitmix64(z);
  return s ? s : GOLDEN;
}

uint64_t oracle_splitmix64(uint64_t z) { return splitmix64(z); }

/* kernels.py:76-80 */
void oracle_xorshift_steps(uint64_t s, int64_t n, uint64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = s = xorshift64(s);
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int oracle_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* kernels.py:52-68 — Algorithm R over col[rowptr[u]:rowptr[u+1]]; returns the take. */
static inline int64_t reservoir(const int32_t* rowptr, const int32_t* col, int64_t node, int64_t k,
                                uint64_t state, int32_t* out) {
  const int64_t start = rowptr[node];
  const int64_t deg = (int64_t)rowptr[node + 1] - start;
  if (deg <= k) {
    for (int64_t i = 0; i < deg; ++i) out[i] = col[start + i];
    return deg;
  }
  for (int64_t i = 0; i < k; ++i) out[i] = col[start + i];
  for (int64_t i = k; i < deg; ++i) {
    state = xorshift64(state);
    const uint64_t j = state % (uint64_t)(i + 1);
    if (j < (uint64_t)k) out[j] = col[start + i];
  }
  return k;
}

/* kernels.py:87-97 (root_off = 0 is the reference; >0 = a shard of a larger batch) */
void oracle_sample_1hop(const int32_t* rowptr, const int32_t* col, const int64_t* seeds, int64_t B,
                        int64_t root_off, int64_t k, uint64_t base, int32_t* samples, int32_t* takes) {
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t i = 0; i < B; ++i) {
    int32_t* row = samples + i * k;
    const uint64_t st = oracle_derive(base, (uint64_t)(i + root_off), 0, 0);
    const int64_t take = reservoir(rowptr, col, seeds[i], k, st, row);
    for (int64_t j = take; j < k; ++j) row[j] = -1;
    takes[i] = (int32_t)take;
  }
}

/* kernels.py:99-120 */
void oracle_sample_2hop(const int32_t* rowptr, const int32_t* col, const int64_t* seeds, int64_t B,
                        int64_t root_off, int64_t k1, int64_t k2, uint64_t base, int32_t* s1,
                        int32_t* s2, int32_t* take1, int32_t* take2) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t r = 0; r < B; ++r) {
    int32_t* u_row = s1 + r * k1;
    const uint64_t st = oracle_derive(base, (uint64_t)(r + root_off), 1, 0);
    const int64_t t1 = reservoir(rowptr, col, seeds[r], k1, st, u_row);
    for (int64_t j = t1; j < k1; ++j) u_row[j] = -1;
    take1[r] = (int32_t)t1;
    for (int64_t j = 0; j < t1; ++j) {
      int32_t* w_row = s2 + (r * k1 + j) * k2;
      const uint64_t st2 = oracle_derive(base, (uint64_t)(r + root_off), 2, (uint64_t)j);
      const int64_t t2 = reservoir(rowptr, col, u_row[j], k2, st2, w_row);
      for (int64_t l = t2; l < k2; ++l) w_row[l] = -1;
      take2[r * k1 + j] = (int32_t)t2;
    }
    for (int64_t j = t1; j < k1; ++j) {
      take2[r * k1 + j] = 0;
      for (int64_t l = 0; l < k2; ++l) s2[(r * k1 + j) * k2 + l] = -1;
    }
  }
}

/* ---- fused forward: kernels.py:127-149 (1-hop) and 152-198 (2-hop) ------------------------ */
#define DEFINE_FUSED(T, SFX)                                                                       \
  void oracle_fused_1hop_##SFX(const int32_t* rowptr, const int32_t* col, const T* X, int64_t D,   \
                               const int64_t* seeds, int64_t B, int64_t root_off, int64_t k,       \
                               uint64_t base, int save, int32_t* samples, int32_t* takes, T* out) { \
    _Pragma("omp parallel")                                                                        \
    {                                                                                              \
      int32_t* scratch = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);                            \
      T* acc = (T*)malloc(sizeof(T) * (size_t)D);                                                  \
      _Pragma("omp for schedule(dynamic, 8)")                                                      \
      for (int64_t i = 0; i < B; ++i) {                                                            \
        int32_t* row = save ? samples + i * k : scratch;                                           \
        const uint64_t st = oracle_derive(base, (uint64_t)(i + root_off), 0, 0);                   \
        const int64_t take = reservoir(rowptr, col, seeds[i], k, st, row);                         \
        if (save) {                                                                                \
          for (int64_t j = take; j < k; ++j) row[j] = -1;                                          \
          takes[i] = (int32_t)take;                                                                \
        }                                                                                          \
        for (int64_t d = 0; d < D; ++d) acc[d] = (T)0;                                             \
        for (int64_t j = 0; j < take; ++j) {                                                       \
          const T* xr = X + (int64_t)row[j] * D;                                                   \
          for (int64_t d = 0; d < D; ++d) acc[d] += xr[d];                                         \
        }                                                                                          \
        const T den = (T)(take > 1 ? take : 1);                                                    \
        for (int64_t d = 0; d < D; ++d) out[i * D + d] = acc[d] / den;                             \
      }                                                                                            \
      free(scratch);                                                                               \
      free(acc);                                                                                   \
    }                                                                                              \
  }                                                                                                \
  void oracle_fused_2hop_##SFX(const int32_t* rowptr, const int32_t* col, const T* X, int64_t D,   \
                               const int64_t* seeds, int64_t B, int64_t root_off, int64_t k1,      \
                               int64_t k2, uint64_t base, int save, int32_t* s1, int32_t* s2,      \
                               int32_t* take1, int32_t* take2, T* out) {                           \
    _Pragma("omp parallel")                                                                        \
    {                                                                                              \
      int32_t* u_loc = (int32_t*)malloc(sizeof(int32_t) * (size_t)k1);                             \
      int32_t* w_loc = (int32_t*)malloc(sizeof(int32_t) * (size_t)k2);                             \
      T* acc = (T*)malloc(sizeof(T) * (size_t)D);                                                  \
      T* acc2 = (T*)malloc(sizeof(T) * (size_t)D);                                                 \
      _Pragma("omp for schedule(dynamic, 2)")                                                      \
      for (int64_t r = 0; r < B; ++r) {                                                            \
        int32_t* u_row = save ? s1 + r * k1 : u_loc;                                               \
        const uint64_t st = oracle_derive(base, (uint64_t)(r + root_off), 1, 0);                   \
        const int64_t t1 = reservoir(rowptr, col, seeds[r], k1, st, u_row);                        \
        if (save) {                                                                                \
          for (int64_t j = t1; j < k1; ++j) u_row[j] = -1;                                         \
          take1[r] = (int32_t)t1;                                                                  \
        }                                                                                          \
        for (int64_t d = 0; d < D; ++d) acc[d] = (T)0;                                             \
        for (int64_t j = 0; j < t1; ++j) {                                                         \
          int32_t* w_row = save ? s2 + (r * k1 + j) * k2 : w_loc;                                  \
          const uint64_t st2 = oracle_derive(base, (uint64_t)(r + root_off), 2, (uint64_t)j);      \
          const int64_t t2 = reservoir(rowptr, col, u_row[j], k2, st2, w_row);                     \
          if (save) {                                                                              \
            for (int64_t l = t2; l < k2; ++l) w_row[l] = -1;                                       \
            take2[r * k1 + j] = (int32_t)t2;                                                       \
          }                                                                                        \
          for (int64_t d = 0; d < D; ++d) acc2[d] = (T)0;                                          \
          for (int64_t l = 0; l < t2; ++l) {                                                       \
            const T* xr = X + (int64_t)w_row[l] * D;                                               \
            for (int64_t d = 0; d < D; ++d) acc2[d] += xr[d];                                      \
          }                                                                                        \
          const T den0 = (T)(t2 > 1 ? t2 : 1);                                                     \
          for (int64_t d = 0; d < D; ++d) acc[d] += acc2[d] / den0;                                \
        }                                                                                          \
        if (save) {                                                                                \
          for (int64_t j = t1; j < k1; ++j) {                                                      \
            take2[r * k1 + j] = 0;                                                                 \
            for (int64_t l = 0; l < k2; ++l) s2[(r * k1 + j) * k2 + l] = -1;                       \
          }                                                                                        \
        }                                                                                          \
        const T den1 = (T)(t1 > 1 ? t1 : 1);                                                       \
        for (int64_t d = 0; d < D; ++d) out[r * D + d] = acc[d] / den1;                            \
      }                                                                                            \
      free(u_loc);                                                                                 \
      free(w_loc);                                                                                 \
      free(acc);                                                                                   \
      free(acc2);                                                                                  \
    }                                                                                              \
  }

DEFINE_FUSED(float, f32)
DEFINE_FUSED(double, f64)

/* kernels.py:296-326 — counting sort of valid slots by target (serial, as the reference). */
static int invert_targets(const int32_t* ids, int64_t T, int64_t N, int64_t** touched_out,
                          int64_t* n_touched, int64_t** offsets_out, int64_t** order_out) {
  int64_t* offsets = (int64_t*)calloc((size_t)N + 1, sizeof(int64_t));
  if (!offsets) return 1;
  int64_t total = 0;
  for (int64_t t = 0; t < T; ++t) {
    const int32_t v = ids[t];
    if (v >= 0) {
      offsets[v + 1] += 1;
      total += 1;
    }
  }
  int64_t nt = 0;
  for (int64_t v = 0; v < N; ++v) {
    if (offsets[v + 1] > 0) nt += 1;
    offsets[v + 1] += offsets[v];
  }
  int64_t* touched = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nt > 0 ? nt : 1));
  int64_t ti = 0;
  for (int64_t v = 0; v < N; ++v)
    if (offsets[v + 1] > offsets[v]) touched[ti++] = v;
  int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
  memcpy(cursor, offsets, sizeof(int64_t) * (size_t)N);
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(total > 0 ? total : 1));
  for (int64_t t = 0; t < T; ++t) {
    const int32_t v = ids[t];
    if (v >= 0) order[cursor[v]++] = t;
  }
  free(cursor);
  *touched_out = touched;
  *n_touched = nt;
  *offsets_out = offsets;
  *order_out = order;
  return 0;
}

/* fused.py:191-255 + kernels.py:329-338.  `out` [N, D] is zero-filled first (fused.py:290-296).
 * 1-hop: denom = max(take, 1), stride = k.   2-hop: denom = max(t1,1)*max(t2,1) recomputed from
 * the -1 pattern, stride = k1*k2.  Returns 0, or 1 on allocation failure. */
#define DEFINE_BWD(T, SFX)                                                                         \
  static int scatter_##SFX(const T* grad_out, int64_t D, const int32_t* ids, int64_t Tn,           \
                           const T* denom_flat, int64_t stride, int64_t N, T* out) {               \
    int64_t *touched, *offsets, *order, nt;                                                        \
    if (invert_targets(ids, Tn, N, &touched, &nt, &offsets, &order)) return 1;                     \
    _Pragma("omp parallel for schedule(dynamic, 64)")                                              \
    for (int64_t ui = 0; ui < nt; ++ui) {                                                          \
      const int64_t v = touched[ui];                                                               \
      for (int64_t pos = offsets[v]; pos < offsets[v + 1]; ++pos) {                                \
        const int64_t t = order[pos];                                                              \
        const int64_t i = t / stride;                                                              \
        for (int64_t d = 0; d < D; ++d) out[v * D + d] += grad_out[i * D + d] / denom_flat[t];     \
      }                                                                                            \
    }                                                                                              \
    free(touched);                                                                                 \
    free(offsets);                                                                                 \
    free(order);                                                                                   \
    return 0;                                                                                      \
  }                                                                                                \
  int oracle_bwd_1hop_##SFX(const T* grad_out, int64_t B, int64_t D, const int32_t* samples,       \
                            const int32_t* takes, int64_t k, int64_t N, T* out) {                  \
    memset(out, 0, sizeof(T) * (size_t)N * (size_t)D);                                             \
    T* denom = (T*)malloc(sizeof(T) * (size_t)(B * k));                                            \
    for (int64_t i = 0; i < B; ++i)                                                                \
      for (int64_t j = 0; j < k; ++j) denom[i * k + j] = (T)(takes[i] > 1 ? takes[i] : 1);         \
    const int rc = scatter_##SFX(grad_out, D, samples, B * k, denom, k, N, out);                   \
    free(denom);                                                                                   \
    return rc;                                                                                     \
  }                                                                                                \
  int oracle_bwd_2hop_##SFX(const T* grad_out, int64_t B, int64_t D, const int32_t* s1,            \
                            const int32_t* s2, int64_t k1, int64_t k2, int64_t N, T* out) {        \
    memset(out, 0, sizeof(T) * (size_t)N * (size_t)D);                                             \
    T* denom = (T*)malloc(sizeof(T) * (size_t)(B * k1 * k2));                                      \
    for (int64_t r = 0; r < B; ++r) {                                                              \
      int64_t t1 = 0;                                                                              \
      for (int64_t j = 0; j < k1; ++j) t1 += s1[r * k1 + j] >= 0;                                  \
      if (t1 < 1) t1 = 1;                                                                          \
      for (int64_t j = 0; j < k1; ++j) {                                                           \
        int64_t t2 = 0;                                                                            \
        for (int64_t l = 0; l < k2; ++l) t2 += s2[(r * k1 + j) * k2 + l] >= 0;                    \
        if (t2 < 1) t2 = 1;                                                                        \
        const T den = (T)(t1 * t2);                                                                \
        for (int64_t l = 0; l < k2; ++l) denom[(r * k1 + j) * k2 + l] = den;                       \
      }                                                                                            \
    }                                                                                              \
    const int rc = scatter_##SFX(grad_out, D, s2, B * k1 * k2, denom, k1 * k2, N, out);            \
    free(denom);                                                                                   \
    return rc;                                                                                     \
  }

DEFINE_BWD(float, f32)
DEFINE_BWD(double, f64)
