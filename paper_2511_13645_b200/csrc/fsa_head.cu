// SAGE-mean classifier head of the training step (reference: pkg/src/fsa/train.py:111-160), fp32.
//
//   k_head_rows    one CTA per R seed rows: concat = [X[seed] | x_agg] staged in shared memory,
//                  hidden = ReLU(concat W1 + b1), logits = hidden W2 + b2, the max-shifted softmax
//                  cross-entropy per row, dlogits = (softmax - onehot) / B, dhidden =
//                  (dlogits W2^T) * (hidden > 0), and d_x_agg = dhidden W1[D:]^T (the rows the
//                  replay backward scatters). W2 sits in shared memory; W1 streams through a ring
//                  of cp.async-filled chunk buffers with HEAD_S - 1 chunks in flight (once for the
//                  forward, once for d_x_agg), so the L2 round trips overlap.
//   The kernel also writes [concat | 1] and [hidden | 1] and dlogits for the caller's two
//   parameter GEMMs ([concat | 1]^T dhidden = [dW1; db1], [hidden | 1]^T dlogits = [dW2; db2]) and
//   the per-row losses.
//
// Labels outside [0, C) make the row's loss and gradients NaN, so the step's finiteness check
// discards the update (the reference raises an IndexError there).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "../../include/fsa_b200.h"

namespace {

constexpr int HEAD_THREADS = 256;
constexpr int HEAD_R = 4;    // seed rows per CTA (256 CTAs at B = 1024, two per SM)
constexpr int HEAD_KC = 16;  // W1 rows per staged chunk
constexpr int HEAD_S = 3;    // chunk buffers in the cp.async ring (HEAD_S - 1 chunks in flight)

#ifdef HEAD_TRACE  // per-CTA phase timestamps (instrumented builds only: -DHEAD_TRACE, tools/head_trace.py)
__device__ unsigned long long g_head_trace[1024][9];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define HEAD_TRACE_START() \
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_head_trace[blockIdx.x][0] = gtimer()
#define HEAD_MARK(i) \
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_head_trace[blockIdx.x][(i) + 1] = gtimer()
#else
#define HEAD_TRACE_START()
#define HEAD_MARK(i)
#endif

__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

struct HeadArgs {
  const float* X; int64_t xs; const int64_t* seeds; const float* agg; int64_t as; const int64_t* labels;
  int B, D, H, C;
  const float* W1; const float* b1; const float* W2; const float* b2;
  float* gagg; int64_t gs;
  float* cat1; float* hid1; float* dhid; float* dlog; float* lrow;  // outputs for the parameter GEMMs
};

// chunk c of rows [base, base + total) of W1 (row length H, H % 4 == 0) into ring slot c % HEAD_S via
// 16-byte cp.async, one commit group per chunk (an empty group past the end keeps the count uniform)
__device__ __forceinline__ void stage_w1(float* ring, const float* W1, int H, int base, int total, int c) {
  const int k0 = c * HEAD_KC, n = min(HEAD_KC, total - k0);
  if (n > 0) {
    float* buf = ring + (c % HEAD_S) * HEAD_KC * H;
    const int q = H >> 2, cnt = n * q;
    const float* src = W1 + (int64_t)(base + k0) * H;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) cpa16(buf + i * 4, src + i * 4);
  }
  cpa_commit();
}

template <int R>
__device__ __forceinline__ void fma_rows(const float* col, float w, float (&acc)[R]) {
#pragma unroll
  for (int q = 0; q < R / 4; ++q) {
    const float4 x = *reinterpret_cast<const float4*>(col + 4 * q);
    acc[4 * q + 0] = fmaf(x.x, w, acc[4 * q + 0]);
    acc[4 * q + 1] = fmaf(x.y, w, acc[4 * q + 1]);
    acc[4 * q + 2] = fmaf(x.z, w, acc[4 * q + 2]);
    acc[4 * q + 3] = fmaf(x.w, w, acc[4 * q + 3]);
  }
}

// Row-indexed shared arrays are stored transposed ([k][R], [j][R], [c][R]) so one pair of 16-byte
// broadcast loads feeds R = 8 FMAs.
template <int R>
__global__ void __launch_bounds__(HEAD_THREADS) k_head_rows(HeadArgs a) {
  static_assert(R % 4 == 0, "float4 loads along the transposed columns");
  extern __shared__ __align__(16) float sm[];
  const int D = a.D, D2 = 2 * D, H = a.H, C = a.C;
  float* ring = sm;                              // [HEAD_S][KC][H] W1 chunk ring
  float* w2 = ring + HEAD_S * HEAD_KC * H;       // [H][C]
  float* ht = w2 + ((H * C + 3) & ~3);           // hidden^T [H][R]
  float* dht = ht + H * R;                       // dhidden^T [H][R]
  float* dl = dht + H * R;                       // logits [R][C]
  float* dlt = dl + ((R * C + 3) & ~3);          // dlogits^T [C][R]
  float* part = dlt + C * R;                     // logit partials [4][C][R]
  float* cct = part + 4 * C * R;                 // concat^T [2D][R]
  const int r0 = blockIdx.x * R;
  const int nr = min(R, a.B - r0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  HEAD_TRACE_START();

  {  // W2 (whole) and the first W1 chunks in flight while the concat rows load
    const int q = (H * C) >> 2;
    for (int i = threadIdx.x; i < q; i += blockDim.x) cpa16(w2 + i * 4, a.W2 + i * 4);
    cpa_commit();
  }
  const int nch = (D2 + HEAD_KC - 1) / HEAD_KC;
  for (int c = 0; c < HEAD_S - 1; ++c) stage_w1(ring, a.W1, H, 0, D2, c);
  for (int i = threadIdx.x; i < R * D2; i += blockDim.x) {
    const int r = i / D2, k = i - r * D2;
    float v = 0.f;
    if (r < nr) {
      const int64_t row = r0 + r;
      v = k < D ? a.X[a.seeds[row] * a.xs + k] : a.agg[row * a.as + (k - D)];
    }
    cct[k * R + r] = v;
  }

  HEAD_MARK(0);
  // hidden = ReLU(concat W1 + b1): thread j keeps R accumulators per column it owns
  constexpr int JMAX = 2;  // H <= JMAX * blockDim.x
  float acc[JMAX][R];
#pragma unroll
  for (int u = 0; u < JMAX; ++u)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[u][r] = 0.f;
  for (int c = 0; c < nch; ++c) {
    const int k0 = c * HEAD_KC, n = min(HEAD_KC, D2 - k0);
    stage_w1(ring, a.W1, H, 0, D2, c + HEAD_S - 1);  // into the slot read in iteration c - 1
    cpa_wait<HEAD_S - 1>();
    __syncthreads();
    const float* w = ring + (c % HEAD_S) * HEAD_KC * H;
#pragma unroll
    for (int u = 0; u < JMAX; ++u) {
      const int j = threadIdx.x + u * blockDim.x;
      if (j < H) {
#pragma unroll 4
        for (int t = 0; t < n; ++t) {
          fma_rows<R>(cct + (k0 + t) * R, w[t * H + j], acc[u]);
        }
      }
    }
    __syncthreads();
  }
  HEAD_MARK(1);
  // the d_x_agg pass streams W1[D:] through the same ring: start its first chunks now
  const int nch2 = (D + HEAD_KC - 1) / HEAD_KC;
  for (int c = 0; c < HEAD_S - 1; ++c) stage_w1(ring, a.W1, H, D, D, c);
#pragma unroll
  for (int u = 0; u < JMAX; ++u) {
    const int j = threadIdx.x + u * blockDim.x;
    if (j < H) {
      const float bj = a.b1[j];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float h = acc[u][r] + bj;
        ht[j * R + r] = h > 0.f ? h : 0.f;
      }
    }
  }
  __syncthreads();

  HEAD_MARK(2);
  // logits = hidden W2 + b2: thread (g, c) sums j in [g*H/4, (g+1)*H/4) for all R rows; the four
  // partials are added in g order
  const int hq = (H + 3) >> 2;
  for (int i = threadIdx.x; i < 4 * C; i += blockDim.x) {
    const int g = i / C, c = i - g * C;
    float s[R];
#pragma unroll
    for (int r = 0; r < R; ++r) s[r] = 0.f;
    const int j1 = min(H, (g + 1) * hq);
    for (int j = g * hq; j < j1; ++j) {
      fma_rows<R>(ht + j * R, w2[j * C + c], s);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) part[(g * C + c) * R + r] = s[r];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < R * C; i += blockDim.x) {
    const int r = i / C, c = i - r * C;
    const float v = ((part[c * R + r] + part[(C + c) * R + r]) + part[(2 * C + c) * R + r]) + part[(3 * C + c) * R + r];
    dl[i] = v + a.b2[c];
  }
  __syncthreads();

  HEAD_MARK(3);
  for (int r = warp; r < R; r += nw) {  // softmax cross-entropy, dlogits (train.py:123-139)
    const float* L = dl + r * C;
    if (r >= nr) {  // padding rows: keep them finite and inert
      for (int c = lane; c < C; c += 32) dlt[c * R + r] = 0.f;
      continue;
    }
    float m = -INFINITY;
    for (int c = lane; c < C; c += 32) m = fmaxf(m, L[c]);
    m = warp_max(m);
    float s = 0.f;
    for (int c = lane; c < C; c += 32) s += expf(L[c] - m);
    s = warp_sum(s);
    const float lse = logf(s);
    const int64_t y = a.labels[r0 + r];
    const bool bad = y < 0 || y >= C;
    const float ly = bad ? NAN : (L[bad ? 0 : y] - m) - lse;
    const float fB = (float)a.B;
    for (int c = lane; c < C; c += 32) {
      const float p = expf(L[c] - m) / s;
      dlt[c * R + r] = bad ? NAN : (p - (c == y ? 1.f : 0.f)) / fB;
    }
    if (lane == 0) a.lrow[r0 + r] = -ly;
  }
  __syncthreads();

  HEAD_MARK(4);
  for (int j = threadIdx.x; j < H; j += blockDim.x) {  // dhidden = (dlogits W2^T) * (hidden > 0)
    float s[R];
#pragma unroll
    for (int r = 0; r < R; ++r) s[r] = 0.f;
    for (int c = 0; c < C; ++c) {
      fma_rows<R>(dlt + c * R, w2[j * C + c], s);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) dht[j * R + r] = s[r] * (ht[j * R + r] > 0.f ? 1.f : 0.f);
  }
  // (the chunk loop's first barrier orders these dht writes before their reads)

  HEAD_MARK(5);
  for (int c = 0; c < nch2; ++c) {  // d_x_agg[r][k] = sum_j dhidden[r][j] W1[D + k][j]
    const int k0 = c * HEAD_KC, n = min(HEAD_KC, D - k0);
    stage_w1(ring, a.W1, H, D, D, c + HEAD_S - 1);
    cpa_wait<HEAD_S - 1>();
    __syncthreads();
    const float* w = ring + (c % HEAD_S) * HEAD_KC * H;
    for (int t = warp; t < n; t += nw) {
      float s[R];
#pragma unroll
      for (int r = 0; r < R; ++r) s[r] = 0.f;
      for (int j = lane; j < H; j += 32) {
        fma_rows<R>(dht + j * R, w[t * H + j], s);
      }
      float mine = 0.f;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float v = warp_sum(s[r]);
        if (lane == r) mine = v;
      }
      if (lane < nr) a.gagg[(int64_t)(r0 + lane) * a.gs + k0 + t] = mine;
    }
    __syncthreads();
  }

  HEAD_MARK(6);
  const int D21 = D2 + 1, H1 = H + 1;  // [concat | 1], [hidden | 1], dhidden, dlogits rows
  for (int i = threadIdx.x; i < nr * D21; i += blockDim.x) {
    const int r = i / D21, k = i - r * D21;
    a.cat1[(int64_t)(r0 + r) * D21 + k] = k < D2 ? cct[k * R + r] : 1.f;
  }
  for (int i = threadIdx.x; i < nr * H1; i += blockDim.x) {
    const int r = i / H1, j = i - r * H1;
    a.hid1[(int64_t)(r0 + r) * H1 + j] = j < H ? ht[j * R + r] : 1.f;
  }
  for (int i = threadIdx.x; i < nr * H; i += blockDim.x) {
    const int r = i / H, j = i - r * H;
    a.dhid[(int64_t)r0 * H + i] = dht[j * R + r];
  }
  for (int i = threadIdx.x; i < nr * C; i += blockDim.x) {
    const int r = i / C, c = i - r * C;
    a.dlog[(int64_t)r0 * C + i] = dlt[c * R + r];
  }
  HEAD_MARK(7);
}

inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

size_t rows_smem(int D, int H, int C) {
  const size_t hc = ((size_t)H * C + 3) & ~(size_t)3, rc = ((size_t)HEAD_R * C + 3) & ~(size_t)3;
  return ((size_t)HEAD_S * HEAD_KC * H + hc + (size_t)HEAD_R * 2 * H + rc + (size_t)C * HEAD_R * 5 +
          (size_t)HEAD_R * 2 * D) * sizeof(float);
}

}  // namespace

extern "C" size_t fsa_sage_head_ws_bytes(int64_t B, int32_t D, int32_t H, int32_t C) {
  if (B <= 0 || D <= 0 || H <= 0 || C <= 0) return 0;
  return align_up((size_t)B * (2 * D + 1) * 4) + align_up((size_t)B * (H + 1) * 4) + align_up((size_t)B * H * 4) +
         align_up((size_t)B * C * 4) + align_up((size_t)B * 4);
}

extern "C" size_t fsa_sage_head_smem_bytes(int32_t D, int32_t H, int32_t C) {
  if (D <= 0 || H <= 0 || C <= 0) return 0;
  return rows_smem(D, H, C);
}

extern "C" int fsa_sage_head_rows(const float* X, int64_t x_stride, const int64_t* seeds, const float* agg,
                                  int64_t agg_stride, const int64_t* labels, int64_t B, int32_t D, int32_t H,
                                  int32_t C, const float* W1, const float* b1, const float* W2, const float* b2,
                                  float* grad_agg, int64_t grad_stride, void* ws, size_t ws_bytes, void* stream) {
  if (B <= 0 || B > (1 << 30) || D <= 0 || H <= 0 || C <= 0 || x_stride < D || agg_stride < D ||
      grad_stride < D || H > 2 * HEAD_THREADS)
    return FSA_ERR_ARG;
  if (!X || !seeds || !agg || !labels || !W1 || !b1 || !W2 || !b2 || !grad_agg || !ws) return FSA_ERR_ARG;
  if ((H & 3) || (reinterpret_cast<uintptr_t>(W1) & 15) || (reinterpret_cast<uintptr_t>(W2) & 15))
    return FSA_ERR_ALIGN;
  if (ws_bytes < fsa_sage_head_ws_bytes(B, D, H, C)) return FSA_ERR_WORKSPACE;
  const size_t smem = rows_smem(D, H, C);
  if (smem > 227 * 1024) return FSA_ERR_ARG;
  char* p = static_cast<char*>(ws);
  HeadArgs a{X, x_stride, seeds, agg, agg_stride, labels, (int)B, D, H, C, W1, b1, W2, b2, grad_agg, grad_stride};
  a.cat1 = reinterpret_cast<float*>(p);
  p += align_up((size_t)B * (2 * D + 1) * 4);
  a.hid1 = reinterpret_cast<float*>(p);
  p += align_up((size_t)B * (H + 1) * 4);
  a.dhid = reinterpret_cast<float*>(p);
  p += align_up((size_t)B * H * 4);
  a.dlog = reinterpret_cast<float*>(p);
  p += align_up((size_t)B * C * 4);
  a.lrow = reinterpret_cast<float*>(p);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaFuncSetAttribute(k_head_rows<HEAD_R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return FSA_ERR_CUDA;
  k_head_rows<HEAD_R><<<(unsigned)((B + HEAD_R - 1) / HEAD_R), HEAD_THREADS, smem, st>>>(a);
  e = cudaGetLastError();
  return e == cudaSuccess ? FSA_OK : FSA_ERR_CUDA;
}

// ---------------------------------------------------------------------------------------------
// AdamW of the training step (reference: pkg/src/fsa/train.py:163-184), fp32 parameters, as two
// grid-wide kernels instead of multi-tensor launches that give each 64 K-element chunk one CTA:
//   k_adamw_check   every gradient element finite? (flag); the last CTA to finish advances the
//                   device step count by `ok` and derives the bias corrections in double, as the
//                   reference does (it raises before incrementing, so a skipped step does not count)
//   k_adamw_update  p -= lr*wd*p; m = b1*m + (1-b1)*g; v = b2*v + (1-b2)*g*g;
//                   p -= lr*(m/bc1)/(sqrt(v/bc2)+eps), each operation rounded in fp32 in the
//                   reference's order (no contraction); nothing is written when a gradient is
//                   non-finite.
namespace {

constexpr int ADAMW_MAX = 8;
constexpr int ADAMW_THREADS = 256;

struct AdamwArgs {
  int n;
  float* p[ADAMW_MAX];
  const float* g[ADAMW_MAX];
  float* m[ADAMW_MAX];
  float* v[ADAMW_MAX];
  int64_t off[ADAMW_MAX + 1];  // prefix sums of the tensor sizes
  double* t;                   // device step count
  unsigned char* ok;           // device bool
  unsigned* flag;              // [0] non-finite seen, [1] CTAs done
  float* coef;                 // [0] bc1, [1] bc2 (fp32, as the reference's weak scalars)
  double beta1, beta2;
  float lr_wd, one_m_b1, one_m_b2, b1f, b2f, lr, eps;
};

__device__ __forceinline__ int adamw_tensor(const AdamwArgs& a, int64_t i) {
  int k = 0;
  while (k + 1 < a.n && i >= a.off[k + 1]) ++k;
  return k;
}

__global__ void __launch_bounds__(ADAMW_THREADS) k_adamw_check(AdamwArgs a) {
  const int64_t total = a.off[a.n];
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = adamw_tensor(a, i);
    bad |= !isfinite(a.g[k][i - a.off[k]]);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&a.flag[0], 1u);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&a.flag[1], 1u) == gridDim.x - 1) {  // last CTA: every flag update is visible
      __threadfence();
      const bool ok = atomicAdd(&a.flag[0], 0u) == 0u;
      a.flag[0] = 0u;  // leave the scratch zero for the next call
      a.flag[1] = 0u;
      const double t = *a.t + (ok ? 1.0 : 0.0);
      *a.t = t;
      *a.ok = ok ? 1 : 0;
      a.coef[0] = (float)(1.0 - pow(a.beta1, t));
      a.coef[1] = (float)(1.0 - pow(a.beta2, t));
    }
  }
}

__global__ void __launch_bounds__(ADAMW_THREADS) k_adamw_update(AdamwArgs a) {
  if (!*a.ok) return;
  const float bc1 = a.coef[0], bc2 = a.coef[1];
  const int64_t total = a.off[a.n];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = adamw_tensor(a, i);
    const int64_t e = i - a.off[k];
    const float g = a.g[k][e];
    float p = a.p[k][e];
    p = __fsub_rn(p, __fmul_rn(a.lr_wd, p));
    const float m = __fadd_rn(__fmul_rn(a.m[k][e], a.b1f), __fmul_rn(a.one_m_b1, g));
    const float v = __fadd_rn(__fmul_rn(a.v[k][e], a.b2f), __fmul_rn(a.one_m_b2, __fmul_rn(g, g)));
    const float den = __fadd_rn(__fsqrt_rn(__fdiv_rn(v, bc2)), a.eps);
    p = __fsub_rn(p, __fdiv_rn(__fmul_rn(a.lr, __fdiv_rn(m, bc1)), den));
    a.m[k][e] = m;
    a.v[k][e] = v;
    a.p[k][e] = p;
  }
}

}  // namespace

extern "C" size_t fsa_adamw_ws_bytes(void) { return 16; }

extern "C" int fsa_adamw_step(int n_tensors, float* const* params, const float* const* grads, float* const* exp_avg,
                              float* const* exp_avg_sq, const int64_t* sizes, double* step_count, double lr,
                              double beta1, double beta2, double weight_decay, double eps, unsigned char* ok_out,
                              void* ws, size_t ws_bytes, void* stream) {
  if (n_tensors <= 0 || n_tensors > ADAMW_MAX || !params || !grads || !exp_avg || !exp_avg_sq || !sizes ||
      !step_count || !ok_out || !ws)
    return FSA_ERR_ARG;
  if (ws_bytes < fsa_adamw_ws_bytes()) return FSA_ERR_WORKSPACE;
  AdamwArgs a{};
  a.n = n_tensors;
  a.off[0] = 0;
  for (int k = 0; k < n_tensors; ++k) {
    if (!params[k] || !grads[k] || !exp_avg[k] || !exp_avg_sq[k] || sizes[k] < 0) return FSA_ERR_ARG;
    a.p[k] = params[k];
    a.g[k] = grads[k];
    a.m[k] = exp_avg[k];
    a.v[k] = exp_avg_sq[k];
    a.off[k + 1] = a.off[k] + sizes[k];
  }
  a.t = step_count;
  a.ok = ok_out;
  a.flag = static_cast<unsigned*>(ws);
  a.coef = reinterpret_cast<float*>(static_cast<char*>(ws) + 8);
  a.beta1 = beta1;
  a.beta2 = beta2;
  // the reference's scalars: python floats meeting float32 arrays (numpy weak scalars -> fp32)
  a.lr_wd = (float)(lr * weight_decay);
  a.one_m_b1 = (float)(1.0 - beta1);
  a.one_m_b2 = (float)(1.0 - beta2);
  a.b1f = (float)beta1;
  a.b2f = (float)beta2;
  a.lr = (float)lr;
  a.eps = (float)eps;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t total = a.off[n_tensors];
  // one element per thread up to 8 CTAs per SM of a 148-SM part: the loops are latency-bound
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(148 * 8, (total + ADAMW_THREADS - 1) /
                                                                                      ADAMW_THREADS));
  k_adamw_check<<<grid, ADAMW_THREADS, 0, st>>>(a);
  k_adamw_update<<<grid, ADAMW_THREADS, 0, st>>>(a);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FSA_OK : FSA_ERR_CUDA;
}

#ifdef HEAD_TRACE
extern "C" int fsa_head_trace_read(unsigned long long* host, int nblocks) {
  return cudaMemcpyFromSymbol(host, g_head_trace, sizeof(unsigned long long) * 9 * (size_t)nblocks) == cudaSuccess ? 0 : 4;
}
#endif
