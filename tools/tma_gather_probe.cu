// Kernel-only times: every kernel folds its blocks' first start / last end (%globaltimer) into
// g_span, so launch latency is not in the numbers (each run follows a 512 MiB L2 flush).
//
// Random-row gather through TMA tile::gather4 (cp.async.bulk.tensor.2d ... tile::gather4: four
// rows of a 2-D tensor map per instruction into shared memory, no registers held in flight)
// versus register loads, on the gather's access pattern: 153,600 random 400-B rows of a
// 2.45 M x 100 fp32 table (products shape), summed in groups of 10 rows (one second-hop slot).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/tma_probe tools/tma_gather_probe.cu -lcuda
//   gpurun_out/tma_probe            -> one line per (variant, CTAs/SM, stages): us, GB/s
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ unsigned long long g_span[2];
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct Span {
  __device__ Span() { if (threadIdx.x == 0) atomicMin(&g_span[0], gt()); }
  __device__ ~Span() { __syncthreads(); if (threadIdx.x == 0) atomicMax(&g_span[1], gt()); }
};

constexpr int D = 100;
constexpr int ROWB = D * 4;
constexpr int GROUP = 10;         // rows per slot mean
constexpr int ROWS_PER_STAGE = 20;  // 5 gather4 ops, two slots
constexpr int G4F = 416;            // floats per gather4 destination (4 rows, padded to 128 B)
constexpr int STAGEF = ROWS_PER_STAGE / 4 * G4F;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" ::"r"(smem_u32(b)), "r"(parity));
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int r0, int r1,
                                            int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}

// persistent: CTA b takes stages b, b + grid, ...; warp 0 lane 0 produces, the CTA's threads
// (one per column) consume: sum each slot's 10 rows, write the mean
__global__ void __launch_bounds__(128) k_tma(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                                             int nstage_total, int S, float* __restrict__ out) {
  Span span_;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + S;
  float* buf = reinterpret_cast<float*>(sm + 1024);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, blockDim.x);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int my = (nstage_total - blockIdx.x + gridDim.x - 1) / gridDim.x;  // stages of this CTA
  if (tid == 0) {  // prologue: fill the ring
    for (int i = 0; i < min(S, my); ++i) {
      const int g = blockIdx.x + i * gridDim.x;
      const int* ix = idx + (size_t)g * ROWS_PER_STAGE;
      float* dst = buf + (size_t)i * STAGEF;
      mbar_expect_tx(full + i, ROWS_PER_STAGE * ROWB);
      for (int q = 0; q < ROWS_PER_STAGE; q += 4)
        tma_gather4(dst + q / 4 * G4F, &tm, full + i, 0, ix[q], ix[q + 1], ix[q + 2], ix[q + 3]);
    }
  }
  for (int i = 0; i < my; ++i) {
    const int s = i % S;
    const uint32_t par = (i / S) & 1;
    mbar_wait(full + s, par);
    const float* src = buf + (size_t)s * STAGEF;
    const int g = blockIdx.x + i * gridDim.x;
    if (tid < D) {
      for (int h = 0; h < ROWS_PER_STAGE / GROUP; ++h) {
        float a = 0.f;
#pragma unroll
        for (int l = 0; l < GROUP; ++l) {
          const int row = h * GROUP + l;
          a += src[row / 4 * G4F + row % 4 * D + tid];
        }
        out[((size_t)g * (ROWS_PER_STAGE / GROUP) + h) * D + tid] = a * 0.1f;
      }
    }
    mbar_arrive(empty + s);
    if (tid == 0 && i + S < my) {  // refill this stage once every thread has consumed it
      mbar_wait(empty + s, par);
      const int g2 = blockIdx.x + (i + S) * gridDim.x;
      const int* ix = idx + (size_t)g2 * ROWS_PER_STAGE;
      float* dst = buf + (size_t)s * STAGEF;
      mbar_expect_tx(full + s, ROWS_PER_STAGE * ROWB);
      for (int q = 0; q < ROWS_PER_STAGE; q += 4)
        tma_gather4(dst + q / 4 * G4F, &tm, full + s, 0, ix[q], ix[q + 1], ix[q + 2], ix[q + 3]);
    }
  }
}

// register loads: warp per slot group, lanes over 16-B chunks (25 per row), R rows in flight
template <int R>
__global__ void k_ldg(const float4* __restrict__ X, const int* __restrict__ idx, int nslots, float* __restrict__ out) {
  Span span_;
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int g = w; g < nslots; g += nw) {
    const int* ix = idx + (size_t)g * GROUP;
    if (lane < D / 4) {
      float4 a = make_float4(0, 0, 0, 0);
      for (int l0 = 0; l0 < GROUP; l0 += R) {
        float4 x[R];
#pragma unroll
        for (int u = 0; u < R; ++u) x[u] = __ldg(X + (size_t)ix[l0 + u] * (D / 4) + lane);
#pragma unroll
        for (int u = 0; u < R; ++u) {
          a.x += x[u].x; a.y += x[u].y; a.z += x[u].z; a.w += x[u].w;
        }
      }
      reinterpret_cast<float4*>(out)[(size_t)g * (D / 4) + lane] = a;
    }
  }
}

// random row writes: warp per row, lanes over 16-byte chunks; `cols16` chunks written per row at
// a row stride of `stride16` chunks (400-B rows dense: 25 / 25; padded stride: 25 / 28; whole
// 64-byte bursts: 28 / 28)
__global__ void k_write(uint4* __restrict__ G, const int* __restrict__ idx, int nrows, int cols16, int stride16) {
  Span span_;
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = w; r < nrows; r += nw) {
    uint4* row = G + (size_t)idx[r] * stride16;
    for (int c = lane; c < cols16; c += 32) row[c] = make_uint4(r, c, 0, 0);
  }
}

int main() {
  const int64_t N = 2449029;
  const int nrows = 153600;
  float* X;
  int* idx;
  float* out;
  CK(cudaMalloc(&X, (size_t)N * ROWB));
  CK(cudaMalloc(&idx, nrows * sizeof(int)));
  CK(cudaMalloc(&out, (size_t)nrows / GROUP * ROWB));
  CK(cudaMemset(X, 0, (size_t)N * ROWB));
  std::vector<int> h(nrows);
  uint64_t z = 88172645463325252ull;
  for (auto& v : h) {
    z ^= z << 13; z ^= z >> 7; z ^= z << 17;
    v = (int)(z % N);
  }
  CK(cudaMemcpy(idx, h.data(), nrows * sizeof(int), cudaMemcpyHostToDevice));
  char* flush;
  const size_t FL = 512ull << 20;
  CK(cudaMalloc(&flush, FL));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));

  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)N};
  cuuint64_t strides[1] = {(cuuint64_t)ROWB};
  cuuint32_t box[2] = {(cuuint32_t)D, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, strides, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    const char* s = nullptr;
    cuGetErrorString(cr, &s);
    printf("tensor map: %s\n", s ? s : "?");
    return 1;
  }
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const double bytes = (double)nrows * ROWB;
  double bytes_now = bytes;
  auto timeit = [&](auto&& launch, const char* name, int p1, int p2) {
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaMemset(flush, rep, FL));
      CK(cudaDeviceSynchronize());
      unsigned long long init[2] = {~0ull, 0ull};
      CK(cudaMemcpyToSymbol(g_span, init, sizeof(init)));
      CK(cudaEventRecord(a));
      launch();
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaGetLastError());
      unsigned long long sp[2];
      CK(cudaMemcpyFromSymbol(sp, g_span, sizeof(sp)));
      const float ms = (float)((sp[1] - sp[0]) * 1e-6);
      if (rep) best = ms < best ? ms : best;
    }
    printf("{\"variant\": \"%s\", \"p1\": %d, \"p2\": %d, \"us\": %.2f, \"gbs\": %.0f}\n", name, p1, p2, best * 1e3,
           bytes_now / (best * 1e-3) / 1e9);
  };
  const int nst = nrows / ROWS_PER_STAGE;
  for (int ctas : {1, 2, 3, 4}) {
    for (int S : {4, 8, 12, 16}) {
      const size_t smem = 1024 + (size_t)S * STAGEF * 4;
      if (smem * ctas > 220 * 1024) continue;
      CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      timeit([&] { k_tma<<<sms * ctas, 128, smem>>>(tm, idx, nst, S, out); }, "tma_gather4", ctas, S);
    }
  }
  for (int wps : {16, 32, 48, 64}) {
    timeit([&] { k_ldg<5><<<sms * wps / 8, 256>>>(reinterpret_cast<const float4*>(X), idx, nrows / GROUP, out); },
           "ldg_R5", wps, 5);
    timeit([&] { k_ldg<10><<<sms * wps / 8, 256>>>(reinterpret_cast<const float4*>(X), idx, nrows / GROUP, out); },
           "ldg_R10", wps, 10);
  }
  // random row writes into a 2.45 M-row gradient: dense 400-B rows, 448-B stride writing 400 B,
  // 448-B stride writing whole 64-byte bursts (bytes counted: the bytes each variant stores)
  uint4* G;
  CK(cudaMalloc(&G, (size_t)N * 448));
  for (auto v : {std::make_pair(25, 25), std::make_pair(25, 28), std::make_pair(28, 28)}) {
    bytes_now = (double)nrows * v.first * 16;
    timeit([&] { k_write<<<sms * 8, 256>>>(G, idx, nrows, v.first, v.second); }, "write_rows", v.first * 16,
           v.second * 16);
  }
  return 0;
}
