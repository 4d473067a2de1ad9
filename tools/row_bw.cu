// Random-row HBM bandwidth probe: the access pattern of the gather (random rows read) and of the
// backward row writers (random rows written), independent of the operator.  Gives the practical
// ceiling the per-kernel roofline fractions should be read against.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/row_bw tools/row_bw.cu
//   gpurun_out/row_bw [rows]     -> one line per (pattern, row bytes): GB/s
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

// one warp per row group: lanes over 16-B chunks, ROWS rows in flight per lane
template <int ROWS>
__global__ void read_rows(const uint4* __restrict__ buf, const int* __restrict__ idx, int nrows,
                          int chunks, int64_t stride16, uint4* sink) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  uint32_t acc = 0;
  for (int r0 = w * ROWS; r0 < nrows; r0 += nw * ROWS) {
    for (int c = lane; c < chunks; c += 32) {
      uint4 x[ROWS];
#pragma unroll
      for (int u = 0; u < ROWS; ++u)
        x[u] = r0 + u < nrows ? __ldg(buf + (int64_t)idx[r0 + u] * stride16 + c) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < ROWS; ++u) acc ^= x[u].x ^ x[u].y ^ x[u].z ^ x[u].w;
    }
  }
  if (acc == 0x12345678u) sink[0] = make_uint4(acc, 0, 0, 0);
}

__global__ void write_rows(uint4* buf, const int* __restrict__ idx, int nrows, int chunks, int64_t stride16) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = w; r < nrows; r += nw) {
    const int64_t base = (int64_t)idx[r] * stride16;
    for (int c = lane; c < chunks; c += 32) buf[base + c] = make_uint4(r, c, 0, 0);
  }
}

int main(int argc, char** argv) {
  const int64_t want_rows = argc > 1 ? atoll(argv[1]) : 0;  // rows per pass (default ~256 MB)
  const int64_t total = 1ll << 30;  // 1 GiB table, far beyond L2
  uint4* buf;
  uint4* sink;
  CK(cudaMalloc(&buf, total));
  CK(cudaMalloc(&sink, 16));
  CK(cudaMemset(buf, 1, total));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  if (argc > 2) {  // MLP sweep: 400-B rows, rows in flight per lane x resident warps per SM
    const int rb = 400, nrows = (int)want_rows;
    const int64_t nslots = total / rb;
    std::vector<int> h(nrows);
    uint64_t s = 88172645463325252ull;
    for (int i = 0; i < nrows; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[i] = (int)(s % (uint64_t)nslots);
    }
    int* idx;
    CK(cudaMalloc(&idx, nrows * sizeof(int)));
    CK(cudaMemcpy(idx, h.data(), nrows * sizeof(int), cudaMemcpyHostToDevice));
    for (int wps : {8, 16, 28, 32, 48, 64}) {
      for (int rows : {4, 8, 10, 16}) {
        float best = 1e9f;
        for (int rep = 0; rep < 5; ++rep) {
          CK(cudaEventRecord(a));
          const int grid = sms * wps / 4;  // 128-thread CTAs
          if (rows == 4) read_rows<4><<<grid, 128>>>(buf, idx, nrows, rb / 16, rb / 16, sink);
          if (rows == 8) read_rows<8><<<grid, 128>>>(buf, idx, nrows, rb / 16, rb / 16, sink);
          if (rows == 10) read_rows<10><<<grid, 128>>>(buf, idx, nrows, rb / 16, rb / 16, sink);
          if (rows == 16) read_rows<16><<<grid, 128>>>(buf, idx, nrows, rb / 16, rb / 16, sink);
          CK(cudaEventRecord(b));
          CK(cudaEventSynchronize(b));
          float ms;
          CK(cudaEventElapsedTime(&ms, a, b));
          if (ms < best) best = ms;
        }
        printf("{\"warps_per_sm\": %d, \"rows_per_lane\": %d, \"inflight_KB_per_sm\": %.0f, \"ms\": %.4f, \"GBps\": %.1f}\n",
               wps, rows, wps * rows * 400 / 1024.0, best, (double)nrows * rb / (best * 1e-3) / 1e9);
      }
    }
    return 0;
  }
  const int row_bytes[] = {400, 512, 1216, 2048, 4096};
  for (int rb : row_bytes) {
    const int64_t stride = rb;  // rows packed, 16-B aligned
    const int64_t nslots = total / stride;
    const int nrows = (int)std::min<int64_t>(nslots, want_rows ? want_rows : (int64_t)(256ll << 20) / rb);
    std::vector<int> h(nrows);
    uint64_t s = 88172645463325252ull;
    for (int i = 0; i < nrows; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[i] = (int)(s % (uint64_t)nslots);
    }
    int* idx;
    CK(cudaMalloc(&idx, nrows * sizeof(int)));
    CK(cudaMemcpy(idx, h.data(), nrows * sizeof(int), cudaMemcpyHostToDevice));
    const int chunks = rb / 16;
    for (int pass = 0; pass < 2; ++pass) {
      float best = 1e9f;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(a));
        if (pass == 0) read_rows<8><<<sms * 8, 256>>>(buf, idx, nrows, chunks, stride / 16, sink);
        else write_rows<<<sms * 8, 256>>>(buf, idx, nrows, chunks, stride / 16);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
      }
      const double bytes = (double)nrows * rb;
      printf("{\"pattern\": \"random_row_%s\", \"row_bytes\": %d, \"rows\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n",
             pass == 0 ? "read" : "write", rb, nrows, best, bytes / (best * 1e-3) / 1e9);
    }
    CK(cudaFree(idx));
  }
  return 0;
}
