// Micro-benchmark: one warp runs the search kernel's antichain<W> on n synthetic rows.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2401_05039_b200/csrc scripts/micro/antichain_bench.cu
#include <cstdio>
#include <vector>
#include <cstdint>
#include "search.cu"

template <int W>
__global__ void bench_kernel(const uint32_t* src, uint32_t n, uint32_t* dst, uint32_t* out, int sorted) {
  const int lane = threadIdx.x & 31;
  uint32_t k = antichain<W>(src, n, dst, false, lane, sorted != 0);
  if (lane == 0) out[0] = k;
}

int main(int argc, char** argv) {
  const uint32_t n = argc > 1 ? atoi(argv[1]) : 8000;
  const int distinct = argc > 2 ? atoi(argv[2]) : 2000;
  const int W = 4;
  std::vector<uint32_t> rows(n * W);
  uint64_t s = 12345;
  auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (uint32_t)s; };
  std::vector<uint32_t> pool(distinct * W);
  for (auto& v : pool) v = rnd() & rnd() & rnd();  // sparse-ish rows
  for (uint32_t t = 0; t < n; ++t) {
    int d = rnd() % distinct;
    for (int q = 0; q < W; ++q) rows[t * W + q] = pool[d * W + q] & (rnd() | rnd());
  }
  uint32_t *dsrc, *ddst, *dout;
  cudaMalloc(&dsrc, n * W * 4); cudaMalloc(&ddst, n * W * 4); cudaMalloc(&dout, 4);
  cudaMemcpy(dsrc, rows.data(), n * W * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int sorted = 0; sorted < 1; ++sorted) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      bench_kernel<4><<<1, 32>>>(dsrc, n, ddst, dout, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      uint32_t k; cudaMemcpy(&k, dout, 4, cudaMemcpyDeviceToHost);
      printf("n=%u W=%d kept=%u  %.3f ms (%s)\n", n, W, k, ms, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
