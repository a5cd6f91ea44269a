// Micro-benchmark: one warp runs the search kernel's sort_radix / dedup_sort_rows.
#include <cstdio>
#include <vector>
#include <cstdint>
#include "search.cu"

__global__ void radix_kernel(unsigned long long* k, uint32_t* v, unsigned long long* k2, uint32_t* v2, uint32_t n) {
  __shared__ WarpSmem sm;
  sort_radix(k, v, k2, v2, n, 24, 7, &sm, threadIdx.x & 31);
}
__global__ void dedup_kernel(const uint32_t* src, uint32_t n, uint32_t* dst, unsigned long long* k, uint32_t* v,
                             unsigned long long* k2, uint32_t* v2, uint32_t* out) {
  __shared__ WarpSmem sm;
  uint32_t m = dedup_sort_rows(src, n, 4, dst, k, v, k2, v2, &sm, threadIdx.x & 31);
  if (threadIdx.x == 0) out[0] = m;
}

int main(int argc, char** argv) {
  const uint32_t n = argc > 1 ? atoi(argv[1]) : 14000;
  std::vector<unsigned long long> keys(n);
  std::vector<uint32_t> rows(n * 4);
  uint64_t s = 777;
  auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
  for (auto& x : keys) x = rnd() & 0x7fffffffffull;
  for (uint32_t t = 0; t < n; ++t) { uint32_t d = rnd() % 2000; for (int q = 0; q < 4; ++q) rows[t*4+q] = (uint32_t)(d * 2654435761u * (q + 1)); }
  unsigned long long *k, *k2; uint32_t *v, *v2, *src, *dst, *out;
  cudaMalloc(&k, 8 * n); cudaMalloc(&k2, 8 * n); cudaMalloc(&v, 4 * n); cudaMalloc(&v2, 4 * n);
  cudaMalloc(&src, 16 * n); cudaMalloc(&dst, 16 * n); cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(k, keys.data(), 8 * n, cudaMemcpyHostToDevice);
    cudaEventRecord(a);
    radix_kernel<<<1, 32>>>(k, v, k2, v2, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("radix n=%u %.3f ms (%s)\n", n, ms, cudaGetErrorString(cudaGetLastError()));
  }
  cudaMemcpy(src, rows.data(), 16 * n, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    dedup_kernel<<<1, 32>>>(src, n, dst, k, v, k2, v2, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    uint32_t m; cudaMemcpy(&m, out, 4, cudaMemcpyDeviceToHost);
    printf("dedup n=%u -> %u  %.3f ms (%s)\n", n, m, ms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
