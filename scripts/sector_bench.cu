// sector_bench.cu -- the practical roofline of random 32-byte-sector reads
// (the MaxEnt / output-row-bias / cache-probe access pattern):
// every thread reads independent 4-byte words at hashed positions of a table
// far larger than L2 (each read = one DRAM sector), plus the plain streaming
// copy bandwidth for comparison.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sector_bench scripts/sector_bench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

template <int ILP>
__global__ void k_random(const float *__restrict__ t, uint64_t mask, uint64_t reads_per_thread, float *out) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  float acc = 0.f;
  for (uint64_t i = 0; i < reads_per_thread; i += ILP) {
    float v[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) v[j] = __ldg(t + (mix(tid * 0x9E3779B97F4A7C15ull + i + j) & mask));
#pragma unroll
    for (int j = 0; j < ILP; ++j) acc += v[j];
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void k_copy(const float4 *__restrict__ a, float4 *__restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  const uint64_t words = 1ull << 28;                 // 1 GiB table of fp32 (like a 2^27..2^28 MaxEnt table)
  float *t, *out;
  cudaMalloc(&t, words * 4);
  cudaMalloc(&out, 64);
  cudaMemset(t, 0, words * 4);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = nsm * 8, threads = 256;
  const uint64_t rpt = 1024;
  float ms = 0;
  for (uint64_t tw : {1ull << 28, 1ull << 27, 1ull << 26}) {     // 1 GiB, 512 MiB (the 2^27 MaxEnt table), 256 MiB
    k_random<8><<<blocks, threads>>>(t, tw - 1, rpt, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_random<8><<<blocks, threads>>>(t, tw - 1, rpt, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double reads = 5.0 * blocks * threads * rpt;
    printf("{\"pattern\": \"random 4-B reads\", \"table_MiB\": %llu, \"reads_per_s\": %.4g, \"sector_GBps\": %.1f}\n",
           (unsigned long long)(tw * 4 >> 20), reads / (ms * 1e-3), reads * 32.0 / (ms * 1e-3) / 1e9);
  }
  // streaming copy (read + write bytes)
  const size_t n4 = words / 4 / 2;
  k_copy<<<nsm * 4, 512>>>(reinterpret_cast<float4 *>(t), reinterpret_cast<float4 *>(t) + n4, n4);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r)
    k_copy<<<nsm * 4, 512>>>(reinterpret_cast<float4 *>(t), reinterpret_cast<float4 *>(t) + n4, n4);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"pattern\": \"streaming copy\", \"GBps\": %.1f}\n", 5.0 * n4 * 32.0 / (ms * 1e-3) / 1e9);
  return 0;
}
