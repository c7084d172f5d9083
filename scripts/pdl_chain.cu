// pdl_chain.cu -- cost of a kernel boundary in the cache front: a chain of K
// dependent kernels (512 blocks x 256 threads, one coalesced load + store per
// thread, like k_qcache .. k_commit at 131k queries) launched plain and with
// programmatic dependent launch (griddepcontrol).  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl_chain scripts/pdl_chain.cu
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_step(const unsigned *in, unsigned *out, unsigned n, int pdl) {
  if (pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i] + 1u;
}

static void launch(int pdl, const unsigned *in, unsigned *out, unsigned n, cudaStream_t s) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = (n + 255) / 256;
  cfg.blockDim = 256;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_step, in, out, n, pdl);
}

int main() {
  const unsigned n = 131072;
  unsigned *a, *b;
  cudaMalloc(&a, n * 4);
  cudaMalloc(&b, n * 4);
  cudaMemset(a, 0, n * 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int pdl = 0; pdl < 2; ++pdl) {
    for (int K : {1, 2, 4, 8, 16}) {
      for (int w = 0; w < 3; ++w)
        for (int k = 0; k < K; ++k) launch(pdl, k & 1 ? b : a, k & 1 ? a : b, n, s);
      cudaStreamSynchronize(s);
      const int R = 50;
      cudaEventRecord(e0, s);
      for (int r = 0; r < R; ++r)
        for (int k = 0; k < K; ++k) launch(pdl, k & 1 ? b : a, k & 1 ? a : b, n, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"pdl\": %d, \"kernels\": %d, \"us_per_kernel\": %.2f}\n", pdl, K, ms * 1e3 / (R * K));
    }
  }
  return 0;
}
