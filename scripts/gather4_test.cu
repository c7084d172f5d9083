// gather4_test.cu -- checks the shared-memory image of a TMA tile::gather4
// load (4 arbitrary rows of a 2D bf16 tensor, 128-byte swizzle) against the
// swizzle rule the MMA descriptors assume (16-byte chunk c of row r at chunk
// c ^ (r % 8) of a 1024-byte atom), for tensor-map boxes {64, 1} and {64, 4}.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o gather4_test scripts/gather4_test.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k(const __grid_constant__ CUtensorMap map, int r0, int r1, int r2, int r3, int col,
                  uint16_t *out) {
  __shared__ __align__(1024) uint16_t buf[8 * 64 * 4];
  __shared__ __align__(8) uint64_t bar;
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar), sd = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(512) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(sd),
        "l"((uint64_t)&map), "r"(sb), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(sb)
        : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * 64; i += blockDim.x) out[i] = buf[i];
}

int main() {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiled enc = (EncodeTiled)p;
  const int R = 64, C = 256;
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 1000 + c);
  uint16_t *d, *o;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&o, 4 * 64 * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  const int rows[4] = {5, 41, 2, 63}, col = 64;
  for (int boxr : {1, 4}) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R}, strides[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)boxr}, es[2] = {1, 1};
    CUresult e = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (e != CUDA_SUCCESS) { printf("box {64,%d}: encode failed %d\n", boxr, (int)e); continue; }
    cudaMemset(o, 0, 512);
    k<<<1, 128>>>(m, rows[0], rows[1], rows[2], rows[3], col, o);
    cudaError_t ce = cudaDeviceSynchronize();
    if (ce != cudaSuccess) { printf("box {64,%d}: launch error %s\n", boxr, cudaGetErrorString(ce)); return 1; }
    std::vector<uint16_t> out(256);
    cudaMemcpy(out.data(), o, 512, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 4; ++r)
      for (int c = 0; c < 64; ++c) {
        const int chunk = c / 8, within = c % 8;
        const int pos = r * 64 + ((chunk ^ (r % 8)) * 8) + within;
        if (out[pos] != h[rows[r] * C + col + c]) ++bad;
      }
    printf("box {64,%d}: gather4 + swizzle128 image %s (%d mismatches)\n", boxr, bad ? "WRONG" : "ok", bad);
  }
  return 0;
}
