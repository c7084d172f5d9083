// umma_bench.cu -- standalone mainloop microbenchmark for the GRU contraction
// shape (not product code): C[M, N] = A[M, K] . B[N, K]^T, bf16 -> fp32 in TMEM,
// persistent, warp-specialised, M x N tiles of 128 x 256 (one CTA,
// cta_group::1) or 256 x 256 (CTA pair, cta_group::2, each CTA loads its 128
// A rows and half of the B tile, both TMA loads signal the leader's barrier).
// The epilogue reads the accumulator and writes one row sum per (row, N-tile)
// (checked against a CPU fp64 reference on sampled rows).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_bench scripts/umma_bench.cu -lcuda
//   ./umma_bench M N K
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int A_BYTES = BM * BK * 2;

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cl(uint32_t cl_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <int PAIR>
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1) {
  if constexpr (PAIR == 2)
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"((uint64_t)map), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"((uint64_t)map), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
template <int PAIR>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  if constexpr (PAIR == 2)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
}
template <int PAIR>
__device__ __forceinline__ void commit(uint32_t bar) {
  if constexpr (PAIR == 2)
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
                 "h"((uint16_t)3)
                 : "memory");
  else
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int PAIR, int ST, bool G = false>
__global__ void __launch_bounds__(192, 1)
    kbench(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int M, int N,
           int K, float *out, const int *gidx = nullptr) {
  constexpr int BH = BN / PAIR;                // B rows this CTA loads
  constexpr int B_BYTES = BH * BK * 2;
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t *sA = sm, *sB = sm + ST * A_BYTES;
  uint64_t *full = (uint64_t *)(sB + ST * B_BYTES), *empty = full + ST, *tfull = empty + ST, *tempty = tfull + 2;
  uint32_t *tbase_s = (uint32_t *)(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR == 2 ? cta_rank() : 0;
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 4 * PAIR); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (PAIR == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tbase_s)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tbase_s)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if constexpr (PAIR == 2) cluster_sync();
  const uint32_t tb = *tbase_s;
  const long long clk0 = clock64();
  const int mt = M / (BM * PAIR), nt = N / BN, KC = K / BK;
  const int ntiles = mt * nt;
  const int unit = blockIdx.x / PAIR, nunits = gridDim.x / PAIR;
  // barrier addresses in the leader CTA (shared::cluster window)
  const uint32_t full_l = PAIR == 2 ? mapa(su32(full), 0) : su32(full);
  const uint32_t tempty_l = PAIR == 2 ? mapa(su32(tempty), 0) : su32(tempty);

  if (warp == 0 && G) {
    // gathered A: lane l issues the tile::gather4 of rows 4l..4l+3 of every stage
    int stage = 0;
    uint32_t ph = 0;
    for (int t = unit; t < ntiles; t += nunits) {
      const int m = t / nt, j = t % nt;
      const int m0 = m * BM, n0 = j * BN;
      const int4 r = *reinterpret_cast<const int4 *>(gidx + m0 + 4 * lane);
      for (int kc = 0; kc < KC; ++kc) {
        if (lane == 0) {
          mbar_wait(su32(&empty[stage]), ph ^ 1);
          mbar_expect_tx(su32(&full[stage]), A_BYTES + B_BYTES);
        }
        __syncwarp();
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su32(sA + stage * A_BYTES) + 512 * lane),
            "l"((uint64_t)&mapA), "r"(full_l + stage * 8), "r"(kc * BK), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w)
            : "memory");
        if (lane == 0) tma2d<PAIR>(su32(sB + stage * B_BYTES), &mapB, full_l + stage * 8, kc * BK, n0);
        if (++stage == ST) { stage = 0; ph ^= 1; }
      }
    }
  } else if (warp == 0 && lane == 0) {
    int stage = 0;
    uint32_t ph = 0;
    for (int t = unit; t < ntiles; t += nunits) {
      const int m = t / nt, j = t % nt;
      const int m0 = m * BM * PAIR + rank * BM, n0 = j * BN + rank * BH;
      for (int kc = 0; kc < KC; ++kc) {
        mbar_wait(su32(&empty[stage]), ph ^ 1);
        if (leader) mbar_expect_tx(su32(&full[stage]), PAIR * (A_BYTES + B_BYTES));
        tma2d<PAIR>(su32(sA + stage * A_BYTES), &mapA, full_l + stage * 8, kc * BK, m0);
        tma2d<PAIR>(su32(sB + stage * B_BYTES), &mapB, full_l + stage * 8, kc * BK, n0);
        if (++stage == ST) { stage = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1 && leader) {
    int stage = 0;
    uint32_t ph = 0;
    int it = 0;
    const uint32_t id = idesc(BM * PAIR, BN);
    for (int t = unit; t < ntiles; t += nunits, ++it) {
      const int acc = it & 1;
      mbar_wait(su32(&tempty[acc]), ((it >> 1) & 1) ^ 1);
      fence_after();
      for (int kc = 0; kc < KC; ++kc) {
        mbar_wait(su32(&full[stage]), ph);
        fence_after();
        if (lane == 0) {
          const uint32_t a0 = su32(sA + stage * A_BYTES), b0 = su32(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) mma<PAIR>(tb + acc * BN, sdesc(a0 + 32 * k), sdesc(b0 + 32 * k), id, (kc | k) != 0);
          commit<PAIR>(su32(&empty[stage]));
          if (kc == KC - 1) commit<PAIR>(su32(&tfull[acc]));
        }
        __syncwarp();
        if (++stage == ST) { stage = 0; ph ^= 1; }
      }
    }
  } else if (warp >= 2) {
    const int q = warp & 3;
    int it = 0;
    for (int t = unit; t < ntiles; t += nunits, ++it) {
      const int m = t / nt, j = t % nt;
      const int acc = it & 1;
      mbar_wait(su32(&tfull[acc]), (it >> 1) & 1);
      fence_after();
      float s = 0.f;
      for (int c = 0; c < BN; c += 16) {
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(tb + acc * BN + ((uint32_t)(q * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; ++i) s += __uint_as_float(r[i]);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR == 2) mbar_arrive_cl(tempty_l + acc * 8);
        else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&tempty[acc])) : "memory");
      }
      const int row = m * BM * PAIR + rank * BM + q * 32 + lane;
      out[(size_t)row * nt + j] = s;
    }
  }
  fence_before();
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[(size_t)M * (N / BN)] = (float)(clock64() - clk0);
  if constexpr (PAIR == 2) cluster_sync();
  if (warp == 1) {
    fence_after();
    if constexpr (PAIR == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tb));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
  }
}

typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static void make_map(CUtensorMap *m, void *base, uint64_t inner, uint64_t outer, uint32_t box_outer) {
  static EncodeTiled enc = nullptr;
  if (!enc) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    enc = (EncodeTiled)p;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t es[2] = {1, 1};
  if (enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    fprintf(stderr, "tensor map failed\n");
    exit(1);
  }
}

template <int PAIR, int ST, bool G = false>
static void run(const char *name, int M, int N, int K, __nv_bfloat16 *dA, __nv_bfloat16 *dB, float *dout,
                const std::vector<float> &hA, const std::vector<float> &hB, int nsm, const int *gidx = nullptr,
                int table_rows = 0, const std::vector<int> *hidx = nullptr) {
  CUtensorMap mA, mB;
  if (G) make_map(&mA, dA, K, table_rows, 1);
  else make_map(&mA, dA, K, M, BM);
  make_map(&mB, dB, K, N, BN / PAIR);
  const size_t smem = 1024 + ST * (A_BYTES + (BN / PAIR) * BK * 2) + 256;
  CK(cudaFuncSetAttribute(kbench<PAIR, ST, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = PAIR;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((nsm / PAIR) * PAIR);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaMemset(dout, 0, ((size_t)M * (N / BN) + 1) * 4));
  for (int i = 0; i < 3; ++i) CK(cudaLaunchKernelEx(&cfg, kbench<PAIR, ST, G>, mA, mB, M, N, K, dout, gidx));
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int R = 20;
  cudaEventRecord(e0);
  for (int i = 0; i < R; ++i) CK(cudaLaunchKernelEx(&cfg, kbench<PAIR, ST, G>, mA, mB, M, N, K, dout, gidx));
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= R;
  std::vector<float> out((size_t)M * (N / BN) + 1);
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  const double cycles = out[(size_t)M * (N / BN)];
  // per-cycle efficiency: ideal cycles = MACs per SM / 4096 (8192 flop/clk/SM dense bf16)
  const double ideal = 2.0 * M * N * K / 8192.0 / nsm;
  double maxerr = 0;
  for (int s = 0; s < 64; ++s) {
    const int row = (int)(((long long)s * 7919) % M), j = s % (N / BN);
    double ref = 0;
    for (int n = j * BN; n < j * BN + BN; ++n)
      for (int k = 0; k < K; ++k) {
        const size_t ar = G ? (size_t)(*hidx)[row] : (size_t)row;
        ref += (double)hA[ar * K + k] * hB[(size_t)n * K + k];
      }
    maxerr = fmax(maxerr, fabs(ref - out[(size_t)row * (N / BN) + j]));
  }
  const double tf = 2.0 * M * N * K / (ms * 1e-3) / 1e12;
  printf("{\"variant\": \"%s\", \"M\": %d, \"N\": %d, \"K\": %d, \"us\": %.2f, \"tflops\": %.1f, \"maxerr\": %.3g, "
         "\"cycles_cta0\": %.0f, \"clock_ghz\": %.3f, \"per_cycle_eff\": %.3f}\n",
         name, M, N, K, ms * 1e3, tf, maxerr, cycles, cycles / (ms * 1e-3) / 1e9, ideal / cycles);
}

int main(int argc, char **argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 15360, N = argc > 2 ? atoi(argv[2]) : 3072,
            K = argc > 3 ? atoi(argv[3]) : 2048;
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  std::vector<float> hA((size_t)M * K), hB((size_t)N * K);
  std::vector<__nv_bfloat16> bA(hA.size()), bB(hB.size());
  uint64_t x = 88172645463325252ull;
  auto rnd = [&]() {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    return (float)((x >> 40) & 0xFFFF) / 65536.0f - 0.5f;
  };
  for (size_t i = 0; i < hA.size(); ++i) { bA[i] = __float2bfloat16(rnd()); hA[i] = __bfloat162float(bA[i]); }
  for (size_t i = 0; i < hB.size(); ++i) { bB[i] = __float2bfloat16(rnd() * 0.1f); hB[i] = __bfloat162float(bB[i]); }
  __nv_bfloat16 *dA, *dB;
  float *dout;
  CK(cudaMalloc(&dA, bA.size() * 2));
  CK(cudaMalloc(&dB, bB.size() * 2));
  CK(cudaMalloc(&dout, ((size_t)M * (N / BN) + 1) * 4));
  CK(cudaMemcpy(dA, bA.data(), bA.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, bB.data(), bB.size() * 2, cudaMemcpyHostToDevice));
  run<1, 4>("one-cta st4", M, N, K, dA, dB, dout, hA, hB, nsm);
  {
    // gathered A: M random rows of the same A table (indices a permutation-free random draw)
    std::vector<int> idx(M);
    for (int i = 0; i < M; ++i) idx[i] = (int)(((unsigned long long)i * 2654435761ull + 12345) % (unsigned long long)M);
    int *didx;
    CK(cudaMalloc(&didx, M * 4));
    CK(cudaMemcpy(didx, idx.data(), M * 4, cudaMemcpyHostToDevice));
    run<1, 4, true>("one-cta st4 gather4-A", M, N, K, dA, dB, dout, hA, hB, nsm, didx, M, &idx);
  }
  run<2, 4>("pair st4", M, N, K, dA, dB, dout, hA, hB, nsm);
  run<2, 6>("pair st6", M, N, K, dA, dB, dout, hA, hB, nsm);
  return 0;
}
