// k_small.cu -- the whole query step of a SMALL frame in ONE launch
// (SURVEY 8(a5) "Small-Q path" / 7 step 9; north_star: a GEMV path where the
// batch does not fill tensor-core tiles).
//
// The paper's frames are small: ~197 rows per frame exchange (P:160-161,
// P:186-189), 256 queries per frame at the moderate config.  Run as the
// ~10-kernel chain of the large-batch path, such a frame costs ~50 us of
// kernel boundaries and dependent launches (measured: 47-54 us per frame,
// scripts/latency_probe.py, profiles/latency_r2.jsonl) for well under a
// microsecond of memory traffic.  Here one cooperative persistent kernel
// (one CTA per SM, co-resident by construction) runs every step with grid
// barriers (three) where the multi-kernel path has kernel boundaries; the
// cache front (n <= 512 queries) runs in ONE CTA with block barriers, which
// are ~20x cheaper than grid barriers (measured per phase: ~4 us with grid
// barriers, profiles/small_phases_r2.txt):
//
//   A  (a2) LM-query cache probe + claim          qcache_query   (cache.cuh)  } CTA 0 alone, block
//   B  (a3) owner resolution, hidden-cache claim  hcache_query                } barriers between; the
//   C  (a4) flags + exclusive scan                scan_flag / scan_store      } other CTAs pull their
//   D  (a4) commit: handles, slots, records       commit_query                } GEMV weights into L1
//   E  (a7) result write + counters               final_query    (warp-collective)
//      (a6) NCE + MaxEnt scores                   score_quad     (score.cuh)
//      (a5) GEMV phase 1                          gemv1_item     (gemv.cuh)
//   F  (a5) GEMV phase 2; same-call duplicates take their owner's score
//   G  (a1) codes of the new states               gemv_encode (encode.cuh)
//
// Every decision is the same device function the multi-kernel path runs, in
// the same claim / barrier / read order, so results are bit-identical to that
// path with the GEMV GRU kernels (tests/test_gpu_small.py).
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "cache.cuh"
#include "gemv.cuh"
#include "score.cuh"

namespace rnnlm_small {
using namespace rnnlm_dev;
using namespace rnnlm_gemv;

constexpr int SMALL_THREADS = 256;
#ifndef RNNLM_SMALL_CTAS
#define RNNLM_SMALL_CTAS 148
#endif
constexpr int SI = 2;                  // scan items per thread
constexpr uint32_t MAX_N = SMALL_THREADS * SI;
static_assert(MAX_N >= RNNLM_GEMV_AUTO_MAX_QUERIES, "the fused kernel takes every AUTO-path GEMV call");

// Software grid barrier over the co-resident CTAs: bar[0] arrivals, bar[1]
// generation.  Release: each CTA's writes are fenced before it arrives;
// acquire: the generation is read with ld.acquire after the last arrival.
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
#ifndef RNNLM_SMALL_SLEEP
#define RNNLM_SMALL_SLEEP 0
#endif
__device__ __forceinline__ void grid_sync(uint32_t *bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t gen = ld_acquire_u32(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (ld_acquire_u32(bar + 1) == gen) {
        if (RNNLM_SMALL_SLEEP) __nanosleep(RNNLM_SMALL_SLEEP);
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// (a4) flags and the exclusive (non-QHIT, MISS) scan of all n <= MAX_N
// queries by one CTA.
__device__ __forceinline__ void block_scan(const Params &P, const CallArgs &A, uint32_t n, bool bad) {
  __shared__ unsigned long long s_warp[SMALL_THREADS / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t q0 = threadIdx.x * SI;
  unsigned long long v[SI], tsum = 0;
#pragma unroll
  for (int i = 0; i < SI; ++i) {
    v[i] = q0 + i < n ? scan_flag(P, A, q0 + i, bad) : 0ull;
    tsum += v[i];
  }
  unsigned long long inc = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  unsigned long long run = 0;
  for (int i = 0; i < wid; ++i) run += s_warp[i];
  run += inc - tsum;
#pragma unroll
  for (int i = 0; i < SI; ++i) {
    if (q0 + i < n) scan_store(P, A, q0 + i, n, bad, run, v[i]);
    run += v[i];
  }
}

template <typename WT, int ACT, int CELL>
__global__ void __launch_bounds__(SMALL_THREADS, 1)
    k_small(Params P, CallArgs A, GemvArgs g, uint32_t *bar, uint32_t rb1, uint32_t rb2,
            unsigned long long *prof) {
  // prof (diagnostics, RNNLM_SMALL_PROF): %globaltimer of CTA 0 after every phase
  auto stamp = [&](int i) {
    if (prof && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      prof[i] = t;
    }
  };
  stamp(0);
  const uint32_t n = call_n(A);
  const uint32_t tid = blockIdx.x * SMALL_THREADS + threadIdx.x, nthr = gridDim.x * SMALL_THREADS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t gw = tid >> 5, ngw = nthr >> 5;
  const uint32_t nb1 = g.H / U1, nb2 = g.H / U2;
  if (blockIdx.x == 0) {
    // A-D: the cache front of all n <= MAX_N queries by CTA 0 alone; its
    // block barriers stand in for the kernel boundaries between claiming and
    // reading an owner (global atomics + __syncthreads: every access before
    // the barrier is visible to the whole CTA after it)
    if (threadIdx.x == 0) P.counts[3] = 0u;
    for (uint32_t q = threadIdx.x; q < n; q += SMALL_THREADS) qcache_query(P, A, q);   // (a2)
    __syncthreads();
    stamp(1);
    const bool bad = P.counts[2] != 0u;
    for (uint32_t q = threadIdx.x; q < n; q += SMALL_THREADS) hcache_query(P, A, q);   // (a3)
    __syncthreads();
    stamp(2);
    if (n == 0 && threadIdx.x == 0) { P.counts[0] = 0u; P.counts[1] = 0u; }
    block_scan(P, A, n, bad);                                                            // (a4)
    __syncthreads();
    stamp(3);
    for (uint32_t q = threadIdx.x; q < n; q += SMALL_THREADS) commit_query(P, A, q, n);
  } else {
    // meanwhile: pull this CTA's phase-1 GEMV weight rows into L1 (CTAs >= 2
    // take the GEMV items in phase E, see below)
    const uint32_t SC = gridDim.x >= 8 ? 2u : 1u;
    if (blockIdx.x >= SC)
      for (uint32_t j = blockIdx.x - SC; j < nb1 * rb1; j += gridDim.x - SC) gemv1_prefetch<WT, CELL>(g, j % nb1);
  }
  grid_sync(bar);
  stamp(4);
  // E: (a7) result write, (a6) scores, (a5) GEMV phase 1
  // the first SC CTAs write results and score, the others run the GEMV, so
  // neither waits behind the other's dependent loads
  const uint32_t total = P.counts[0], Q = P.counts[1];
  const uint32_t SC = gridDim.x >= 8 ? 2u : 1u;
  if (blockIdx.x < SC || gridDim.x == 1) {
    const uint32_t w0 = blockIdx.x * (SMALL_THREADS / 32) + warp, nw0 = SC * (SMALL_THREADS / 32);
    for (uint32_t base = w0 * 32; base < n; base += nw0 * 32) final_query(P, A, base + lane, n);
    for (uint32_t base = w0 * 4; base < total; base += nw0 * 4) score_quad(P, A, base, total);
  }
  if (blockIdx.x >= SC || gridDim.x == 1) {
    const uint32_t c0 = gridDim.x == 1 ? 0u : blockIdx.x - SC, nc = gridDim.x == 1 ? 1u : gridDim.x - SC;
    for (uint32_t j = c0; j < nb1 * rb1; j += nc)
      gemv1_item<WT, ACT, CELL>(g, Q, j % nb1, j / nb1, rb1, warp, SMALL_THREADS / 32);
  }
  grid_sync(bar);
  stamp(5);
  // F: (a5) GEMV phase 2; duplicates of this call's new queries take their owner's score
  for (uint32_t j = blockIdx.x; j < nb2 * rb2; j += gridDim.x)
    gemv2_item<WT, ACT, CELL>(g, Q, j % nb2, j / nb2, rb2, warp, SMALL_THREADS / 32);
  const uint32_t nd = P.counts[3];
  for (uint32_t i = tid; i < nd; i += nthr) {
    const uint32_t q = P.dup_list[i];
    A.score[q] = A.score[P.aux[q]];
  }
  if (!g.cache) {
    if (tid == 0) P.counts[2] = 0u;
    return;
  }
  grid_sync(bar);
  stamp(6);
  // G: (a1) codes of the new states; the bad-batch flag is cleared for the next call
  gemv_encode(g, Q, gw, ngw);
  if (tid == 0) P.counts[2] = 0u;
  __syncthreads();
  stamp(7);
}

}  // namespace rnnlm_small

namespace rnnlm_host {
using namespace rnnlm_small;

int gemv_args(void *state, const Params &P, rnnlm_gemv::GemvArgs *out, int *act);

template <typename WT, int ACT, int CELL>
static cudaError_t launch_small_t(const Params &P, const CallArgs &A, const rnnlm_gemv::GemvArgs &g, uint32_t *bar,
                                  uint32_t grid, uint32_t rb1, uint32_t rb2, cudaStream_t s) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = SMALL_THREADS;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  static unsigned long long *prof = nullptr;
  static const bool want = getenv("RNNLM_SMALL_PROF") != nullptr;
  if (want && !prof) { cudaMalloc(&prof, 8 * sizeof(unsigned long long)); cudaMemset(prof, 0, 64); }
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_small<WT, ACT, CELL>, P, A, g, bar, rb1, rb2, prof);
  if (want && e == cudaSuccess) {        // diagnostics: phase durations of this call to stderr
    unsigned long long h[8];
    cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "[k_small prof] grid=%u us:", grid);
    for (int i = 1; i < 8; ++i) fprintf(stderr, " %.2f", (h[i] - h[i - 1]) * 1e-3);
    fprintf(stderr, " total %.2f\n", (h[7] - h[0]) * 1e-3);
  }
  return e;
}

uint32_t small_max_queries() { return MAX_N; }

// One launch for the whole step of a call with A.n <= MAX_N queries.
int launch_small(const Params &P, const CallArgs &A, void *gemv_state, uint32_t *bar, int num_sms,
                 cudaStream_t s) {
  rnnlm_gemv::GemvArgs g;
  int act = 0;
  if (gemv_args(gemv_state, P, &g, &act) != 0) return -1;
  // CTAs (<= one per SM, co-resident); GEMV work items: unit blocks x row
  // blocks (~ one per CTA).  RNNLM_SMALL_GRID overrides (A/B).
  static const int grid_env = getenv("RNNLM_SMALL_GRID") ? atoi(getenv("RNNLM_SMALL_GRID")) : 0;
  uint32_t grid = grid_env > 0 ? (uint32_t)grid_env : (uint32_t)RNNLM_SMALL_CTAS;
  if (grid > (uint32_t)num_sms) grid = (uint32_t)num_sms;
  const uint32_t nb1 = P.H / U1, nb2 = P.H / U2, rmax = (A.n + 7) / 8;
  uint32_t rb1 = (grid + nb1 - 1) / nb1, rb2 = (grid + nb2 - 1) / nb2;
  rb1 = rb1 < rmax ? rb1 : rmax; rb2 = rb2 < rmax ? rb2 : rmax;
  rb1 = rb1 ? rb1 : 1; rb2 = rb2 ? rb2 : 1;
  const int cell = (int)P.cell;
  cudaError_t e;
  if (act == ACT_BF16) {
    e = cell == 0 ? launch_small_t<__nv_bfloat16, ACT_BF16, 0>(P, A, g, bar, grid, rb1, rb2, s)
        : cell == 1 ? launch_small_t<__nv_bfloat16, ACT_BF16, 1>(P, A, g, bar, grid, rb1, rb2, s)
                    : launch_small_t<__nv_bfloat16, ACT_BF16, 2>(P, A, g, bar, grid, rb1, rb2, s);
  } else if (act == ACT_TF32) {
    e = cell == 0 ? launch_small_t<float, ACT_TF32, 0>(P, A, g, bar, grid, rb1, rb2, s)
        : cell == 1 ? launch_small_t<float, ACT_TF32, 1>(P, A, g, bar, grid, rb1, rb2, s)
                    : launch_small_t<float, ACT_TF32, 2>(P, A, g, bar, grid, rb1, rb2, s);
  } else {
    e = cell == 0 ? launch_small_t<float, ACT_F32, 0>(P, A, g, bar, grid, rb1, rb2, s)
        : cell == 1 ? launch_small_t<float, ACT_F32, 1>(P, A, g, bar, grid, rb1, rb2, s)
                    : launch_small_t<float, ACT_F32, 2>(P, A, g, bar, grid, rb1, rb2, s);
  }
  return e == cudaSuccess ? 1 : -1;
}
}  // namespace rnnlm_host
