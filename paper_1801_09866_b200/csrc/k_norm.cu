// k_norm.cu -- SURVEY 8(f)-2: the exact log-normaliser that NCE avoids.
//
// "In order to guarantee that the scores calculated at the output layer of an
// RNNLM are valid probabilities, they need to be normalized ... a highly
// computationally intensive task considering the vocabulary size V";
// NCE lets the decoder use unnormalised scores.  This computes, for n
// stored histories (session, handle), what that normalisation would be:
//
//   log Z = log sum_{v < V} exp(s_v),
//   s_v   = Theta_v . h + b_v + sum_{k=1..K} maxent[idx_k(ctx, v)]
//
// (the combined score of step a6 for EVERY word; SPEC exact_log_prob
// S:201-209), so exact log-probabilities are score - log Z.
//
// B200 mapping.  The NCE part is a dense [n, H] x [H, V] contraction: a
// persistent tcgen05 kernel (M = 128 histories, N = 256 words, K = H) whose
// epilogue adds the bias and the MaxEnt terms and folds its 128 x 256 scores
// into per-row online log-sum-exp partials (max, sum) -- the [n, V] score
// matrix never exists in memory.  The A operand is the state split into two
// bf16 halves, h = hi + lo (lo = bf16(h - hi)), both multiplied with the bf16
// output rows (two MMAs per K-step), so the contraction carries ~16
// significant bits of h instead of bf16's 8 at no cost that matters here.
// Output rows that are not bf16-exact are split the same way, Theta = Theta_hi
// + Theta_lo, and a third MMA adds h_hi . Theta_lo (k_norm_tc<true>; the
// dropped h_lo . Theta_lo is ~2^-18 relative): the normaliser then carries
// ~16 significant bits of both operands in every math mode.
// The MaxEnt terms: idx_k(v) = (alpha_k v + beta_k) mod M with
// alpha_k = 237967^(k-1) and beta_k fixed by the context (the S:177
// recurrence unrolled; M is a power of two, so mod M is a mask and the
// unrolling is exact), order 1 (beta = 0) folded into a per-word bias
// b_v + maxent[v mod M]; orders >= 2 are random 4-byte gathers from the 2^m
// table, (K-1) per (history, word) -- these, not the GEMM, bound the kernel
// at realistic V.  A last kernel combines the partials
// of each row in a fixed order (deterministic).
#include <cuda.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "rnnlm_impl.cuh"
#include "tc_common.cuh"

namespace rnnlm_norm {
using namespace rnnlm_dev;
using namespace rnnlm_tc;

constexpr int NM = 128;                        // histories per tile (UMMA M)
constexpr int NN = 256;                        // words per tile (UMMA N)
constexpr int NK = 64;                         // K elements per stage (one 128-byte swizzle atom)
constexpr int A_B = NM * NK * 2;               // 16 KB (hi or lo)
constexpr int B_B = NN * NK * 2;               // 32 KB (Theta_hi or Theta_lo)
// smem stages: [h_hi | h_lo | Theta_hi] (64 KB, 3 deep) or, with the Theta_lo
// operand, [h_hi | h_lo | Theta_hi | Theta_lo] (96 KB, 2 deep)
template <bool LO> __host__ __device__ constexpr int nst_of() { return LO ? 2 : 3; }
template <bool LO> __host__ __device__ constexpr int stage_of() { return 2 * A_B + (LO ? 2 : 1) * B_B; }
template <bool LO> constexpr size_t nsmem_of() { return 1024 + (size_t)nst_of<LO>() * stage_of<LO>() + 256; }
constexpr int NEPI = 8;                        // epilogue warps
constexpr int NTHREADS = (2 + NEPI) * 32;
constexpr int MAXORD = 8;

struct NormArgs {
  uint32_t n, H, V, nT, mt;
  unsigned long long mask;                     // M - 1
  unsigned long long alpha[MAXORD];            // alpha_k (index k-1)
  const float *bias1;                          // V: b_v + maxent[v mod M]
  const float *maxent;
  const unsigned long long *beta;              // [n][MAXORD]: beta_k at index k-1
  const uint32_t *nord;                        // [n]: K (0 = invalid history)
  float2 *part;                                // [n][nT][2]: (max, sum exp(s - max))
};

__device__ __forceinline__ uint32_t ctx_count(const Rec &r, uint32_t N) {
  uint32_t c = 0;
  for (uint32_t j = 0; j + 1 < N && j < (uint32_t)MAX_CTX; ++j) c += (r.ctx[j] != NONE);
  return c;
}

// One warp per history: validate, write the A row [hi | lo] (bf16, 2H), the
// number of MaxEnt orders K and the offsets beta_k of orders 2..K.
__global__ void __launch_bounds__(256) k_norm_prep(Params P, uint32_t n, const uint32_t *__restrict__ sess,
                                                   const uint32_t *__restrict__ hist, __nv_bfloat16 *A,
                                                   unsigned long long *beta, uint32_t *nord) {
  pdl_entry();
  const uint32_t lane = threadIdx.x & 31, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    const uint32_t s = sess[i], hd = hist[i];
    const bool ok = s < P.S && hd < P.ctr[s].next_handle;
    Rec r;
    r.slot = 0;
    for (int j = 0; j < MAX_CTX; ++j) r.ctx[j] = NONE;
    if (ok) r = P.rec[(size_t)s * P.cap + hd];
    const float4 *h = reinterpret_cast<const float4 *>(P.state + ((size_t)s * P.cap + r.slot) * P.H);
    uint4 *hi = reinterpret_cast<uint4 *>(A + (size_t)i * 2 * P.H);
    uint4 *lo = reinterpret_cast<uint4 *>(A + (size_t)i * 2 * P.H + P.H);
    for (uint32_t c = lane; c < P.H / 8; c += 32) {
      float x[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (ok) {
        const float4 u = h[2 * c], v = h[2 * c + 1];
        x[0] = u.x; x[1] = u.y; x[2] = u.z; x[3] = u.w; x[4] = v.x; x[5] = v.y; x[6] = v.z; x[7] = v.w;
      }
      uint32_t wh[4], wl[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const __nv_bfloat162 a = __floats2bfloat162_rn(x[2 * j], x[2 * j + 1]);
        const float2 af = __bfloat1622float2(a);
        const __nv_bfloat162 b = __floats2bfloat162_rn(x[2 * j] - af.x, x[2 * j + 1] - af.y);
        wh[j] = *reinterpret_cast<const uint32_t *>(&a);
        wl[j] = *reinterpret_cast<const uint32_t *>(&b);
      }
      hi[c] = make_uint4(wh[0], wh[1], wh[2], wh[3]);
      lo[c] = make_uint4(wl[0], wl[1], wl[2], wl[3]);
    }
    if (lane == 0) {
      const uint32_t K = ok ? min(P.N, ctx_count(r, P.N) + 1) : 0u;
      nord[i] = K;
      unsigned long long b = 0;                // beta_1 = 0
      beta[(size_t)i * MAXORD] = 0;
      for (uint32_t k = 2; k <= K; ++k) {
        b = (b * 237967ull + (unsigned long long)r.ctx[k - 2] + 1ull) & P.M_mask;
        beta[(size_t)i * MAXORD + k - 1] = b;
      }
    }
  }
}

// bias1[v] = b_v + maxent[v mod M] (the order-1 MaxEnt feature depends on v only)
__global__ void k_norm_bias1(Params P, float *bias1) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < P.V) bias1[v] = P.nce_b[v] + P.maxent[v & P.M_mask];
}

// fp32 output rows -> bf16 parts hi = bf16(w), lo = bf16(w - hi) (only when
// the engine keeps no bf16 copy); *any_lo = 1 if some lo part is non-zero
__global__ void k_norm_theta16(const float *w, __nv_bfloat16 *o, __nv_bfloat16 *lo, size_t count, int *any_lo) {
  int nz = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    const __nv_bfloat16 hi = __float2bfloat16_rn(w[i]);
    const __nv_bfloat16 l = __float2bfloat16_rn(w[i] - __bfloat162float(hi));
    o[i] = hi;
    lo[i] = l;
    nz |= __bfloat162float(l) != 0.0f;
  }
  if (__syncthreads_or(nz) && threadIdx.x == 0) atomicOr(any_lo, 1);
}

// Persistent GEMM + epilogue.  Tiles t -> (word tile j = t / mt, history
// tile m = t % mt): consecutive tiles share the same output rows (L2 reuse).
// warp 0: TMA producer; warp 1: TMEM owner + MMA issue; warps 2-9: epilogue
// (TMEM lane quarter warp % 4, column half (warp - 2) / 4).
template <bool LO>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_norm_tc(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_t,
              const __grid_constant__ CUtensorMap map_tl, NormArgs a) {
  constexpr int NST = nst_of<LO>(), STAGE = stage_of<LO>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + NST * STAGE), *empty = full + NST, *tfull = empty + NST,
           *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    prefetch_map(&map_a);
    prefetch_map(&map_t);
    if (LO) prefetch_map(&map_tl);
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], NEPI * 32); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_entry();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t ntiles = a.mt * a.nT, KC = a.H / NK;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int m0 = (int)((t % a.mt) * NM), n0 = (int)((t / a.mt) * NN);
        for (uint32_t kc = 0; kc < KC; ++kc) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], STAGE);
          const uint32_t d = smem_u32(sm + stage * STAGE);
          tma_load_2d(d, &map_a, &full[stage], (int)(kc * NK), m0);                  // hi
          tma_load_2d(d + A_B, &map_a, &full[stage], (int)(a.H + kc * NK), m0);      // lo
          tma_load_2d(d + 2 * A_B, &map_t, &full[stage], (int)(kc * NK), n0);        // Theta rows
          if (LO) tma_load_2d(d + 2 * A_B + B_B, &map_tl, &full[stage], (int)(kc * NK), n0);   // Theta_lo
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    uint32_t stage = 0, phase = 0, it = 0;
    const uint32_t id = idesc_bf16(NM, NN);
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const uint32_t acc = it & 1;
      mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t tm = tmem_base + acc * NN;
      for (uint32_t kc = 0; kc < KC; ++kc) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t d = smem_u32(sm + stage * STAGE);
#pragma unroll
          for (int k = 0; k < NK / 16; ++k) {
            umma_bf16(tm, sdesc(d + k * 32), sdesc(d + 2 * A_B + k * 32), id, (kc | k) != 0);
            umma_bf16(tm, sdesc(d + A_B + k * 32), sdesc(d + 2 * A_B + k * 32), id, 1u);
            if (LO) umma_bf16(tm, sdesc(d + k * 32), sdesc(d + 2 * A_B + B_B + k * 32), id, 1u);
          }
          umma_commit(&empty[stage]);
          if (kc == KC - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == NST) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    const int q = warp & 3, half = (warp - 2) >> 2;
    uint32_t it = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const uint32_t m = t % a.mt, j = t / a.mt, acc = it & 1;
      const uint32_t row = m * NM + q * 32 + lane;
      const bool valid = row < a.n;
      const uint32_t K = valid ? a.nord[row] : 0u;
      unsigned long long bk[MAXORD - 1];
#pragma unroll
      for (int k = 0; k < MAXORD - 1; ++k) bk[k] = (uint32_t)(k + 1) < K ? a.beta[(size_t)row * MAXORD + k + 1] : 0ull;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tcol = tmem_base + acc * NN + ((uint32_t)(q * 32) << 16) + half * (NN / 2);
      float m_run = -INFINITY, l_run = 0.0f;
#pragma unroll 1
      for (int g = 0; g < NN / 32; ++g) {
        const uint32_t v0 = j * NN + half * (NN / 2) + g * 16;
        float x[16], e[16];
        tmem_ld16(tcol + g * 16, x);
#pragma unroll
        for (int u = 0; u < 16; ++u) e[u] = (v0 + u < a.V) ? __ldg(a.bias1 + v0 + u) : 0.0f;
        // MaxEnt orders 2..K: independent random gathers, all issued before use
#pragma unroll
        for (int k = 0; k < MAXORD - 1; ++k) {
          if ((uint32_t)(k + 1) >= K) break;
          const unsigned long long al = a.alpha[k + 1], be = bk[k];
#pragma unroll
          for (int u = 0; u < 16; ++u)
            if (v0 + u < a.V) e[u] += __ldg(a.maxent + ((al * (unsigned long long)(v0 + u) + be) & a.mask));
        }
        tmem_ld_wait();
        float gm = -INFINITY;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          x[u] += e[u];
          if (v0 + u < a.V) gm = fmaxf(gm, x[u]);
        }
        if (gm > m_run) {
          l_run *= __expf(m_run - gm);
          m_run = gm;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (v0 + u < a.V) l_run += __expf(x[u] - m_run);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (valid) a.part[((size_t)row * a.nT + j) * 2 + half] = make_float2(m_run, l_run);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// One warp per history: the 2 nT partials combined in a fixed order (lane
// l takes partials l, l + 32, ...; then a fixed xor tree), log Z = m + log l.
__global__ void __launch_bounds__(256) k_norm_reduce(uint32_t n, uint32_t nT, const float2 *__restrict__ part,
                                                     const uint32_t *__restrict__ nord, float *__restrict__ log_z) {
  pdl_entry();
  const uint32_t lane = threadIdx.x & 31, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    float m = -INFINITY, l = 0.0f;
    for (uint32_t p = lane; p < 2 * nT; p += 32) {
      const float2 c = part[(size_t)i * 2 * nT + p];
      if (c.y <= 0.0f) continue;                // an empty half tile (words >= V)
      if (c.x > m) {
        l = l * __expf(m - c.x) + c.y;
        m = c.x;
      } else {
        l += c.y * __expf(c.x - m);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xFFFFFFFFu, m, o), l2 = __shfl_xor_sync(0xFFFFFFFFu, l, o);
      const float mm = fmaxf(m, m2);
      if (mm != -INFINITY) {
        l = l * __expf(m - mm) + l2 * __expf(m2 - mm);
        m = mm;
      }
    }
    if (lane == 0) log_z[i] = nord[i] ? m + logf(l) : __int_as_float(0x7FC00000);
  }
}

struct NormState {
  uint32_t bmax = 0, bmax_pad = 0, nT = 0;
  __nv_bfloat16 *theta16 = nullptr;            // owned only when converted here
  __nv_bfloat16 *theta_lo = nullptr;           // Theta - Theta_hi (bf16), when some entry is not bf16-exact
  bool own_theta = false, lo = false;
  __nv_bfloat16 *A = nullptr;
  float *bias1 = nullptr;
  unsigned long long *beta = nullptr;
  uint32_t *nord = nullptr;
  float2 *part = nullptr;
  CUtensorMap map_a, map_t, map_tl;
};

}  // namespace rnnlm_norm

namespace rnnlm_host {
using namespace rnnlm_norm;

int norm_supported(uint32_t H, uint32_t N) { return H % 64 == 0 && N <= (uint32_t)MAXORD; }

void norm_release(void *state) {
  NormState *t = static_cast<NormState *>(state);
  if (!t) return;
  if (t->own_theta) cudaFree(t->theta16);
  cudaFree(t->theta_lo);
  cudaFree(t->A);
  cudaFree(t->bias1);
  cudaFree(t->beta);
  cudaFree(t->nord);
  cudaFree(t->part);
  delete t;
}

// Lazily sized for max_queries_per_call histories per call.
int norm_prepare(const Params &P, uint32_t bmax, void **state_out, cudaStream_t s) {
  *state_out = nullptr;
  if (!norm_supported(P.H, P.N)) return -1;
  NormState *t = new NormState;
  t->bmax = bmax;
  t->bmax_pad = (bmax + NM - 1) / NM * NM;
  t->nT = (P.V + NN - 1) / NN;
  bool ok = true;
  if (P.nce_w16) {
    t->theta16 = const_cast<__nv_bfloat16 *>(P.nce_w16);
  } else {
    int *d_any = nullptr, any = 0;
    ok = cudaMalloc(&t->theta16, (size_t)P.V * P.H * 2) == cudaSuccess;
    t->own_theta = ok;
    ok = ok && cudaMalloc(&t->theta_lo, (size_t)P.V * P.H * 2) == cudaSuccess &&
         cudaMalloc(&d_any, sizeof(int)) == cudaSuccess && cudaMemsetAsync(d_any, 0, sizeof(int), s) == cudaSuccess;
    if (ok) k_norm_theta16<<<1184, 256, 0, s>>>(P.nce_w, t->theta16, t->theta_lo, (size_t)P.V * P.H, d_any);
    ok = ok && cudaMemcpyAsync(&any, d_any, sizeof(int), cudaMemcpyDeviceToHost, s) == cudaSuccess &&
         cudaStreamSynchronize(s) == cudaSuccess;
    cudaFree(d_any);
    t->lo = any != 0;
    if (!t->lo) {                               // bf16-exact rows: no third product
      cudaFree(t->theta_lo);
      t->theta_lo = nullptr;
    }
  }
  ok = ok && cudaMalloc(&t->A, (size_t)t->bmax_pad * 2 * P.H * 2) == cudaSuccess &&
       cudaMemsetAsync(t->A, 0, (size_t)t->bmax_pad * 2 * P.H * 2, s) == cudaSuccess &&
       cudaMalloc(&t->bias1, (size_t)P.V * 4) == cudaSuccess &&
       cudaMalloc(&t->beta, (size_t)bmax * MAXORD * 8) == cudaSuccess &&
       cudaMalloc(&t->nord, (size_t)bmax * 4) == cudaSuccess &&
       cudaMalloc(&t->part, (size_t)bmax * t->nT * 2 * sizeof(float2)) == cudaSuccess;
  if (ok) k_norm_bias1<<<(P.V + 255) / 256, 256, 0, s>>>(P, t->bias1);
  ok = ok && make_map(&t->map_a, t->A, 2ull * P.H, t->bmax_pad, NM) &&
       make_map(&t->map_t, t->theta16, P.H, P.V, NN) &&
       (!t->lo || make_map(&t->map_tl, t->theta_lo, P.H, P.V, NN)) &&
       cudaFuncSetAttribute(k_norm_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nsmem_of<false>()) == cudaSuccess &&
       cudaFuncSetAttribute(k_norm_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nsmem_of<true>()) == cudaSuccess;
  if (ok && !t->lo) t->map_tl = t->map_t;
  if (!ok) {
    (void)cudaGetLastError();
    norm_release(t);
    return -1;
  }
  *state_out = t;
  return 0;
}

// Returns the number of kernels launched.
int launch_norm(const Params &P, void *state, uint32_t n, const uint32_t *sess, const uint32_t *hist,
                float *log_z, int num_sms, cudaStream_t s) {
  NormState *t = static_cast<NormState *>(state);
  if (!n) return 0;
  NormArgs a;
  a.n = n; a.H = P.H; a.V = P.V; a.nT = t->nT; a.mt = (n + NM - 1) / NM;
  a.mask = P.M_mask;
  unsigned long long al = 1;
  for (int k = 0; k < MAXORD; ++k) {
    a.alpha[k] = al;
    al = (al * 237967ull) & P.M_mask;
  }
  a.bias1 = t->bias1; a.maxent = P.maxent; a.beta = t->beta; a.nord = t->nord; a.part = t->part;
  uint32_t gp = (n + 7) / 8;
  if (gp > (uint32_t)num_sms * 4) gp = num_sms * 4;
  launch_pdl(k_norm_prep, gp, 256, 0, s, P, n, sess, hist, t->A, t->beta, t->nord);
  uint32_t g = a.mt * a.nT;
  if (g > (uint32_t)num_sms) g = num_sms;
  if (t->lo) launch_pdl(k_norm_tc<true>, g, NTHREADS, nsmem_of<true>(), s, t->map_a, t->map_t, t->map_tl, a);
  else launch_pdl(k_norm_tc<false>, g, NTHREADS, nsmem_of<false>(), s, t->map_a, t->map_t, t->map_tl, a);
  launch_pdl(k_norm_reduce, gp, 256, 0, s, n, t->nT, t->part, t->nord, log_z);
  return 3;
}
}  // namespace rnnlm_host
