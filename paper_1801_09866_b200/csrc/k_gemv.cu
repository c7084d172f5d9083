// k_gemv.cu -- step (a5) for SMALL frames: embedding gather + GRU update as
// two memory-bound GEMV-style kernels (SURVEY 8(a5) "Small-Q path";
// BASELINE north_star: "a vectorised memory-bound GEMV path where [the batch]
// does not [make the gate projection a real dense contraction]").
//
// The paper's frames are small: ~197 rows per frame exchange (P:160-161,
// P:186-189); at paper-shaped hit rates a 256-query frame has ~30 GRU rows,
// which fills a quarter of ONE 128-row tensor-core tile while the tile
// kernels' weight streams run on 3-6 SMs.  Here the work is cut by OUTPUT
// UNITS instead: every CTA owns U units of every row, reads their weight rows
// once (L2-resident: 3H(E+H) elements for the whole model, 0.8 / 1.6 MB at
// H = E = 256 bf16 / fp32) and walks all Q rows, so all SMs pull weights at
// once and the frame's latency is a few dependent L2 round trips.
//
//   k_gemv1  z = s(Wz x + Uz h + bz), r = s(Wr x + Ur h + br), Wh x + bh
//            (x = E[word], h = parent state, gathered in place -- no A1 block);
//            writes z, r.h (GRU; r for LBR) and Wh x + bh per (row, unit)
//   k_gemv2  Uh (r.h) (GRU) or Uh h (LBR, RNN), the cell's update, the new
//            fp32 state; the last CTA to finish encodes the new states'
//            compression codes (encode.cuh, step a1) -- no extra launch.
//
// Operand rounding follows the engine's math mode so the GEMV stands in for
// the tile kernels with the same arithmetic model (products exact in fp32,
// fp32 accumulation, only the summation order differs): BF16 -- bf16
// weights (the tensor path's W1/W2), x from the bf16 embedding copy, h and
// r.h rounded to bf16; TF32 -- TF32-rounded weights and operands; FP32 and
// TF32X3 -- plain fp32 (FFMA; more accurate than 3xTF32).  Lanes split K in
// 8-element chunks, a fixed xor-butterfly reduces across the warp
// (deterministic, batch-invariant for a given path).
#include <cstdlib>
#include <cstring>
#include <vector>

#include "encode.cuh"

namespace rnnlm_gemv {
using namespace rnnlm_dev;

constexpr int U1 = 4;          // units per CTA, phase 1 (x 3 gates)
constexpr int U2 = 8;          // units per CTA, phase 2
constexpr int THREADS = 128;   // four warps; rows are dealt to warps
enum { ACT_F32 = 0, ACT_BF16 = 1, ACT_TF32 = 2 };

struct GemvArgs {
  uint32_t E, H, RW;           // W1 / W2 row width (elements)
  uint32_t tc_layout;          // 1: z row of unit u = (u/128)*256 + u%128, r = +128; 0: z = u, r = H + u
  const void *w1, *w2;         // W1: z and r rows [Wz|Uz], [Wr|Ur]; W2: rows [Wh|Uh] (K-major, width RW)
  const float *bz, *br, *bh;
  const float *emb;            // V x E fp32
  const __nv_bfloat16 *emb16;  // V x E bf16 (BF16)
  float *state;
  const uint32_t *row_src, *row_dst, *row_word, *counts;
  float *gz, *grh, *gwxb;      // [rows][H] scratch
  uint32_t *done;              // phase-2 CTAs finished (last one encodes; it resets the counter)
  uint32_t cache, cstride;
  KeySpec key;
  uint8_t *codes;
  unsigned long long *codehash;
};

__device__ __forceinline__ float sigm(float a) { return 1.0f / (1.0f + expf(-a)); }
__device__ __forceinline__ float rnd_bf16(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
__device__ __forceinline__ float rnd_tf32(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}
template <int ACT>
__device__ __forceinline__ float op(float v) {
  if constexpr (ACT == ACT_BF16) return rnd_bf16(v);
  else if constexpr (ACT == ACT_TF32) return rnd_tf32(v);
  else return v;
}

// 8 consecutive elements of a weight row (bf16 or fp32 storage) as fp32
template <typename WT>
__device__ __forceinline__ void ld8(const WT *p, float *w) {
  if constexpr (sizeof(WT) == 2) {
    const uint4 t = __ldg(reinterpret_cast<const uint4 *>(p));
    const uint32_t u[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      w[2 * j] = __uint_as_float(u[j] << 16);
      w[2 * j + 1] = __uint_as_float(u[j] & 0xFFFF0000u);
    }
  } else {
    const float4 a = __ldg(reinterpret_cast<const float4 *>(p));
    const float4 b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w; w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
  }
}
__device__ __forceinline__ void ld8f(const float *p, float *v) {
  const float4 a = *reinterpret_cast<const float4 *>(p);
  const float4 b = *(reinterpret_cast<const float4 *>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// Activation chunk c (8 elements) of row r's phase-1 operand [x | h], rounded
// like the tile kernels' operands.
template <int ACT>
__device__ __forceinline__ void act8(const GemvArgs &g, uint32_t word, uint32_t src, uint32_t k, float *a) {
  if (k < g.E) {
    if constexpr (ACT == ACT_BF16) {
      const uint4 t = __ldg(reinterpret_cast<const uint4 *>(g.emb16 + (size_t)word * g.E + k));
      const uint32_t u[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        a[2 * j] = __uint_as_float(u[j] << 16);
        a[2 * j + 1] = __uint_as_float(u[j] & 0xFFFF0000u);
      }
    } else {
      const float4 *p = reinterpret_cast<const float4 *>(g.emb + (size_t)word * g.E + k);
      const float4 x0 = __ldg(p), x1 = __ldg(p + 1);
      a[0] = x0.x; a[1] = x0.y; a[2] = x0.z; a[3] = x0.w; a[4] = x1.x; a[5] = x1.y; a[6] = x1.z; a[7] = x1.w;
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = op<ACT>(a[j]);
    }
  } else {
    ld8f(g.state + (size_t)src * g.H + (k - g.E), a);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = op<ACT>(a[j]);
  }
}

__device__ __forceinline__ size_t z_row(const GemvArgs &g, uint32_t u) {
  return g.tc_layout ? (size_t)(((u >> 7) << 8) + (u & 127)) : (size_t)u;
}
__device__ __forceinline__ size_t r_row(const GemvArgs &g, uint32_t u) {
  return z_row(g, u) + (g.tc_layout ? 128u : g.H);
}

template <int N>
__device__ __forceinline__ void warp_sum(float *v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
}

// Phase 1: units [U1 * blockIdx.x, +U1) of rows blockIdx.y, +gridDim.y, ...
template <typename WT, int ACT, int CELL>
__global__ void __launch_bounds__(THREADS) k_gemv1(GemvArgs g) {
  pdl_entry();
  const uint32_t Q = g.counts[1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t u0 = blockIdx.x * U1;
  const uint32_t K1 = g.E + g.H, nch = K1 / 8, nchx = g.E / 8;
  constexpr bool RNN = CELL == RNNLM_CELL_RNN;
  const WT *w1 = static_cast<const WT *>(g.w1), *w2 = static_cast<const WT *>(g.w2);
  for (uint32_t row = blockIdx.y * (THREADS / 32) + warp; row < Q; row += gridDim.y * (THREADS / 32)) {
    const uint32_t word = g.row_word[row], src = g.row_src[row];
    float acc[3 * U1];
#pragma unroll
    for (int i = 0; i < 3 * U1; ++i) acc[i] = 0.0f;
    for (uint32_t c = lane; c < nch; c += 32) {
      const uint32_t k = c * 8;
      if (RNN && c >= nchx) break;                      // the RNN cell needs only Wh x here
      float a[8];
      act8<ACT>(g, word, src, k, a);
#pragma unroll
      for (int j = 0; j < U1; ++j) {
        const uint32_t u = u0 + j;
        float w[8];
        if (!RNN) {
          ld8(w1 + z_row(g, u) * g.RW + k, w);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[3 * j] = fmaf(a[e], w[e], acc[3 * j]);
          ld8(w1 + r_row(g, u) * g.RW + k, w);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[3 * j + 1] = fmaf(a[e], w[e], acc[3 * j + 1]);
        }
        if (c < nchx) {
          ld8(w2 + (size_t)u * g.RW + k, w);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[3 * j + 2] = fmaf(a[e], w[e], acc[3 * j + 2]);
        }
      }
    }
    warp_sum<3 * U1>(acc);
    if (lane < U1) {
      const uint32_t u = u0 + lane;
      float sz = acc[0], sr = acc[1], sh = acc[2];
#pragma unroll
      for (int j = 1; j < U1; ++j)
        if (lane == j) { sz = acc[3 * j]; sr = acc[3 * j + 1]; sh = acc[3 * j + 2]; }
      const size_t o = (size_t)row * g.H + u;
      g.gwxb[o] = sh + g.bh[u];
      if (!RNN) {
        const float z = sigm(sz + g.bz[u]), r = sigm(sr + g.br[u]);
        g.gz[o] = z;
        if (CELL == RNNLM_CELL_GRU_LBR) {
          g.grh[o] = r;                                 // applied after Uh h
        } else {
          const float h = g.state[(size_t)src * g.H + u];
          // r.h as the tile kernels form their phase-2 A operand
          g.grh[o] = ACT == ACT_TF32 ? rnd_tf32(r * h) : op<ACT>(r * op<ACT>(h));
        }
      }
    }
  }
}

// Phase 2: units [U2 * blockIdx.x, +U2) of rows blockIdx.y, +gridDim.y, ...;
// then the last CTA encodes every new state (one warp per row).
template <typename WT, int ACT, int CELL>
__global__ void __launch_bounds__(THREADS) k_gemv2(GemvArgs g) {
  pdl_entry();
  __shared__ uint32_t s_last;
  const uint32_t Q = g.counts[1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t u0 = blockIdx.x * U2;
  const uint32_t nch = g.H / 8;
  const WT *w2 = static_cast<const WT *>(g.w2);
  for (uint32_t row = blockIdx.y * (THREADS / 32) + warp; row < Q; row += gridDim.y * (THREADS / 32)) {
    const uint32_t dst = g.row_dst[row], src = g.row_src[row];
    float acc[U2];
#pragma unroll
    for (int i = 0; i < U2; ++i) acc[i] = 0.0f;
    for (uint32_t c = lane; c < nch; c += 32) {
      const uint32_t k = c * 8;
      float a[8];
      if (CELL == RNNLM_CELL_GRU) {
        ld8f(g.grh + (size_t)row * g.H + k, a);
      } else {
        ld8f(g.state + (size_t)src * g.H + k, a);
#pragma unroll
        for (int e = 0; e < 8; ++e) a[e] = op<ACT>(a[e]);
      }
#pragma unroll
      for (int j = 0; j < U2; ++j) {
        float w[8];
        ld8(w2 + (size_t)(u0 + j) * g.RW + g.E + k, w);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[j] = fmaf(a[e], w[e], acc[j]);
      }
    }
    warp_sum<U2>(acc);
    if (lane < U2 && dst != NONE) {
      const uint32_t u = u0 + lane;
      float s = acc[0];
#pragma unroll
      for (int j = 1; j < U2; ++j)
        if (lane == j) s = acc[j];
      const size_t o = (size_t)row * g.H + u;
      float hn;
      if (CELL == RNNLM_CELL_RNN) {
        hn = sigm(g.gwxb[o] + s);
      } else {
        const float z = g.gz[o], h = g.state[(size_t)src * g.H + u];
        const float c = tanhf(g.gwxb[o] + (CELL == RNNLM_CELL_GRU_LBR ? g.grh[o] * s : s));
        hn = (1.0f - z) * h + z * c;
      }
      g.state[(size_t)dst * g.H + u] = hn;
    }
  }
  if (!g.cache) return;
  // (a1) codes of the new states: the last CTA to finish (threadfence
  // reduction pattern) encodes every row, one warp per row
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t t = atomicAdd(g.done, 1u);
    s_last = t == gridDim.x * gridDim.y - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (uint32_t row = warp; row < Q; row += THREADS / 32) {
    const uint32_t dst = g.row_dst[row];
    if (dst == NONE) continue;
    uint8_t *code = g.key.mode == RNNLM_KEY_OFF ? nullptr : g.codes + (size_t)dst * g.cstride;
    const unsigned long long hs = encode_row_warp(g.key, g.cstride, g.state + (size_t)dst * g.H, code);
    if (lane == 0) g.codehash[dst] = hs;
  }
  if (threadIdx.x == 0) *g.done = 0u;
}

struct GemvState {
  GemvArgs g{};
  uint32_t rows = 0;            // scratch rows (the largest call that may take this path)
  int wt_bf16 = 0, act = ACT_F32;
  std::vector<void *> allocs;
};

}  // namespace rnnlm_gemv

namespace rnnlm_host {
using namespace rnnlm_gemv;

// Weights: BF16 / TF32 engines pass the tensor path's W1 / W2 (tc_layout 1,
// already rounded); FP32 / TF32X3 engines get their own fp32 rows here.
int gemv_prepare(const Params &P, const rnnlm_weights *w, uint32_t math, const void *tc_w1, const void *tc_w2,
                 uint32_t tc_rw, uint32_t rows, void **state_out) {
  *state_out = nullptr;
  GemvState *st = new GemvState;
  GemvArgs &g = st->g;
  const size_t E = P.E, H = P.H, K1 = E + H;
  auto dup = [&](const float *src, size_t n) -> float * {
    void *d = nullptr;
    if (cudaMalloc(&d, n * 4) != cudaSuccess) return nullptr;
    st->allocs.push_back(d);
    cudaMemcpy(d, src, n * 4, cudaMemcpyHostToDevice);
    return static_cast<float *>(d);
  };
  g.E = P.E; g.H = P.H;
  g.bz = dup(w->bz, H); g.br = dup(w->br, H); g.bh = dup(w->bh, H);
  if (math == RNNLM_MATH_BF16 || math == RNNLM_MATH_TF32) {
    g.w1 = tc_w1; g.w2 = tc_w2; g.RW = tc_rw; g.tc_layout = 1;
    st->wt_bf16 = math == RNNLM_MATH_BF16;
    st->act = math == RNNLM_MATH_BF16 ? ACT_BF16 : ACT_TF32;
  } else {
    std::vector<float> w1(2 * H * K1), w2(H * K1);
    for (size_t u = 0; u < H; ++u) {
      std::memcpy(&w1[u * K1], w->Wz + u * E, E * 4);
      std::memcpy(&w1[u * K1 + E], w->Uz + u * H, H * 4);
      std::memcpy(&w1[(H + u) * K1], w->Wr + u * E, E * 4);
      std::memcpy(&w1[(H + u) * K1 + E], w->Ur + u * H, H * 4);
      std::memcpy(&w2[u * K1], w->Wh + u * E, E * 4);
      std::memcpy(&w2[u * K1 + E], w->Uh + u * H, H * 4);
    }
    g.w1 = dup(w1.data(), w1.size()); g.w2 = dup(w2.data(), w2.size());
    g.RW = (uint32_t)K1; g.tc_layout = 0;
  }
  st->rows = rows;
  void *scratch = nullptr, *done = nullptr;
  if (cudaMalloc(&scratch, (size_t)3 * rows * H * 4) != cudaSuccess || cudaMalloc(&done, 4) != cudaSuccess) {
    (void)cudaGetLastError();
    delete st;
    return -1;
  }
  st->allocs.push_back(scratch);
  st->allocs.push_back(done);
  cudaMemset(done, 0, 4);
  g.gz = static_cast<float *>(scratch);
  g.grh = g.gz + (size_t)rows * H;
  g.gwxb = g.grh + (size_t)rows * H;
  g.done = static_cast<uint32_t *>(done);
  *state_out = st;
  return (g.bz && g.br && g.bh && g.w1 && g.w2) ? 0 : -1;
}

void gemv_release(void *state) {
  GemvState *st = static_cast<GemvState *>(state);
  if (!st) return;
  for (void *p : st->allocs) cudaFree(p);
  delete st;
}

template <typename WT, int ACT, int CELL>
static void launch2(const GemvArgs &g, dim3 gr1, dim3 gr2, cudaStream_t s) {
  launch_pdl(k_gemv1<WT, ACT, CELL>, gr1, THREADS, 0, s, g);
  launch_pdl(k_gemv2<WT, ACT, CELL>, gr2, THREADS, 0, s, g);
}

// Rows per call are <= st->rows (checked by the caller).
int launch_gemv(const Params &P, void *state, int num_sms, cudaStream_t s) {
  GemvState *st = static_cast<GemvState *>(state);
  GemvArgs g = st->g;
  g.emb = P.emb; g.emb16 = P.emb16; g.state = P.state;
  g.row_src = P.row_src; g.row_dst = P.row_dst; g.row_word = P.row_word; g.counts = P.counts;
  g.cache = P.cache; g.cstride = P.cstride; g.codes = P.codes; g.codehash = P.codehash;
  g.key = KeySpec{P.key_mode, P.round_digits, P.H, P.round_scale};
  // unit blocks x row blocks: about two CTAs per SM, row blocks only as far as
  // the rows go (each row block re-reads its units' weights from L2)
  const uint32_t nb1 = P.H / U1, nb2 = P.H / U2;
  const uint32_t want = 2u * (uint32_t)num_sms, rmax = (st->rows + 3) / 4;
  uint32_t rb1 = (want + nb1 - 1) / nb1, rb2 = (want + nb2 - 1) / nb2;
  rb1 = rb1 < rmax ? rb1 : rmax; rb2 = rb2 < rmax ? rb2 : rmax;
  rb1 = rb1 ? rb1 : 1; rb2 = rb2 ? rb2 : 1;
  const dim3 gr1(nb1, rb1), gr2(nb2, rb2);
  const int cell = (int)P.cell;
  if (st->act == ACT_BF16) {
    if (cell == 0) launch2<__nv_bfloat16, ACT_BF16, 0>(g, gr1, gr2, s);
    else if (cell == 1) launch2<__nv_bfloat16, ACT_BF16, 1>(g, gr1, gr2, s);
    else launch2<__nv_bfloat16, ACT_BF16, 2>(g, gr1, gr2, s);
  } else if (st->act == ACT_TF32) {
    if (cell == 0) launch2<float, ACT_TF32, 0>(g, gr1, gr2, s);
    else if (cell == 1) launch2<float, ACT_TF32, 1>(g, gr1, gr2, s);
    else launch2<float, ACT_TF32, 2>(g, gr1, gr2, s);
  } else {
    if (cell == 0) launch2<float, ACT_F32, 0>(g, gr1, gr2, s);
    else if (cell == 1) launch2<float, ACT_F32, 1>(g, gr1, gr2, s);
    else launch2<float, ACT_F32, 2>(g, gr1, gr2, s);
  }
  return 2;
}
}  // namespace rnnlm_host
