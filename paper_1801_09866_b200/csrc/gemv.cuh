// gemv.cuh -- the small-frame GEMV form of step (a5) as device functions,
// shared by the two-kernel GEMV path (k_gemv.cu) and the fused small-frame
// kernel (k_small.cu).  Design notes: k_gemv.cu.
#pragma once

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

// Phase 1 of unit block ub (units [U1 * ub, +U1)) for rows rb * nwarps + warp,
// stepping nrb * nwarps: one warp per row at a time.
template <typename WT, int ACT, int CELL>
__device__ __forceinline__ void gemv1_item(const GemvArgs &g, uint32_t Q, uint32_t ub, uint32_t rb, uint32_t nrb,
                                           int warp, int nwarps) {
  const int lane = threadIdx.x & 31;
  const uint32_t u0 = ub * U1;
  const uint32_t K1 = g.E + g.H, nch = K1 / 8, nchx = g.E / 8;
  constexpr bool RNN = CELL == RNNLM_CELL_RNN;
  const WT *w1 = static_cast<const WT *>(g.w1), *w2 = static_cast<const WT *>(g.w2);
  for (uint32_t row = rb * nwarps + warp; row < Q; row += nrb * nwarps) {
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

// L1 prefetch of unit block ub's phase-1 weight rows (128-byte lines), so a
// CTA that waits for the frame's rows already holds its weights.
template <typename WT, int CELL>
__device__ __forceinline__ void gemv1_prefetch(const GemvArgs &g, uint32_t ub) {
  const uint32_t K1 = g.E + g.H;
  const uint32_t lines = (uint32_t)((size_t)K1 * sizeof(WT) / 128);          // per weight row
  const WT *w1 = static_cast<const WT *>(g.w1), *w2 = static_cast<const WT *>(g.w2);
  const uint32_t nrows = CELL == RNNLM_CELL_RNN ? U1 : 3 * U1;
  for (uint32_t i = threadIdx.x; i < nrows * lines; i += blockDim.x) {
    const uint32_t r = i / lines, l = i % lines, u = ub * U1 + r % U1, gate = r / U1;
    const WT *row = CELL == RNNLM_CELL_RNN || gate == 2 ? w2 + (size_t)u * g.RW
                    : w1 + (gate == 0 ? z_row(g, u) : r_row(g, u)) * g.RW;
    asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char *>(row) + (size_t)l * 128));
  }
}

// Phase 2 of unit block ub (units [U2 * ub, +U2)), rows as gemv1_item.
template <typename WT, int ACT, int CELL>
__device__ __forceinline__ void gemv2_item(const GemvArgs &g, uint32_t Q, uint32_t ub, uint32_t rb, uint32_t nrb,
                                           int warp, int nwarps) {
  const int lane = threadIdx.x & 31;
  const uint32_t u0 = ub * U2;
  const uint32_t nch = g.H / 8;
  const WT *w2 = static_cast<const WT *>(g.w2);
  for (uint32_t row = rb * nwarps + warp; row < Q; row += nrb * nwarps) {
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
}

// (a1) codes + code hashes of the new states of rows gw, gw + ngw, ... (one
// warp per row; encode.cuh).
__device__ __forceinline__ void gemv_encode(const GemvArgs &g, uint32_t Q, uint32_t gw, uint32_t ngw) {
  const int lane = threadIdx.x & 31;
  for (uint32_t row = gw; row < Q; row += ngw) {
    const uint32_t dst = g.row_dst[row];
    if (dst == NONE) continue;
    uint8_t *code = g.key.mode == RNNLM_KEY_OFF ? nullptr : g.codes + (size_t)dst * g.cstride;
    const unsigned long long hs = encode_row_warp(g.key, g.cstride, g.state + (size_t)dst * g.H, code);
    if (lane == 0) g.codehash[dst] = hs;
  }
}

}  // namespace rnnlm_gemv
