// k_gru_simt.cu -- step (a5), FP32 path: embedding gather + GRU update.
//
// GRU of the paper's RNNLM: "a total of six weight matrices and three bias
// vectors", gate form of the cited GRU (Chung 2014, reading 1):
//   z = s(Wz x + Uz h + bz);  r = s(Wr x + Ur h + br)
//   c = tanh(Wh x + Uh (r . h) + bh);  h' = (1 - z) . h + z . c
// x = E[word] ("Index Table"), h = the parent state; one row per MISS of
// the frame (the frame's contiguous block).
//
// Because Uh multiplies r . h, the contraction runs in two dependent phases:
//   phase 1: [Q, E+H] x [E+H, 2H] for z, r plus [Q, E] x [E, H] for Wh x,
//            gate-interleaved per 64-unit block so one CTA tile holds all
//            three pre-activations of its units; epilogue writes z, r . h and
//            Wh x + bh.
//   phase 2: [Q, H] x [H, H] for Uh (r . h); epilogue: tanh, the update,
//            the new fp32 state (and its bf16 shadow when the engine keeps one).
// Cell variants: GRU_LBR -- phase 1 stores r instead of
// r . h, phase 2 contracts the parent state h and applies r after:
// c = tanh(Wh x + bh + r . (Uh h)); RNN -- phase 2 contracts h, the new state
// is sigma(Wh x + bh + Uh h) (phase 1's z, r are not used).
// Register-tiled FFMA (64 x 64 tile, 4 x 4 per thread) with A rows gathered
// through row_word / row_src; fp32 accumulation.  This is the 1e-5 path; the
// tensor-core path lives in k_gru_tc.cu.
#include "rnnlm_impl.cuh"

namespace rnnlm_dev {

constexpr int BM = 64, BU = 64, BK = 16, NT = 256, AST = BM + 4;

__device__ __forceinline__ float sigmoidf_(float a) { return 1.0f / (1.0f + expf(-a)); }

__global__ void __launch_bounds__(NT) k_gru1_f32(Params P) {
  pdl_entry();
  __shared__ __align__(16) float As[BK][AST];
  __shared__ __align__(16) float Bs[BK][3 * BU];
  const uint32_t Q = P.counts[1];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const uint32_t ub = blockIdx.x, nub = P.Hp / 64;
  const uint32_t E = P.E, H = P.H;
  const int lr = tid >> 2, lk = (tid & 3) * 4;
  for (uint32_t rt = blockIdx.y; rt * BM < Q; rt += gridDim.y) {
    const uint32_t r0 = rt * BM;
    float acc[3][4][4];
#pragma unroll
    for (int g = 0; g < 3; ++g)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[g][i][j] = 0.0f;
    const uint32_t lrow = r0 + lr;
    const bool rv = lrow < Q;
    const float *xs = rv ? P.emb + (size_t)P.row_word[lrow] * E : P.emb;
    const float *hs = rv ? P.state + (size_t)P.row_src[lrow] * H : P.state;
    // ---- x part: z, r, h gates
    for (uint32_t k0 = 0; k0 < E; k0 += BK) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      if (rv && k0 + lk < E) a = *reinterpret_cast<const float4 *>(xs + k0 + lk);
      As[lk + 0][lr] = a.x; As[lk + 1][lr] = a.y; As[lk + 2][lr] = a.z; As[lk + 3][lr] = a.w;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int f = tid + i * NT, kk = f / 48, c = (f % 48) * 4;
        float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k0 + kk < E)
          b = __ldg(reinterpret_cast<const float4 *>(P.w1x + ((size_t)(k0 + kk) * nub + ub) * 192 + c));
        *reinterpret_cast<float4 *>(&Bs[kk][c]) = b;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        const float4 a4 = *reinterpret_cast<const float4 *>(&As[kk][ty * 4]);
        const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
        for (int g = 0; g < 3; ++g) {
          const float4 b4 = *reinterpret_cast<const float4 *>(&Bs[kk][g * 64 + tx * 4]);
          const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[g][i][j] = fmaf(av[i], bv[j], acc[g][i][j]);
        }
      }
      __syncthreads();
    }
    // ---- h part: z, r gates only (the h gate sees r . h in phase 2)
    for (uint32_t k0 = 0; k0 < H; k0 += BK) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      if (rv && k0 + lk < H) a = *reinterpret_cast<const float4 *>(hs + k0 + lk);
      As[lk + 0][lr] = a.x; As[lk + 1][lr] = a.y; As[lk + 2][lr] = a.z; As[lk + 3][lr] = a.w;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int f = tid + i * NT, kk = f / 32, c = (f % 32) * 4;
        float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k0 + kk < H)
          b = __ldg(reinterpret_cast<const float4 *>(P.w1h + ((size_t)(k0 + kk) * nub + ub) * 128 + c));
        *reinterpret_cast<float4 *>(&Bs[kk][c]) = b;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        const float4 a4 = *reinterpret_cast<const float4 *>(&As[kk][ty * 4]);
        const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const float4 b4 = *reinterpret_cast<const float4 *>(&Bs[kk][g * 64 + tx * 4]);
          const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[g][i][j] = fmaf(av[i], bv[j], acc[g][i][j]);
        }
      }
      __syncthreads();
    }
    // ---- epilogue: z, r . h, Wh x + bh
    const uint32_t u0 = ub * 64 + tx * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t row = r0 + ty * 4 + i;
      if (row >= Q) continue;
      const float *hp = P.state + (size_t)P.row_src[row] * H;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t u = u0 + j;
        if (u >= H) continue;
        const float *bb = P.b1 + (size_t)ub * 192 + tx * 4 + j;
        const float z = sigmoidf_(acc[0][i][j] + bb[0]);
        const float r = sigmoidf_(acc[1][i][j] + bb[64]);
        const size_t o = (size_t)row * H + u;
        P.g_z[o] = z;
        P.g_rh[o] = P.cell == RNNLM_CELL_GRU_LBR ? r : r * hp[u];   // LBR: r itself (applied after Uh h)
        P.g_wxb[o] = acc[2][i][j] + bb[128];
      }
    }
  }
}

__global__ void __launch_bounds__(NT) k_gru2_f32(Params P) {
  pdl_entry();
  __shared__ __align__(16) float As[BK][AST];
  __shared__ __align__(16) float Bs[BK][BU];
  const uint32_t Q = P.counts[1];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const uint32_t ub = blockIdx.x;
  const uint32_t H = P.H;
  const int lr = tid >> 2, lk = (tid & 3) * 4;
  for (uint32_t rt = blockIdx.y; rt * BM < Q; rt += gridDim.y) {
    const uint32_t r0 = rt * BM;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    const uint32_t lrow = r0 + lr;
    const bool rv = lrow < Q;
    // A operand: r . h (GRU) or the parent state h itself (LBR: Uh h, reset applied after)
    const bool lbr = P.cell == RNNLM_CELL_GRU_LBR, rnn = P.cell == RNNLM_CELL_RNN;
    const float *as = (lbr || rnn) ? P.state + (size_t)(rv ? P.row_src[lrow] : 0) * H : P.g_rh + (size_t)(rv ? lrow : 0) * H;
    for (uint32_t k0 = 0; k0 < H; k0 += BK) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      if (rv && k0 + lk < H) a = *reinterpret_cast<const float4 *>(as + k0 + lk);
      As[lk + 0][lr] = a.x; As[lk + 1][lr] = a.y; As[lk + 2][lr] = a.z; As[lk + 3][lr] = a.w;
      {
        const int kk = tid / 16, c = (tid % 16) * 4;
        float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k0 + kk < H)
          b = __ldg(reinterpret_cast<const float4 *>(P.w2 + (size_t)(k0 + kk) * P.Hp + ub * 64 + c));
        *reinterpret_cast<float4 *>(&Bs[kk][c]) = b;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        const float4 a4 = *reinterpret_cast<const float4 *>(&As[kk][ty * 4]);
        const float4 b4 = *reinterpret_cast<const float4 *>(&Bs[kk][tx * 4]);
        const float av[4] = {a4.x, a4.y, a4.z, a4.w};
        const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
    const uint32_t u0 = ub * 64 + tx * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t row = r0 + ty * 4 + i;
      if (row >= Q) continue;
      const uint32_t dst = P.row_dst[row];
      if (dst == NONE) continue;
      const float *hp = P.state + (size_t)P.row_src[row] * H;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t u = u0 + j;
        if (u >= H) continue;
        const size_t o = (size_t)row * H + u;
        float hn;
        if (rnn) {                                           // vanilla RNN: sigma(Wh x + bh + Uh h)
          hn = sigmoidf_(P.g_wxb[o] + acc[i][j]);
        } else {
          const float z = P.g_z[o];
          const float c = tanhf(P.g_wxb[o] + (lbr ? P.g_rh[o] * acc[i][j] : acc[i][j]));
          hn = (1.0f - z) * hp[u] + z * c;
        }
        P.state[(size_t)dst * H + u] = hn;
      }
    }
  }
}

}  // namespace rnnlm_dev

namespace rnnlm_host {
using namespace rnnlm_dev;

int launch_gru_simt(const Params &P, uint32_t max_rows, int num_sms, cudaStream_t s) {
  if (!max_rows) return 0;
  const uint32_t nub = P.Hp / 64;
  const uint32_t tiles = (max_rows + BM - 1) / BM;
  uint32_t gy = ((uint32_t)num_sms * 2 + nub - 1) / nub;
  if (gy > tiles) gy = tiles;
  if (gy < 1) gy = 1;
  launch_pdl(k_gru1_f32, dim3(nub, gy), NT, 0, s, P);
  launch_pdl(k_gru2_f32, dim3(nub, gy), NT, 0, s, P);
  return 2;
}
}  // namespace rnnlm_host
