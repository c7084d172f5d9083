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
// A rows gathered through row_word / row_src; fp32 accumulation.  This is the 1e-5 path; the
// tensor-core path lives in k_gru_tc.cu.
#include "rnnlm_impl.cuh"

namespace rnnlm_dev {

constexpr int BM = 128, BU = 64, BK = 16, NT = 256, AST = BM + 4;
constexpr int BU2 = 128;                  // phase-2 units per tile

__device__ __forceinline__ float sigmoidf_(float a) { return 1.0f / (1.0f + expf(-a)); }

// Register-tiled FFMA: 128-row tiles, 256 threads as 16 x 16; a thread owns 8
// rows x (3 gates x 4 units) in phase 1 and 8 rows x 8 units in phase 2, so
// one K step costs 5 (4) shared loads for 96 (64) FMAs.  The next K slice is
// fetched from global into registers while the current one is multiplied.
__global__ void __launch_bounds__(NT) k_gru1_f32(Params P) {
  pdl_entry();
  __shared__ __align__(16) float As[BK][AST];
  __shared__ __align__(16) float Bs[BK][3 * BU];
  const uint32_t Q = P.counts[1];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const uint32_t nub = P.Hp / 64, ntile = (Q + BM - 1) / BM;
  const uint32_t E = P.E, H = P.H;
  const int lr = tid >> 2, lk = (tid & 3) * 4;          // A loader: rows lr, lr + 64; k lk..lk+3
  // persistent: (unit block, row tile) work items, unit block fastest (weights stay in L2)
  for (uint32_t w = blockIdx.x; w < nub * ntile; w += gridDim.x) {
    const uint32_t ub = w % nub, r0 = (w / nub) * BM;
    float acc[3][8][4];
#pragma unroll
    for (int g = 0; g < 3; ++g)
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[g][i][j] = 0.0f;
    const bool rv0 = r0 + lr < Q, rv1 = r0 + lr + 64 < Q;
    const float *xs0 = rv0 ? P.emb + (size_t)P.row_word[r0 + lr] * E : P.emb;
    const float *xs1 = rv1 ? P.emb + (size_t)P.row_word[r0 + lr + 64] * E : P.emb;
    const float *hs0 = rv0 ? P.state + (size_t)P.row_src[r0 + lr] * H : P.state;
    const float *hs1 = rv1 ? P.state + (size_t)P.row_src[r0 + lr + 64] * H : P.state;
    // two K ranges: x part (3 gates, w1x) then h part (z, r gates, w1h)
    for (int part = 0; part < 2; ++part) {
      const uint32_t K = part == 0 ? E : H;
      const int ng = part == 0 ? 3 : 2;
      const float *a0p = part == 0 ? xs0 : hs0, *a1p = part == 0 ? xs1 : hs1;
      const float *wp = part == 0 ? P.w1x : P.w1h;
      float4 ra0, ra1, rb[3];
      auto fetch = [&](uint32_t k0) {
        ra0 = (rv0 && k0 + lk < K) ? *reinterpret_cast<const float4 *>(a0p + k0 + lk) : make_float4(0.f, 0.f, 0.f, 0.f);
        ra1 = (rv1 && k0 + lk < K) ? *reinterpret_cast<const float4 *>(a1p + k0 + lk) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int f = tid + i * NT, kk = f / (ng * 16), c = (f % (ng * 16)) * 4;
          rb[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (i < ng && k0 + kk < K)
            rb[i] = __ldg(reinterpret_cast<const float4 *>(wp + ((size_t)(k0 + kk) * nub + ub) * (ng * 64) + c));
        }
      };
      auto store = [&]() {
        As[lk + 0][lr] = ra0.x; As[lk + 1][lr] = ra0.y; As[lk + 2][lr] = ra0.z; As[lk + 3][lr] = ra0.w;
        As[lk + 0][lr + 64] = ra1.x; As[lk + 1][lr + 64] = ra1.y; As[lk + 2][lr + 64] = ra1.z; As[lk + 3][lr + 64] = ra1.w;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          if (i >= ng) break;
          const int f = tid + i * NT, kk = f / (ng * 16), c = (f % (ng * 16)) * 4;
          *reinterpret_cast<float4 *>(&Bs[kk][c]) = rb[i];
        }
      };
      fetch(0);
      for (uint32_t k0 = 0; k0 < K; k0 += BK) {
        __syncthreads();
        store();
        __syncthreads();
        if (k0 + BK < K) fetch(k0 + BK);                 // in flight during the FMAs below
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
          const float4 a4 = *reinterpret_cast<const float4 *>(&As[kk][ty * 8]);
          const float4 a5 = *reinterpret_cast<const float4 *>(&As[kk][ty * 8 + 4]);
          const float av[8] = {a4.x, a4.y, a4.z, a4.w, a5.x, a5.y, a5.z, a5.w};
#pragma unroll
          for (int g = 0; g < 3; ++g) {
            if (g >= ng) break;
            const float4 b4 = *reinterpret_cast<const float4 *>(&Bs[kk][g * 64 + tx * 4]);
            const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) acc[g][i][j] = fmaf(av[i], bv[j], acc[g][i][j]);
          }
        }
      }
      __syncthreads();
    }
    // ---- epilogue: z, r . h (GRU) or r (LBR), Wh x + bh
    const uint32_t u0 = ub * 64 + tx * 4;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t row = r0 + ty * 8 + i;
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

__global__ void __launch_bounds__(NT, 2) k_gru2_f32(Params P) {
  pdl_entry();
  __shared__ __align__(16) float As[BK][AST];
  __shared__ __align__(16) float Bs[BK][BU2];
  const uint32_t Q = P.counts[1];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const uint32_t H = P.H, nub2 = (P.Hp + BU2 - 1) / BU2, ntile = (Q + BM - 1) / BM;
  const int lr = tid >> 2, lk = (tid & 3) * 4;
  const bool lbr = P.cell == RNNLM_CELL_GRU_LBR, rnn = P.cell == RNNLM_CELL_RNN;
  for (uint32_t w = blockIdx.x; w < nub2 * ntile; w += gridDim.x) {
    const uint32_t ub = w % nub2, r0 = (w / nub2) * BM;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
    const bool rv0 = r0 + lr < Q, rv1 = r0 + lr + 64 < Q;
    // A operand: r . h (GRU) or the parent state h itself (LBR: Uh h, reset applied after; RNN)
    auto arow = [&](bool rv, uint32_t lrow) -> const float * {
      if (!rv) return P.g_rh;
      return (lbr || rnn) ? P.state + (size_t)P.row_src[lrow] * H : P.g_rh + (size_t)lrow * H;
    };
    const float *as0 = arow(rv0, r0 + lr), *as1 = arow(rv1, r0 + lr + 64);
    float4 ra0, ra1, rb[2];
    auto fetch = [&](uint32_t k0) {
      ra0 = (rv0 && k0 + lk < H) ? *reinterpret_cast<const float4 *>(as0 + k0 + lk) : make_float4(0.f, 0.f, 0.f, 0.f);
      ra1 = (rv1 && k0 + lk < H) ? *reinterpret_cast<const float4 *>(as1 + k0 + lk) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int f = tid + i * NT, kk = f / 32, c = (f % 32) * 4;
        const uint32_t u = ub * BU2 + c;
        rb[i] = (k0 + kk < H && u < P.Hp)
                    ? __ldg(reinterpret_cast<const float4 *>(P.w2 + (size_t)(k0 + kk) * P.Hp + u))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    fetch(0);
    for (uint32_t k0 = 0; k0 < H; k0 += BK) {
      __syncthreads();
      As[lk + 0][lr] = ra0.x; As[lk + 1][lr] = ra0.y; As[lk + 2][lr] = ra0.z; As[lk + 3][lr] = ra0.w;
      As[lk + 0][lr + 64] = ra1.x; As[lk + 1][lr + 64] = ra1.y; As[lk + 2][lr + 64] = ra1.z; As[lk + 3][lr + 64] = ra1.w;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int f = tid + i * NT, kk = f / 32, c = (f % 32) * 4;
        *reinterpret_cast<float4 *>(&Bs[kk][c]) = rb[i];
      }
      __syncthreads();
      if (k0 + BK < H) fetch(k0 + BK);
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        const float4 a4 = *reinterpret_cast<const float4 *>(&As[kk][ty * 8]);
        const float4 a5 = *reinterpret_cast<const float4 *>(&As[kk][ty * 8 + 4]);
        const float4 b4 = *reinterpret_cast<const float4 *>(&Bs[kk][tx * 8]);
        const float4 b5 = *reinterpret_cast<const float4 *>(&Bs[kk][tx * 8 + 4]);
        const float av[8] = {a4.x, a4.y, a4.z, a4.w, a5.x, a5.y, a5.z, a5.w};
        const float bv[8] = {b4.x, b4.y, b4.z, b4.w, b5.x, b5.y, b5.z, b5.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
    }
    const uint32_t u0 = ub * BU2 + tx * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t row = r0 + ty * 8 + i;
      if (row >= Q) continue;
      const uint32_t dst = P.row_dst[row];
      if (dst == NONE) continue;
      const float *hp = P.state + (size_t)P.row_src[row] * H;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
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
    __syncthreads();
  }
}

}  // namespace rnnlm_dev

namespace rnnlm_host {
using namespace rnnlm_dev;

int launch_gru_simt(const Params &P, uint32_t max_rows, int num_sms, cudaStream_t s) {
  if (!max_rows) return 0;
  // persistent grids sized to the resident CTAs (1 per SM for phase 1, 2 for phase 2);
  // the row count is read on the device, so the grid is capped by the maximum
  const uint32_t tiles = (max_rows + BM - 1) / BM;
  const uint32_t nub = P.Hp / 64, nub2 = (P.Hp + BU2 - 1) / BU2;
  uint32_t g1 = nub * tiles, g2 = nub2 * tiles;
  if (g1 > (uint32_t)num_sms) g1 = num_sms;
  if (g2 > (uint32_t)num_sms * 2) g2 = num_sms * 2;
  launch_pdl(k_gru1_f32, g1, NT, 0, s, P);
  launch_pdl(k_gru2_f32, g2, NT, 0, s, P);
  return 2;
}
}  // namespace rnnlm_host
