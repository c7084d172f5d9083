// score.cuh -- step (a6) device functions (the NCE gather-dot + hashed MaxEnt
// score of one warp's four non-QHIT queries), shared by k_score (k_score.cu)
// and the fused small-frame kernel (k_small.cu).  Semantics: k_score.cu.
#pragma once

#include "rnnlm_impl.cuh"

namespace rnnlm_dev {

__device__ __forceinline__ uint32_t ctx_len(const Rec &r, uint32_t N) {
  uint32_t n = 0;
  for (uint32_t j = 0; j + 1 < N && j < (uint32_t)MAX_CTX; ++j) n += (r.ctx[j] != NONE);
  return n;
}

// MaxEnt index of order k (1-based) for word w and record r.
__device__ __forceinline__ unsigned long long maxent_index(const Rec &r, uint32_t w, uint32_t k,
                                                           unsigned long long mask) {
  unsigned long long idx = (unsigned long long)w & mask;
  for (uint32_t j = 2; j <= k; ++j) idx = (idx * 237967ull + (unsigned long long)r.ctx[j - 2] + 1ull) & mask;
  return idx;
}

__device__ __forceinline__ float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

// Four queries per warp, eight lanes per query: each lane streams H/8 output
// weights and state elements with 16-byte loads (many independent loads in
// flight), then a fixed xor-tree over the eight lanes.  Warp-collective: the
// warp scores work items [base, base + 4) of the call's non-QHIT list.
__device__ __forceinline__ void score_quad(const Params &P, const CallArgs &A, uint32_t base, uint32_t total) {
  const uint32_t lane = threadIdx.x & 31, gid = lane >> 3, gl = lane & 7;
  {
    const uint32_t i = base + gid;
    ScoreItem it;
    it.pr.slot = NONE;
    for (int j = 0; j < MAX_CTX; ++j) it.pr.ctx[j] = NONE;
    it.q = it.s = it.w = 0u;
    if (i < total) it = P.score_items[i];               // one record per query (k_commit)
    const bool act = i < total && it.pr.slot != NONE;
    const uint32_t q = it.q, s = act ? it.s : 0u, w = act ? it.w : 0u;
    Rec pr = it.pr;
    if (!act) pr.slot = 0;
    const float *h = P.state + ((size_t)s * P.cap + pr.slot) * P.H;
    // the MaxEnt weight and the output bias depend only on the record and the
    // word: issue them before the dot product so their latency overlaps it
    const uint32_t K = act ? min(P.N, ctx_len(pr, P.N) + 1) : 0u;
    float me = 0.0f;
    if (gl < K) me = __ldg(P.maxent + maxent_index(pr, w, gl + 1, P.M_mask));
    const float bias = act ? __ldg(P.nce_b + w) : 0.0f;
    float acc = 0.0f;
    if (act) {
      if (P.nce_w16) {
        const uint4 *row = reinterpret_cast<const uint4 *>(P.nce_w16 + (size_t)w * P.H);
#pragma unroll 4
        for (uint32_t j = gl; j < P.H / 8; j += 8) {
          const uint4 t = __ldg(row + j);
          const float4 h0 = reinterpret_cast<const float4 *>(h)[2 * j];
          const float4 h1 = reinterpret_cast<const float4 *>(h)[2 * j + 1];
          acc = fmaf(bf16lo(t.x), h0.x, acc); acc = fmaf(bf16hi(t.x), h0.y, acc);
          acc = fmaf(bf16lo(t.y), h0.z, acc); acc = fmaf(bf16hi(t.y), h0.w, acc);
          acc = fmaf(bf16lo(t.z), h1.x, acc); acc = fmaf(bf16hi(t.z), h1.y, acc);
          acc = fmaf(bf16lo(t.w), h1.z, acc); acc = fmaf(bf16hi(t.w), h1.w, acc);
        }
      } else {
        const float4 *row = reinterpret_cast<const float4 *>(P.nce_w + (size_t)w * P.H);
#pragma unroll 4
        for (uint32_t j = gl; j < P.H / 4; j += 8) {
          const float4 t = __ldg(row + j);
          const float4 hv = reinterpret_cast<const float4 *>(h)[j];
          acc = fmaf(t.x, hv.x, acc); acc = fmaf(t.y, hv.y, acc);
          acc = fmaf(t.z, hv.z, acc); acc = fmaf(t.w, hv.w, acc);
        }
      }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    float sc = acc + bias;
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k) {
      const float v = __shfl_sync(0xffffffffu, me, (lane & ~7u) + k);
      if (k < K) sc += v;
    }
    if (act && gl == 0) {
      A.score[q] = sc;
      if (P.cache) P.qtab[(size_t)s * (P.qmask + 1) + P.qent[q]].score = sc;
    }
  }
}

}  // namespace rnnlm_dev
