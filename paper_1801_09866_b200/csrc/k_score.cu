// k_score.cu -- step (a6): unnormalised NCE score + hashed MaxEnt bypass.
//
// "the only required computations are inner products between the GRU outputs
// and NCE weights corresponding to the current word"; "an n-gram based
// MaxEnt bypass ... we implemented a hash-based MaxEnt ... to retrieve a
// probability for the given n-gram in constant time"; the two
// "operate as an ensemble model": additive in log-score space
// (reading 13).  The score conditions on the PARENT history (reading 2), so
// this kernel does not depend on this call's GRU work.
//
// Eight lanes per non-QHIT query (compacted list from k_commit), four queries
// per warp: lanes stream the word's output row (fp32, or bf16 when every entry
// is bf16-exact) and the parent state with 16-byte loads, then a fixed
// xor-butterfly reduction over the eight lanes (deterministic, independent of
// the batch).  Lane k < K of the group evaluates the order-(k+1) MaxEnt index
// and gathers one table entry; the K values are added in order 1..K.
//   idx_1 = w mod M;  idx_k = (idx_{k-1} * 237967 + ctx_{k-1} + 1) mod M
// (reading 11; ctx_{k-1} = (k-1)-th most recent word, u64).
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
// flight), then a fixed xor-tree over the eight lanes.
__global__ void __launch_bounds__(128) k_score(Params P, CallArgs A) {
  pdl_entry();
  const uint32_t total = P.counts[0];
  const uint32_t lane = threadIdx.x & 31, gid = lane >> 3, gl = lane & 7;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (uint32_t base = wg * 4; base < total; base += nw * 4) {
    const uint32_t i = base + gid;
    ScoreItem it;
    it.pr.slot = NONE;
    for (int j = 0; j < MAX_CTX; ++j) it.pr.ctx[j] = NONE;
    it.q = it.s = it.w = 0u;
    if (i < total) it = P.score_items[i];               // one 48-byte record per query (k_commit)
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

// rnnlm_maxent_indices: n x N u64 (UINT64_MAX beyond K).
__global__ void k_maxent_indices(Params P, uint32_t n, const uint32_t *__restrict__ sess,
                                 const uint32_t *__restrict__ par, const uint32_t *__restrict__ word,
                                 unsigned long long *__restrict__ out) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const uint32_t s = sess[q], p = par[q], w = word[q];
  const bool ok = s < P.S && p < P.ctr[s].next_handle;
  Rec r;
  if (ok) r = P.rec[(size_t)s * P.cap + p];
  const uint32_t K = ok ? min(P.N, ctx_len(r, P.N) + 1) : 0;
  for (uint32_t k = 0; k < P.N; ++k)
    out[(size_t)q * P.N + k] = k < K ? maxent_index(r, w, k + 1, P.M_mask) : ~0ull;
}

}  // namespace rnnlm_dev

namespace rnnlm_host {
using namespace rnnlm_dev;

int launch_score(const Params &P, const CallArgs &A, int num_sms, cudaStream_t s) {
  if (!A.n) return 0;
  // 128-thread blocks (four warps) so that they fit beside a GRU CTA on the same SM
  uint32_t blocks = (A.n + 15) / 16;                  // <= one 8-lane group per query
  const uint32_t cap = (uint32_t)num_sms * 8;
  if (blocks > cap) blocks = cap;
  launch_pdl(k_score, blocks, 128, 0, s, P, A);
  return 1;
}

int launch_maxent_indices(const Params &P, uint32_t n, const uint32_t *sess, const uint32_t *par,
                          const uint32_t *word, unsigned long long *out, cudaStream_t s) {
  if (!n) return 0;
  k_maxent_indices<<<(n + 255) / 256, 256, 0, s>>>(P, n, sess, par, word, out);
  return 1;
}
}  // namespace rnnlm_host
