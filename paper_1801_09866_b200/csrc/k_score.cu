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
#include "score.cuh"

namespace rnnlm_dev {

// register bound of the scoring kernel: it runs beside the fused GRU kernel,
// one warp per SM sub-partition in the 1,024 registers the GRU's three warps
// leave there (k_gru_tc.cu GRU_MAXREG)
#ifndef RNNLM_SCORE_MAXREG
#define RNNLM_SCORE_MAXREG 32
#endif
#define SCORE_BOUNDS __maxnreg__(RNNLM_SCORE_MAXREG)
__global__ void SCORE_BOUNDS k_score(Params P, CallArgs A) {
  pdl_entry();
  const uint32_t total = P.counts[0];
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (uint32_t base = wg * 4; base < total; base += nw * 4) score_quad(P, A, base, total);
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
