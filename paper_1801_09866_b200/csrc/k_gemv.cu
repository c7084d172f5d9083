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

#include "gemv.cuh"

namespace rnnlm_gemv {

template <typename WT, int ACT, int CELL>
__global__ void __launch_bounds__(THREADS) k_gemv1(GemvArgs g) {
  pdl_entry();
  gemv1_item<WT, ACT, CELL>(g, g.counts[1], blockIdx.x, blockIdx.y, gridDim.y, threadIdx.x >> 5, THREADS / 32);
}

// Phase 2, then the last CTA to finish (threadfence reduction pattern)
// encodes every new state, one warp per row.
template <typename WT, int ACT, int CELL>
__global__ void __launch_bounds__(THREADS) k_gemv2(GemvArgs g) {
  pdl_entry();
  __shared__ uint32_t s_last;
  const uint32_t Q = g.counts[1];
  gemv2_item<WT, ACT, CELL>(g, Q, blockIdx.x, blockIdx.y, gridDim.y, threadIdx.x >> 5, THREADS / 32);
  if (!g.cache) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t t = atomicAdd(g.done, 1u);
    s_last = t == gridDim.x * gridDim.y - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  gemv_encode(g, Q, threadIdx.x >> 5, THREADS / 32);
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

// The kernels' arguments for the engine's pools (k_small.cu uses them too).
int gemv_args(void *state, const Params &P, GemvArgs *out, int *act) {
  GemvState *st = static_cast<GemvState *>(state);
  if (!st) return -1;
  GemvArgs g = st->g;
  g.emb = P.emb; g.emb16 = P.emb16; g.state = P.state;
  g.row_src = P.row_src; g.row_dst = P.row_dst; g.row_word = P.row_word; g.counts = P.counts;
  g.cache = P.cache; g.cstride = P.cstride; g.codes = P.codes; g.codehash = P.codehash;
  g.key = KeySpec{P.key_mode, P.round_digits, P.H, P.round_scale};
  *out = g;
  *act = st->act;
  return 0;
}

// Rows per call are <= st->rows (checked by the caller).
int launch_gemv(const Params &P, void *state, int num_sms, cudaStream_t s) {
  GemvState *st = static_cast<GemvState *>(state);
  GemvArgs g;
  int act = 0;
  gemv_args(state, P, &g, &act);
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
