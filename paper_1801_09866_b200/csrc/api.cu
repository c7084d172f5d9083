// api.cu -- the C ABI (include/rnnlm.h): engine creation, pools, weight
// layouts, and the per-frame orchestration of rnnlm_query_batch.
#include <nvtx3/nvToolsExt.h>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "rnnlm_impl.cuh"

using namespace rnnlm_dev;

namespace rnnlm_host {
// Tensor-core path (k_gru_tc.cu).  Returns kernels launched, or -1 if the
// configuration is not supported by it.
int gru_tc_supported(uint32_t E, uint32_t H);
int gru_tc_prepare(const rnnlm_weights *w, uint32_t V, uint32_t E, uint32_t H, int tf32, int x3, int cell,
                   void **state_out);
void gru_tc_release(void *state);
int gru_tc_bind(void *state, void *rh, uint32_t bmax);
int gru_tc_weights(void *state, const void **w1, const void **w2, uint32_t *rw);
double gru_tc_x3_products(void *state);
// Small-frame GEMV path (k_gemv.cu).
int gemv_prepare(const Params &P, const rnnlm_weights *w, uint32_t math, const void *tc_w1, const void *tc_w2,
                 uint32_t tc_rw, uint32_t rows, void **state_out);
void gemv_release(void *state);
int launch_gemv(const Params &P, void *state, int num_sms, cudaStream_t s);
// Fused small-frame step (k_small.cu).
uint32_t small_max_queries();
int launch_small(const Params &P, const CallArgs &A, void *gemv_state, uint32_t *bar, int num_sms, cudaStream_t s);
int launch_gru_tc(const Params &P, void *tc_state, uint32_t max_rows, int num_sms, cudaStream_t s,
                  cudaEvent_t ev_gathered, cudaEvent_t ev_phase1, cudaEvent_t ev_fork);
// Exact log-normaliser (k_norm.cu).
int norm_supported(uint32_t H, uint32_t N);
int norm_prepare(const Params &P, uint32_t bmax, void **state_out, cudaStream_t s);
void norm_release(void *state);
int launch_norm(const Params &P, void *state, uint32_t n, const uint32_t *sess, const uint32_t *hist,
                float *log_z, int num_sms, cudaStream_t s);
}  // namespace rnnlm_host

struct rnnlm {
  rnnlm_config cfg{};
  Params P{};
  int num_sms = 148;
  std::vector<void *> allocs;
  void *tc = nullptr;                 // tensor-core GRU state (descriptors, weights)
  void *gemv = nullptr;               // small-frame GEMV path (k_gemv.cu), or null
  uint32_t gemv_max_n = 0;            // calls with n <= this run the GRU on it
  void *norm = nullptr;               // log-normaliser scratch (first rnnlm_log_normalizer call)
  uint64_t launches = 0;
  // scoring + result write run on a side stream, concurrently with the GRU
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // timing
  int timing = 0;
  std::vector<cudaEvent_t> ev_pool;
  struct Pending {
    std::vector<cudaEvent_t> ev;      // NEV events per timed call
    bool fused;                       // the call ran the fused small-frame kernel (ev[0] -> ev[1])
  };
  std::vector<Pending> ev_pending;
  uint32_t *bar = nullptr;            // grid barrier of the fused small-frame kernel
  rnnlm_timing acc{};
};

namespace {

// per timed call: [0] start, [1] fork (after commit), [2] final end, [3] score end (side
// stream), [4] gathered (level 2), [5] GRU end, [6] encode end (main stream)
constexpr int NEV = 7;

rnnlm_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return RNNLM_OK;
  return e == cudaErrorMemoryAllocation ? RNNLM_E_OOM : RNNLM_E_CUDA;
}

template <typename T>
rnnlm_status dalloc(rnnlm *h, T **p, size_t count) {
  *p = nullptr;
  if (count == 0) return RNNLM_OK;
  void *v = nullptr;
  cudaError_t e = cudaMalloc(&v, count * sizeof(T));
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return RNNLM_E_OOM;
  }
  h->allocs.push_back(v);
  *p = static_cast<T *>(v);
  return RNNLM_OK;
}

uint32_t next_pow2(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return (uint32_t)p;
}

bool all_finite(const float *p, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

bool all_bf16_exact(const float *p, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    uint32_t u;
    std::memcpy(&u, &p[i], 4);
    if (u & 0xFFFFu) return false;
  }
  return true;
}

uint32_t code_bytes_of(uint32_t mode, uint32_t k, uint32_t H) {
  if (mode == RNNLM_KEY_SIGN) return (H + 7) / 8;
  if (mode == RNNLM_KEY_ROUND) return k <= 2 ? H : 2 * H;
  return 4 * H;
}

template <typename T>
rnnlm_status upload(rnnlm *h, T **dst, const T *src, size_t count) {
  rnnlm_status st = dalloc(h, dst, count);
  if (st != RNNLM_OK) return st;
  return cuda_status(cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice));
}

rnnlm_status upload_bf16(rnnlm *h, __nv_bfloat16 **dst, const float *src, size_t count) {
  std::vector<__nv_bfloat16> tmp(count);
  for (size_t i = 0; i < count; ++i) tmp[i] = __float2bfloat16_rn(src[i]);
  return upload(h, dst, tmp.data(), count);
}

void free_all(rnnlm *h) {
  if (h->tc) rnnlm_host::gru_tc_release(h->tc);
  if (h->gemv) rnnlm_host::gemv_release(h->gemv);
  h->gemv = nullptr;
  h->tc = nullptr;
  if (h->norm) rnnlm_host::norm_release(h->norm);
  h->norm = nullptr;
  for (void *p : h->allocs) cudaFree(p);
  h->allocs.clear();
  for (auto &v : h->ev_pending)
    for (cudaEvent_t e : v.ev)
      if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  h->ev_pending.clear();
  h->ev_pool.clear();
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->side) cudaStreamDestroy(h->side);
  h->ev_fork = h->ev_join = nullptr;
  h->side = nullptr;
}

// NVTX range over a host-side scope (tracing): the calls and the
// enqueue of each hot-path row group show up on an nsys / ncu --nvtx timeline.
// Header-only NVTX3: a no-op unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Every call that launches or synchronises runs on the handle's device and
// restores the caller's current device on return (one handle per device).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const rnnlm *h) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != h->cfg.device) cudaSetDevice(h->cfg.device);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

cudaEvent_t take_event(rnnlm *h) {
  if (!h->ev_pool.empty()) {
    cudaEvent_t e = h->ev_pool.back();
    h->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

}  // namespace

extern "C" {

int rnnlm_abi_version(void) { return RNNLM_ABI_VERSION; }

const char *rnnlm_status_string(rnnlm_status s) {
  switch (s) {
    case RNNLM_OK: return "ok";
    case RNNLM_E_INVALID_ARG: return "invalid argument";
    case RNNLM_E_DIMENSION: return "invalid dimension";
    case RNNLM_E_NONFINITE: return "non-finite weight";
    case RNNLM_E_VOCAB: return "word id >= vocab";
    case RNNLM_E_HISTORY: return "unknown or unborn parent history";
    case RNNLM_E_CAPACITY: return "history capacity exhausted";
    case RNNLM_E_CUDA: return "CUDA error";
    case RNNLM_E_OOM: return "out of device memory";
  }
  return "unknown status";
}

uint32_t rnnlm_code_bytes(const rnnlm_t *h) { return h ? h->P.code_bytes : 0; }
uint64_t rnnlm_launch_count(const rnnlm_t *h) { return h ? h->launches : 0; }
double rnnlm_tf32x3_products(const rnnlm_t *h) { return h && h->tc ? rnnlm_host::gru_tc_x3_products(h->tc) : 0.0; }

rnnlm_status rnnlm_create(const rnnlm_config *cfg, const rnnlm_weights *w, rnnlm_t **out) {
  if (!out) return RNNLM_E_INVALID_ARG;
  *out = nullptr;
  if (!cfg || !w) return RNNLM_E_INVALID_ARG;
  const rnnlm_config c = *cfg;
  if (c.vocab < 2 || c.embed == 0 || c.hidden == 0 || c.embed % 8 || c.hidden % 8 ||
      c.maxent_order < 1 || c.maxent_order > 8 || c.maxent_log2 > 31 || c.num_sessions == 0 ||
      c.max_queries_per_call == 0 || c.max_histories_per_session < 2 ||
      c.max_histories_per_session > 0x7FFFFFFFu || c.max_queries_per_call > 0x7FFFFFFFu ||
      c.vocab > 0x7FFFFFFFu)
    return RNNLM_E_DIMENSION;
  if (c.key_mode > RNNLM_KEY_SIGN) return RNNLM_E_INVALID_ARG;
  if (c.key_mode == RNNLM_KEY_ROUND && (c.round_digits < 1 || c.round_digits > 4))
    return RNNLM_E_INVALID_ARG;
  if (c.math > RNNLM_MATH_BF16X3) return RNNLM_E_INVALID_ARG;
  const bool split = c.math == RNNLM_MATH_TF32X3 || c.math == RNNLM_MATH_BF16X3;   // fp32-accurate splits
  if (split && c.cell != RNNLM_CELL_GRU) return RNNLM_E_INVALID_ARG;
  if (c.cell > RNNLM_CELL_RNN) return RNNLM_E_INVALID_ARG;
  if (c.gru_path > RNNLM_GRU_GEMV) return RNNLM_E_INVALID_ARG;
  const bool tc = c.math != RNNLM_MATH_FP32;           // tcgen05 path (BF16 or TF32 operands)
  if (tc && !rnnlm_host::gru_tc_supported(c.embed, c.hidden))
    return RNNLM_E_DIMENSION;
  const size_t V = c.vocab, E = c.embed, H = c.hidden, M = (size_t)1 << c.maxent_log2;
  const float *arrs[] = {w->emb, w->Wz, w->Uz, w->bz, w->Wr, w->Ur, w->br,
                         w->Wh, w->Uh, w->bh, w->nce_w, w->nce_b, w->maxent};
  const size_t lens[] = {V * E, H * E, H * H, H, H * E, H * H, H, H * E, H * H, H, V * H, V, M};
  for (int i = 0; i < 13; ++i)
    if (!arrs[i]) return RNNLM_E_INVALID_ARG;
  for (int i = 0; i < 13; ++i)
    if (!all_finite(arrs[i], lens[i])) return RNNLM_E_NONFINITE;

  if (cudaSetDevice(c.device) != cudaSuccess) {
    (void)cudaGetLastError();
    return RNNLM_E_CUDA;
  }
  rnnlm *h = new (std::nothrow) rnnlm;
  if (!h) return RNNLM_E_OOM;
  h->cfg = c;
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, c.device);
  Params &P = h->P;
  P.V = c.vocab; P.E = c.embed; P.H = c.hidden; P.N = c.maxent_order; P.S = c.num_sessions;
  P.cap = c.max_histories_per_session;
  // Each session's tables hold >= cap + Bs keys at load <= 0.5, Bs = the most
  // queries one session has in one call: the keys claimed before a session's
  // first capacity failure (< cap) plus one call's worth of claims (<= Bs)
  // always fit, so claiming never depends on thread order.
  const uint64_t bs = c.max_queries_per_session_call && c.max_queries_per_session_call < c.max_queries_per_call
                          ? c.max_queries_per_session_call : c.max_queries_per_call;
  const uint32_t tcap = next_pow2(2ull * ((uint64_t)P.cap + bs));
  P.qmask = tcap - 1;
  P.hmask = tcap - 1;
  P.key_mode = c.key_mode; P.round_digits = c.round_digits; P.cache = c.cache_enabled ? 1 : 0;
  P.math = c.math;
  P.cell = c.cell;
  P.M_mask = (unsigned long long)M - 1;
  P.code_bytes = code_bytes_of(c.key_mode, c.round_digits, P.H);
  P.code_words = (P.code_bytes + 3) / 4;
  P.cstride = c.key_mode == RNNLM_KEY_OFF ? 0 : (P.code_bytes + 15) / 16 * 16;
  P.Hp = (P.H + 63) / 64 * 64;
  const float scales[5] = {1.0f, 10.0f, 100.0f, 1000.0f, 10000.0f};
  P.round_scale = c.key_mode == RNNLM_KEY_ROUND ? scales[c.round_digits] : 1.0f;

  rnnlm_status st = RNNLM_OK;
  const size_t S = c.num_sessions, cap = P.cap, B = c.max_queries_per_call;
  const size_t Hp = P.Hp, nub = Hp / 64;
  auto chk = [&](rnnlm_status s2) { if (st == RNNLM_OK) st = s2; };
  // ---- weights
  chk(upload(h, const_cast<float **>(&P.emb), w->emb, V * E));
  chk(upload(h, const_cast<float **>(&P.nce_b), w->nce_b, V));
  chk(upload(h, const_cast<float **>(&P.maxent), w->maxent, M));
  if (c.math == RNNLM_MATH_BF16 && all_bf16_exact(w->nce_w, V * H))
    chk(upload_bf16(h, const_cast<__nv_bfloat16 **>(&P.nce_w16), w->nce_w, V * H));
  else
    chk(upload(h, const_cast<float **>(&P.nce_w), w->nce_w, V * H));
  if (c.math == RNNLM_MATH_FP32) {
    std::vector<float> w1x(E * nub * 192, 0.0f), w1h(H * nub * 128, 0.0f), b1(nub * 192, 0.0f),
        w2(H * Hp, 0.0f);
    const float *Wg[3] = {w->Wz, w->Wr, w->Wh};
    const float *Ug[2] = {w->Uz, w->Ur};
    const float *bg[3] = {w->bz, w->br, w->bh};
    for (size_t u = 0; u < H; ++u) {
      const size_t ub = u / 64, uu = u % 64;
      for (int g = 0; g < 3; ++g) {
        for (size_t k = 0; k < E; ++k) w1x[(k * nub + ub) * 192 + g * 64 + uu] = Wg[g][u * E + k];
        b1[ub * 192 + g * 64 + uu] = bg[g][u];
      }
      for (int g = 0; g < 2; ++g)
        for (size_t k = 0; k < H; ++k) w1h[(k * nub + ub) * 128 + g * 64 + uu] = Ug[g][u * H + k];
      for (size_t k = 0; k < H; ++k) w2[k * Hp + u] = w->Uh[u * H + k];
    }
    chk(upload(h, const_cast<float **>(&P.w1x), w1x.data(), w1x.size()));
    chk(upload(h, const_cast<float **>(&P.w1h), w1h.data(), w1h.size()));
    chk(upload(h, const_cast<float **>(&P.b1), b1.data(), b1.size()));
    chk(upload(h, const_cast<float **>(&P.w2), w2.data(), w2.size()));
  } else {
    // bf16 embedding rows: the BF16 operands, and BF16X3's x_hi part when every entry is bf16-exact
    if (c.math == RNNLM_MATH_BF16 || (c.math == RNNLM_MATH_BF16X3 && all_bf16_exact(w->emb, V * E)))
      chk(upload_bf16(h, const_cast<__nv_bfloat16 **>(&P.emb16), w->emb, V * E));
    if (st == RNNLM_OK &&
        rnnlm_host::gru_tc_prepare(w, c.vocab, c.embed, c.hidden, c.math == RNNLM_MATH_TF32 || c.math == RNNLM_MATH_TF32X3,
                                   c.math == RNNLM_MATH_TF32X3 ? 2 : (c.math == RNNLM_MATH_BF16X3 ? 3 : 0),
                                   (int)c.cell, &h->tc) != 0)
      st = RNNLM_E_OOM;
  }
  // ---- pools
  chk(dalloc(h, &P.rec, S * cap));
  chk(dalloc(h, &P.state, S * cap * H));
  if (P.cache) {
    if (c.key_mode != RNNLM_KEY_OFF) chk(dalloc(h, &P.codes, S * cap * P.cstride));
    chk(dalloc(h, &P.codehash, S * cap));
    chk(dalloc(h, &P.qtab, S * tcap));
    chk(dalloc(h, &P.qowner, S * tcap));
    chk(dalloc(h, &P.htab, S * tcap));
    chk(dalloc(h, &P.howner, S * tcap));
    chk(dalloc(h, &P.phash, B));
  }
  chk(dalloc(h, &P.ctr, S));
  chk(dalloc(h, &P.sticky, 1));
  // ---- scratch
  uint32_t **u32s[] = {&P.st, &P.qent, &P.aux, &P.hent, &P.pslot, &P.cslot, &P.excl_nonq,
                       &P.excl_miss, &P.dup_list, &P.row_src, &P.row_dst, &P.row_word};
  for (uint32_t **p : u32s) chk(dalloc(h, p, B));
  chk(dalloc(h, &P.claimed, B));
  chk(dalloc(h, &P.score_items, B));
  uint32_t **segs[] = {&P.seg_excl_nonq, &P.seg_excl_miss, &P.seg_cnt_nonq, &P.seg_cnt_miss};
  for (uint32_t **p : segs) chk(dalloc(h, p, S));
  chk(dalloc(h, &P.tile_status, (B + rnnlm_host::SCAN_TILE - 1) / rnnlm_host::SCAN_TILE));
  chk(dalloc(h, &P.tile_ticket, 1));
  chk(dalloc(h, &P.counts, 4));
  chk(dalloc(h, &h->bar, 2));
  // z: the tensor-core path keeps it in 128-row blocks (k_gru_tc.cu zq4), so whole blocks
  chk(dalloc(h, &P.g_z, (B + 127) / 128 * 128 * H));
  if (c.math == RNNLM_MATH_FP32) chk(dalloc(h, &P.g_wxb, B * H));
  const bool rh16 = c.math == RNNLM_MATH_BF16 || c.math == RNNLM_MATH_BF16X3;
  if (rh16) chk(dalloc(h, &P.g_rh16, (c.math == RNNLM_MATH_BF16X3 ? 3 : 1) * B * H));   // BF16X3: [hi | mid | lo]
  else chk(dalloc(h, &P.g_rh, (c.math == RNNLM_MATH_TF32X3 ? 2 : 1) * B * H));      // 3xTF32: [hi | lo]
  if (st == RNNLM_OK && tc &&
      rnnlm_host::gru_tc_bind(h->tc, rh16 ? (void *)P.g_rh16 : (void *)P.g_rh,
                              (uint32_t)B) != 0)
    st = RNNLM_E_CUDA;
  if (st == RNNLM_OK && c.gru_path != RNNLM_GRU_TILES) {
    // small-frame GEMV path: calls of up to gemv_max_n queries (so <= that many GRU rows)
    h->gemv_max_n = c.gru_path == RNNLM_GRU_GEMV ? c.max_queries_per_call
                                                 : (c.max_queries_per_call < RNNLM_GEMV_AUTO_MAX_QUERIES
                                                        ? c.max_queries_per_call : RNNLM_GEMV_AUTO_MAX_QUERIES);
    const void *w1 = nullptr, *w2 = nullptr;
    uint32_t rw = 0;
    if (tc && !split) rnnlm_host::gru_tc_weights(h->tc, &w1, &w2, &rw);
    if (rnnlm_host::gemv_prepare(P, w, c.math, w1, w2, rw, h->gemv_max_n, &h->gemv) != 0) st = RNNLM_E_OOM;
  }
  if (st == RNNLM_OK) {
    // scoring + result write are short; give them priority over the GRU's CTAs
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    chk(cuda_status(cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, hi)));
  }
  if (st == RNNLM_OK) chk(cuda_status(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming)));
  if (st == RNNLM_OK) chk(cuda_status(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming)));
  if (st == RNNLM_OK) chk(cuda_status(cudaMemset(P.sticky, 0, sizeof(int))));
  if (st == RNNLM_OK) chk(cuda_status(cudaMemset(P.counts, 0, 4 * sizeof(uint32_t))));
  if (st == RNNLM_OK) chk(cuda_status(cudaMemset(h->bar, 0, 2 * sizeof(uint32_t))));
  if (st == RNNLM_OK) chk(cuda_status(cudaMemset(P.row_dst, 0xFF, B * sizeof(uint32_t))));
  if (st == RNNLM_OK) {
    st = rnnlm_reset_session(h, 0xFFFFFFFFu, nullptr);
    if (st == RNNLM_OK) st = cuda_status(cudaDeviceSynchronize());
  }
  if (st != RNNLM_OK) {
    free_all(h);
    delete h;
    (void)cudaGetLastError();
    return st;
  }
  *out = h;
  return RNNLM_OK;
}

void rnnlm_destroy(rnnlm_t *h) {
  if (!h) return;
  cudaSetDevice(h->cfg.device);
  cudaDeviceSynchronize();
  free_all(h);
  delete h;
}

rnnlm_status rnnlm_reset_session(rnnlm_t *h, uint32_t session, rnnlm_stream_t stream) {
  if (!h) return RNNLM_E_INVALID_ARG;
  DeviceGuard dg(h);
  const Params &P = h->P;
  uint32_t lo = session, hi = session + 1;
  if (session == 0xFFFFFFFFu) { lo = 0; hi = P.S; }
  else if (session >= P.S) return RNNLM_E_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t n = hi - lo, tcap = (size_t)P.qmask + 1;
  cudaError_t e = cudaSuccess;
  if (P.cache) {
    e = cudaMemsetAsync(P.qtab + lo * tcap, 0xFF, n * tcap * sizeof(QEntry), s);
    if (!e) e = cudaMemsetAsync(P.qowner + lo * tcap, 0xFF, n * tcap * sizeof(uint32_t), s);
    if (!e) e = cudaMemsetAsync(P.htab + lo * tcap, 0xFF, n * tcap * sizeof(HEntry), s);
    if (!e) e = cudaMemsetAsync(P.howner + lo * tcap, 0xFF, n * tcap * sizeof(uint32_t), s);
  }
  if (!e) e = cudaMemsetAsync(P.ctr + lo, 0, n * sizeof(SessCtr), s);
  if (e) return cuda_status(e);
  h->launches += rnnlm_host::launch_reset_root(P, lo, hi, s);
  // the root is handle 0 / slot 0: cursors start at 1
  std::vector<SessCtr> init(n);
  for (auto &c : init) { std::memset(&c, 0, sizeof c); c.next_handle = 1; c.next_slot = 1; }
  e = cudaMemcpyAsync(P.ctr + lo, init.data(), n * sizeof(SessCtr), cudaMemcpyHostToDevice, s);
  if (!e) e = cudaStreamSynchronize(s);     // init lives on the host stack
  return cuda_status(e);
}

}  // extern "C"

namespace {
// One call's kernels on stream s (k launches returned): (a1)-(a4) on the
// caller's stream, then the fork: (a6) scoring and (a7) result write depend
// only on the commit, the GRU (a5) too.  Scoring + result write go to the
// side stream and run beside the tensor-core GRU (co-resident CTAs); on the
// tensor-core path the fork is taken after the A1 gather, so the memory-bound
// gather has the GPU to itself.  s joins the side stream at the end.
int enqueue_step(rnnlm *h, const CallArgs &A, cudaStream_t s, bool timed) {
  const Params &P = h->P;
  std::vector<cudaEvent_t> ev;
  if (timed) {
    for (int i = 0; i < NEV; ++i) ev.push_back(take_event(h));
    cudaEventRecord(ev[0], s);
  }
  // a small frame on the AUTO path: the whole step is ONE cooperative kernel
  if (h->gemv && h->cfg.gru_path == RNNLM_GRU_AUTO && A.n <= h->gemv_max_n &&
      A.n <= rnnlm_host::small_max_queries()) {
    NvtxRange r("rnnlm fused small-frame step (a1-a7)");
    const int k = rnnlm_host::launch_small(P, A, h->gemv, h->bar, h->num_sms, s);
    cudaEventRecord(h->ev_join, s);                     // results ready (rnnlm_results_ready)
    if (timed) {
      cudaEventRecord(ev[1], s);
      for (int i = 2; i < NEV; ++i) { h->ev_pool.push_back(ev[i]); ev[i] = nullptr; }
      h->ev_pending.push_back({ev, true});
      h->acc.calls += 1;
      h->acc.launches += (uint64_t)(k > 0 ? k : 0);
    }
    return k > 0 ? k : 0;
  }
  int k = 0;
  {
    NvtxRange r("rnnlm (a1-a4) cache front + commit");
    k += rnnlm_host::launch_cache_front(P, A, s);
    k += rnnlm_host::launch_commit(P, A, s);
  }
  NvtxRange r5("rnnlm (a5) gather + GRU, (a6-a7) score + result");
  cudaEvent_t fork = h->ev_fork;
  if (timed) cudaEventRecord(ev[1], s);                 // ms_cache ends at the commit
  const bool gemv = h->gemv && A.n <= h->gemv_max_n;
  if (gemv) {                                           // small frame: GEMV kernels, codes encoded in place
    cudaEventRecord(fork, s);
    k += rnnlm_host::launch_gemv(P, h->gemv, h->num_sms, s);
  } else if (P.math != RNNLM_MATH_FP32) {
    k += rnnlm_host::launch_gru_tc(P, h->tc, A.n, h->num_sms, s, timed && h->timing >= 2 ? ev[4] : nullptr,
                                   nullptr, fork);
  } else {
    cudaEventRecord(fork, s);
    k += rnnlm_host::launch_gru_simt(P, A.n, h->num_sms, s);
  }
  cudaStreamWaitEvent(h->side, fork, 0);
  k += rnnlm_host::launch_final(P, A, h->side);
  if (timed) cudaEventRecord(ev[2], h->side);
  k += rnnlm_host::launch_score(P, A, h->num_sms, h->side);
  k += rnnlm_host::launch_dup_scores(P, A, h->num_sms, h->side);
  if (timed) cudaEventRecord(ev[3], h->side);
  cudaEventRecord(h->ev_join, h->side);
  if (timed) cudaEventRecord(ev[5], s);
  if (P.math == RNNLM_MATH_FP32 && !gemv)              // the tcgen05 / GEMV kernels encode in place
    k += rnnlm_host::launch_encode_rows(P, A.n, h->num_sms, s);
  if (timed) cudaEventRecord(ev[6], s);
  cudaStreamWaitEvent(s, h->ev_join, 0);
  if (timed) {
    if (h->timing < 2) { h->ev_pool.push_back(ev[4]); ev[4] = nullptr; }
    h->ev_pending.push_back({ev, false});
    h->acc.calls += 1;
    h->acc.launches += (uint64_t)k;
  }
  return k;
}
}  // namespace

struct rnnlm_graph {
  rnnlm *h = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int kernels = 0;
};

extern "C" {

rnnlm_status rnnlm_query_batch(rnnlm_t *h, uint32_t n, const uint32_t *d_session,
                               const uint32_t *d_parent, const uint32_t *d_word, float *d_score,
                               uint32_t *d_child, uint8_t *d_outcome, rnnlm_stream_t stream) {
  if (!h) return RNNLM_E_INVALID_ARG;
  NvtxRange nv("rnnlm_query_batch");
  DeviceGuard dg(h);
  if (n == 0) return RNNLM_OK;
  if (n > h->cfg.max_queries_per_call) return RNNLM_E_INVALID_ARG;
  if (!d_session || !d_parent || !d_word || !d_score || !d_child) return RNNLM_E_INVALID_ARG;
  CallArgs A;
  A.n = n;
  A.d_n = nullptr;
  A.session = d_session; A.parent = d_parent; A.word = d_word;
  A.score = d_score; A.child = d_child; A.outcome = d_outcome;
  h->launches += (uint64_t)enqueue_step(h, A, reinterpret_cast<cudaStream_t>(stream), h->timing != 0);
  return cuda_status(cudaGetLastError());
}

rnnlm_status rnnlm_graph_create(rnnlm_t *h, uint32_t max_n, const uint32_t *d_n, const uint32_t *d_session,
                                const uint32_t *d_parent, const uint32_t *d_word, float *d_score,
                                uint32_t *d_child, uint8_t *d_outcome, rnnlm_graph_t **out) {
  if (!out) return RNNLM_E_INVALID_ARG;
  *out = nullptr;
  if (!h || max_n == 0 || max_n > h->cfg.max_queries_per_call) return RNNLM_E_INVALID_ARG;
  if (!d_session || !d_parent || !d_word || !d_score || !d_child) return RNNLM_E_INVALID_ARG;
  DeviceGuard dg(h);
  CallArgs A;
  A.n = max_n;
  A.d_n = d_n;
  A.session = d_session; A.parent = d_parent; A.word = d_word;
  A.score = d_score; A.child = d_child; A.outcome = d_outcome;
  rnnlm_graph *g = new (std::nothrow) rnnlm_graph;
  if (!g) return RNNLM_E_OOM;
  g->h = h;
  cudaStream_t cs = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (!e) e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (!e) {
    g->kernels = enqueue_step(h, A, cs, false);
    e = cudaStreamEndCapture(cs, &g->graph);
  }
  if (!e) e = cudaGraphInstantiateWithFlags(&g->exec, g->graph, 0);
  if (cs) cudaStreamDestroy(cs);
  if (e) {
    (void)cudaGetLastError();
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
    return cuda_status(e);
  }
  *out = g;
  return RNNLM_OK;
}

rnnlm_status rnnlm_graph_launch(rnnlm_graph_t *g, rnnlm_stream_t stream) {
  if (!g) return RNNLM_E_INVALID_ARG;
  NvtxRange nv("rnnlm_graph_launch");
  DeviceGuard dg(g->h);
  g->h->launches += (uint64_t)g->kernels;
  return cuda_status(cudaGraphLaunch(g->exec, reinterpret_cast<cudaStream_t>(stream)));
}

void rnnlm_graph_destroy(rnnlm_graph_t *g) {
  if (!g) return;
  DeviceGuard dg(g->h);
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
}

rnnlm_status rnnlm_cache_stats(rnnlm_t *h, uint32_t session, rnnlm_stats *out) {
  if (!h || !out) return RNNLM_E_INVALID_ARG;
  DeviceGuard dg(h);
  const Params &P = h->P;
  if (session != 0xFFFFFFFFu && session >= P.S) return RNNLM_E_INVALID_ARG;
  cudaError_t e = cudaDeviceSynchronize();
  if (e) return cuda_status(e);
  std::vector<SessCtr> c(P.S);
  e = cudaMemcpy(c.data(), P.ctr, P.S * sizeof(SessCtr), cudaMemcpyDeviceToHost);
  int sticky = 0;
  if (!e) e = cudaMemcpy(&sticky, P.sticky, sizeof(int), cudaMemcpyDeviceToHost);
  if (e) return cuda_status(e);
  std::memset(out, 0, sizeof *out);
  for (uint32_t i = 0; i < P.S; ++i) {
    if (session != 0xFFFFFFFFu && session != i) continue;
    out->total_queries += c[i].total;
    out->query_hits += c[i].qhits;
    out->hidden_lookups += c[i].hlookups;
    out->hidden_hits += c[i].hhits;
    out->gru_computations += c[i].gru;
  }
  out->sticky_error = sticky;
  return (rnnlm_status)sticky;
}

rnnlm_status rnnlm_read_states(rnnlm_t *h, uint32_t session, uint32_t n, const uint32_t *d_handles,
                               float *d_states, rnnlm_stream_t stream) {
  if (!h || (n && (!d_handles || !d_states))) return RNNLM_E_INVALID_ARG;
  DeviceGuard dg(h);
  h->launches += rnnlm_host::launch_read_states(h->P, session, n, d_handles, d_states,
                                                reinterpret_cast<cudaStream_t>(stream));
  return cuda_status(cudaGetLastError());
}

rnnlm_status rnnlm_read_slots(rnnlm_t *h, uint32_t session, uint32_t n, const uint32_t *d_handles,
                              uint32_t *d_slots, rnnlm_stream_t stream) {
  if (!h || (n && (!d_handles || !d_slots))) return RNNLM_E_INVALID_ARG;
  DeviceGuard dg(h);
  h->launches += rnnlm_host::launch_read_slots(h->P, session, n, d_handles, d_slots,
                                               reinterpret_cast<cudaStream_t>(stream));
  return cuda_status(cudaGetLastError());
}

rnnlm_status rnnlm_read_codes(rnnlm_t *h, uint32_t session, uint32_t n, const uint32_t *d_handles,
                              uint8_t *d_codes, rnnlm_stream_t stream) {
  if (!h || (n && (!d_handles || !d_codes))) return RNNLM_E_INVALID_ARG;
  DeviceGuard dg(h);
  if (!h->P.cache && h->P.key_mode != RNNLM_KEY_OFF) return RNNLM_E_INVALID_ARG;  // no arena
  h->launches += rnnlm_host::launch_read_codes(h->P, session, n, d_handles, d_codes,
                                               reinterpret_cast<cudaStream_t>(stream));
  return cuda_status(cudaGetLastError());
}

rnnlm_status rnnlm_encode_states(rnnlm_t *h, uint32_t n, const float *d_states, uint8_t *d_codes,
                                 rnnlm_stream_t stream) {
  if (!h || (n && (!d_states || !d_codes))) return RNNLM_E_INVALID_ARG;
  DeviceGuard dg(h);
  Params P = h->P;
  if (P.key_mode != RNNLM_KEY_OFF && P.cstride == 0) return RNNLM_E_INVALID_ARG;
  h->launches += rnnlm_host::launch_encode_states(P, n, d_states, d_codes,
                                                  reinterpret_cast<cudaStream_t>(stream));
  return cuda_status(cudaGetLastError());
}

rnnlm_status rnnlm_maxent_indices(rnnlm_t *h, uint32_t n, const uint32_t *d_session,
                                  const uint32_t *d_parent, const uint32_t *d_word, uint64_t *d_idx,
                                  rnnlm_stream_t stream) {
  if (!h || (n && (!d_session || !d_parent || !d_word || !d_idx))) return RNNLM_E_INVALID_ARG;
  DeviceGuard dg(h);
  h->launches += rnnlm_host::launch_maxent_indices(
      h->P, n, d_session, d_parent, d_word, reinterpret_cast<unsigned long long *>(d_idx),
      reinterpret_cast<cudaStream_t>(stream));
  return cuda_status(cudaGetLastError());
}

rnnlm_status rnnlm_results_ready(rnnlm_t *h, rnnlm_stream_t stream) {
  if (!h) return RNNLM_E_INVALID_ARG;
  DeviceGuard dg(h);
  // every result write (k_commit on the caller's stream before the fork;
  // k_final, k_score, k_dup_scores on the side stream) precedes ev_join
  return cuda_status(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), h->ev_join, 0));
}

rnnlm_status rnnlm_log_normalizer(rnnlm_t *h, uint32_t n, const uint32_t *d_session,
                                  const uint32_t *d_history, float *d_log_z, rnnlm_stream_t stream) {
  if (!h) return RNNLM_E_INVALID_ARG;
  NvtxRange nv("rnnlm_query_batch");
  DeviceGuard dg(h);
  if (n == 0) return RNNLM_OK;
  if (n > h->cfg.max_queries_per_call || !d_session || !d_history || !d_log_z) return RNNLM_E_INVALID_ARG;
  if (!rnnlm_host::norm_supported(h->P.H, h->P.N)) return RNNLM_E_DIMENSION;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!h->norm) {
    if (rnnlm_host::norm_prepare(h->P, h->cfg.max_queries_per_call, &h->norm, s) != 0) return RNNLM_E_OOM;
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e);
  }
  h->launches += (uint64_t)rnnlm_host::launch_norm(h->P, h->norm, n, d_session, d_history, d_log_z,
                                                   h->num_sms, s);
  return cuda_status(cudaGetLastError());
}

rnnlm_status rnnlm_resolve_parents(uint32_t n, const int64_t *d_ref, const uint32_t *d_log,
                                   uint32_t *d_parent, rnnlm_stream_t stream) {
  if (n && (!d_ref || !d_log || !d_parent)) return RNNLM_E_INVALID_ARG;
  rnnlm_host::launch_resolve_parents(n, d_ref, d_log, d_parent,
                                     reinterpret_cast<cudaStream_t>(stream));
  return cuda_status(cudaGetLastError());
}

rnnlm_status rnnlm_set_timing(rnnlm_t *h, int level) {
  if (!h) return RNNLM_E_INVALID_ARG;
  h->timing = level < 0 ? 0 : level;
  return RNNLM_OK;
}

rnnlm_status rnnlm_get_timing(rnnlm_t *h, rnnlm_timing *out, int reset) {
  if (!h || !out) return RNNLM_E_INVALID_ARG;
  DeviceGuard dg(h);
  auto el = [](cudaEvent_t x, cudaEvent_t y) {
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, x, y);
    return (double)ms;
  };
  for (auto &pd : h->ev_pending) {
    auto &ev = pd.ev;
    if (pd.fused) {
      const cudaError_t e = cudaEventSynchronize(ev[1]);
      if (e) return cuda_status(e);
      h->acc.ms_fused += el(ev[0], ev[1]);
    } else {
      cudaError_t e = cudaEventSynchronize(ev[6]);
      if (!e) e = cudaEventSynchronize(ev[3]);
      if (e) return cuda_status(e);
      h->acc.ms_cache += el(ev[0], ev[1]);
      h->acc.ms_final += el(ev[1], ev[2]);
      h->acc.ms_score += el(ev[2], ev[3]);
      h->acc.ms_gru += el(ev[1], ev[5]);
      h->acc.ms_encode += el(ev[5], ev[6]);
      if (ev[4]) {
        h->acc.ms_gru_gather += el(ev[1], ev[4]);
        h->acc.ms_gru_phase1 += el(ev[4], ev[5]);
      }
    }
    for (cudaEvent_t e2 : ev)
      if (e2) h->ev_pool.push_back(e2);
  }
  h->ev_pending.clear();
  *out = h->acc;
  if (reset) h->acc = rnnlm_timing{};
  return RNNLM_OK;
}

}  // extern "C"
