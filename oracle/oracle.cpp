// oracle.cpp -- CPU oracle of the frame-batched GRU-RNNLM query step.
//
// TEST INFRASTRUCTURE ONLY (see oracle.h).  Nothing here is used by, or uses,
// the CUDA path.  Citations: P:n = PAPER.md line n; S:n = SPEC.md line n;
// "reading k" = SURVEY.md 8(c) ambiguity table row k (listed in DESIGN.md).
//
// Build: g++ -O2 -fno-fast-math -ffp-contract=off -shared -fPIC (see
// __graft_entry__.build).  No FMA contraction, no fast-math: every fp32
// operation below is the one written.
#include "oracle.h"

#ifdef _OPENMP
#include <omp.h>
#endif

#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

namespace {

struct Record {                 // a history: its state slot and word context
  uint32_t slot;
  std::vector<uint32_t> ctx;    // last <= N-1 words, MOST RECENT LAST
};

struct Session {
  std::vector<Record> rec;                   // by history handle
  std::vector<std::vector<float>> state;     // by state slot, fp32 (reading 15)
  // LM-query cache: (history, word) -> (score, child)       (Fig. 1)
  std::map<std::pair<uint32_t, uint32_t>, std::pair<float, uint32_t>> qcache;
  // history-vector cache: (word, compressed history) -> slot (Fig. 2)
  std::map<std::pair<uint32_t, std::string>, uint32_t> hcache;
  uint64_t total = 0, query_hits = 0, hidden_lookups = 0, hidden_hits = 0, gru = 0;
  int sticky = 0;
  bool poisoned = false;        // ran out of handles: later frames are rejected until reset
};

struct Pending {                // a GRU evaluation owed at the end of the frame
  uint32_t session, slot, word, parent_slot;
};

}  // namespace

struct orc {
  orc_config cfg;
  orc_weights w;
  std::vector<Session> sess;
};

extern "C" {

uint32_t orc_code_bytes(uint32_t mode, uint32_t k, uint32_t H) {
  if (mode == ORC_KEY_SIGN) return (H + 7) / 8;
  if (mode == ORC_KEY_ROUND) return k <= 2 ? H : 2 * H;
  return 4 * H;
}

// compress(h, mode) -- "quantize the history vectors by controlling the
// precision ... rounding up to a specified decimal point" and "store
// only the signs of each element".
//   sign:    bit i = (h_i >= 0.0f); bit i lives in byte i/8 at bit i%8.  0 and
//            -0 give 1 (reading 5).
//   round:k: q_i = (int) roundf(h_i * 10^k), the product taken in fp32, C
//            roundf = half away from zero (readings 3, 4); int8 for k <= 2,
//            little-endian int16 for k = 3, 4 (reading 6).
//   off:     the 32-bit patterns of h (exact key, P:95-style dedup of vectors).
int orc_compress(uint32_t mode, uint32_t k, uint32_t H, const float *h, uint8_t *code) {
  for (uint32_t i = 0; i < H; ++i)
    if (!std::isfinite(h[i])) return ORC_E_NONFINITE;
  if (mode == ORC_KEY_SIGN) {
    std::memset(code, 0, (H + 7) / 8);
    for (uint32_t i = 0; i < H; ++i)
      if (h[i] >= 0.0f) code[i / 8] |= (uint8_t)(1u << (i % 8));
    return ORC_OK;
  }
  if (mode == ORC_KEY_ROUND) {
    float scale;
    if (k == 1) scale = 10.0f;
    else if (k == 2) scale = 100.0f;
    else if (k == 3) scale = 1000.0f;
    else if (k == 4) scale = 10000.0f;
    else return ORC_E_INVALID_ARG;
    for (uint32_t i = 0; i < H; ++i) {
      float prod = h[i] * scale;            // fp32 product (reading 4)
      int q = (int)roundf(prod);
      if (k <= 2) {
        int8_t b = (int8_t)q;
        std::memcpy(code + i, &b, 1);
      } else {
        int16_t b = (int16_t)q;
        std::memcpy(code + 2 * i, &b, 2);   // x86-64: little-endian
      }
    }
    return ORC_OK;
  }
  if (mode == ORC_KEY_OFF) {
    std::memcpy(code, h, 4 * (size_t)H);
    return ORC_OK;
  }
  return ORC_E_INVALID_ARG;
}

// Hash-based MaxEnt features ("we implemented a hash-based MaxEnt").
// The paper gives no hash; SPEC S:177 fixes it (reading 11):
//   idx_1 = w mod M
//   idx_k = (idx_{k-1} * 237967 + ctx[(k-1)-th most recent] + 1) mod M,
//   k = 2 .. min(N, |ctx|+1), unsigned 64-bit before each modulus.
uint32_t orc_maxent_indices(const uint32_t *ctx, uint32_t ctx_len, uint32_t w, uint32_t N,
                            uint64_t M, uint64_t *idx) {
  uint32_t K = N < ctx_len + 1 ? N : ctx_len + 1;
  if (K == 0) return 0;
  idx[0] = (uint64_t)w % M;
  for (uint32_t k = 2; k <= K; ++k) {
    uint64_t c = ctx[ctx_len - (k - 1)];   // (k-1)-th most recent word
    idx[k - 1] = (idx[k - 2] * 237967ull + c + 1ull) % M;
  }
  return K;
}

static double sigmoid(double a) { return 1.0 / (1.0 + std::exp(-a)); }

// GRU hidden layer ("for each gate and a candidate activation, two
// weight matrices and one bias vector"), gate equations of the cited GRU
// (Chung 2014; reading 1):
//   z  = sigma(Wz x + Uz h + bz)
//   r  = sigma(Wr x + Ur h + br)
//   h~ = tanh(Wh x + Uh (r . h) + bh)
//   h' = (1 - z) . h + z . h~
// fp64 accumulation in ascending index order, one rounding to fp32 (reading 16).
// Cell variant (cfg->cell = ORC_CELL_GRU_LBR): the reset gate
// applied AFTER the recurrent product ("linear before reset"):
//   h~ = tanh(Wh x + bh + r . (Uh h))
// with the same z, r and update; every other step of the method is unchanged.
// Cell variant ORC_CELL_RNN: the paper's comparison "vanilla-RNNLM"
// as the Elman layer of the RNNLM it cites, h' = sigma(Wh x + Uh h + bh).
void orc_gru(const orc_config *cfg, const orc_weights *w, const float *x, const float *h,
             double *out64, float *out32) {
  const uint32_t H = cfg->H, E = cfg->E;
  std::vector<double> z(H), r(H), rh(H);
  for (uint32_t i = 0; i < H; ++i) {
    double az = 0.0, ar = 0.0, uz = 0.0, ur = 0.0;
    for (uint32_t j = 0; j < E; ++j) {
      az += (double)w->Wz[(size_t)i * E + j] * (double)x[j];
      ar += (double)w->Wr[(size_t)i * E + j] * (double)x[j];
    }
    for (uint32_t j = 0; j < H; ++j) {
      uz += (double)w->Uz[(size_t)i * H + j] * (double)h[j];
      ur += (double)w->Ur[(size_t)i * H + j] * (double)h[j];
    }
    z[i] = sigmoid(az + uz + (double)w->bz[i]);
    r[i] = sigmoid(ar + ur + (double)w->br[i]);
  }
  const bool lbr = cfg->cell == ORC_CELL_GRU_LBR, rnn = cfg->cell == ORC_CELL_RNN;
  for (uint32_t j = 0; j < H; ++j) rh[j] = (lbr || rnn) ? (double)h[j] : r[j] * (double)h[j];
  for (uint32_t i = 0; i < H; ++i) {
    double ax = 0.0, au = 0.0;
    for (uint32_t j = 0; j < E; ++j) ax += (double)w->Wh[(size_t)i * E + j] * (double)x[j];
    for (uint32_t j = 0; j < H; ++j) au += (double)w->Uh[(size_t)i * H + j] * rh[j];
    double cand = lbr ? std::tanh(ax + (double)w->bh[i] + r[i] * au) : std::tanh(ax + au + (double)w->bh[i]);
    double hn = rnn ? sigmoid(ax + au + (double)w->bh[i]) : (1.0 - z[i]) * (double)h[i] + z[i] * cand;
    if (out64) out64[i] = hn;
    if (out32) out32[i] = (float)hn;
  }
}

// Unnormalised NCE score ("the only required computations are inner
// products between the GRU outputs and NCE weights corresponding to the
// current word"; no normalisation, reading 12) of the PARENT history (reading
// 2) plus the hashed MaxEnt bypass as an additive ensemble (reading 13).
float orc_score(const orc_config *cfg, const orc_weights *wt, const float *h,
                const uint32_t *ctx, uint32_t ctx_len, uint32_t w) {
  const uint32_t H = cfg->H;
  double acc = 0.0;
  for (uint32_t i = 0; i < H; ++i) acc += (double)wt->nce_w[(size_t)w * H + i] * (double)h[i];
  acc += (double)wt->nce_b[w];
  uint64_t idx[16];
  uint32_t K = orc_maxent_indices(ctx, ctx_len, w, cfg->N, 1ull << cfg->maxent_log2, idx);
  for (uint32_t k = 0; k < K; ++k) acc += (double)wt->maxent[idx[k]];
  return (float)acc;
}

// Exact log-normaliser of the combined score over the whole vocabulary: the
// normalisation NCE avoids at run time ("they need to be normalized over
// different word sequences ... a highly computationally intensive task",
// P:73-74; SPEC exact_log_prob S:201-209).
//   log Z(h, ctx) = log sum_{v < V} exp(s_v),
//   s_v = Theta_v . h + b_v + sum_k maxent[idx_k(ctx, v)]
// i.e. orc_score's sum for every word v, kept in fp64 (no fp32 rounding),
// then max-subtraction: log Z = m + log sum_v exp(s_v - m), m = max_v s_v,
// words in ascending order.
double orc_log_normalizer(const orc_config *cfg, const orc_weights *wt, const float *h,
                          const uint32_t *ctx, uint32_t ctx_len) {
  const uint32_t H = cfg->H, V = cfg->V;
  std::vector<double> s(V);
  uint64_t idx[16];
  for (uint32_t v = 0; v < V; ++v) {
    double acc = 0.0;
    for (uint32_t i = 0; i < H; ++i) acc += (double)wt->nce_w[(size_t)v * H + i] * (double)h[i];
    acc += (double)wt->nce_b[v];
    const uint32_t K = orc_maxent_indices(ctx, ctx_len, v, cfg->N, 1ull << cfg->maxent_log2, idx);
    for (uint32_t k = 0; k < K; ++k) acc += (double)wt->maxent[idx[k]];
    s[v] = acc;
  }
  double m = -INFINITY;
  for (uint32_t v = 0; v < V; ++v) m = s[v] > m ? s[v] : m;
  double z = 0.0;
  for (uint32_t v = 0; v < V; ++v) z += std::exp(s[v] - m);
  return m + std::log(z);
}

static int check_finite(const float *p, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return 0;
  return 1;
}

orc_t *orc_create(const orc_config *cfg, const orc_weights *w, int *status) {
  int st = ORC_OK;
  if (!cfg || !w) st = ORC_E_INVALID_ARG;
  else if (cfg->V < 2 || cfg->E == 0 || cfg->H == 0 || cfg->N == 0 || cfg->N > 8 ||
           cfg->maxent_log2 > 40 || cfg->num_sessions == 0 || cfg->max_histories < 2)
    st = ORC_E_DIMENSION;
  else if (cfg->key_mode > 2 || (cfg->key_mode == ORC_KEY_ROUND &&
                                 (cfg->round_digits < 1 || cfg->round_digits > 4)))
    st = ORC_E_INVALID_ARG;
  if (st == ORC_OK) {
    const size_t V = cfg->V, E = cfg->E, H = cfg->H, M = (size_t)1 << cfg->maxent_log2;
    const float *arrs[] = {w->emb, w->Wz, w->Uz, w->bz, w->Wr, w->Ur, w->br,
                           w->Wh, w->Uh, w->bh, w->nce_w, w->nce_b, w->maxent};
    const size_t lens[] = {V * E, H * E, H * H, H, H * E, H * H, H, H * E, H * H, H,
                           V * H, V, M};
    for (int i = 0; i < 13 && st == ORC_OK; ++i) {
      if (!arrs[i]) st = ORC_E_INVALID_ARG;
      else if (!check_finite(arrs[i], lens[i])) st = ORC_E_NONFINITE;
    }
  }
  if (status) *status = st;
  if (st != ORC_OK) return nullptr;
  orc_t *o = new orc_t;
  o->cfg = *cfg;
  o->w = *w;
  o->sess.resize(cfg->num_sessions);
  for (uint32_t s = 0; s < cfg->num_sessions; ++s) orc_reset_session(o, s);
  return o;
}

void orc_destroy(orc_t *o) { delete o; }

// Utterance start: history 0 = zero state, context [<s>]; caches
// empty; counters zero (reading 9).
int orc_reset_session(orc_t *o, uint32_t s) {
  if (!o || s >= o->cfg.num_sessions) return ORC_E_INVALID_ARG;
  Session fresh;
  Record root;
  root.slot = 0;
  if (o->cfg.N > 1) root.ctx.push_back(0u);
  fresh.rec.push_back(root);
  fresh.state.push_back(std::vector<float>(o->cfg.H, 0.0f));
  o->sess[s] = std::move(fresh);
  return ORC_OK;
}

// One decoder frame of LM queries (all hypotheses emitted for one
// frame form one batch), processed in stream (index) order, following the
// Fig. 1 / Fig. 2 flow as SURVEY 8(c) spells it out:
//  1. validate (word < V, parent created in an earlier frame, reading 17);
//  2. LM-query cache on (parent, word): hit returns the stored (score, child);
//  3. history-vector cache on (word, compress(parent state)): hit reuses the
//     first occupant's full-precision state (reading 8); miss owes a GRU;
//  4. score from the parent state and context;
//  5. new history handle (dense, non-QHIT only, reading 20); cache insert.
// After the frame every owed GRU is evaluated (states made in a frame are only
// read in later frames).
int orc_query_frame(orc_t *o, uint32_t n, const uint32_t *session, const uint32_t *parent,
                    const uint32_t *word, float *score, uint32_t *child, uint8_t *outcome) {
  if (!o || (n && (!session || !parent || !word || !score || !child))) return ORC_E_INVALID_ARG;
  const orc_config &c = o->cfg;
  std::vector<uint32_t> limit(c.num_sessions);
  std::vector<char> dead(c.num_sessions);
  for (uint32_t s = 0; s < c.num_sessions; ++s) {
    limit[s] = (uint32_t)o->sess[s].rec.size();
    dead[s] = o->sess[s].poisoned;
  }
  std::vector<Pending> pending;
  // scores are evaluated after the sequential pass (they only read parent
  // states of earlier frames); a same-frame duplicate copies its first
  // occurrence's score afterwards
  struct PendingScore { uint32_t q, s, slot, p, w; };   // p: the parent handle
  std::vector<PendingScore> pscore;
  std::vector<std::pair<uint32_t, uint32_t>> dup_of;           // (query, earlier query of this frame)
  std::map<std::pair<uint32_t, std::pair<uint32_t, uint32_t>>, uint32_t> first_q;   // (s, (p, w)) -> q
  const uint32_t cb = orc_code_bytes(c.key_mode, c.round_digits, c.H);
  std::string code(cb, '\0');
  int first_err = ORC_OK;
  for (uint32_t q = 0; q < n; ++q) {
    const uint32_t s = session[q], w = word[q], p = parent[q];
    int err = ORC_OK;
    if (s >= c.num_sessions) err = ORC_E_INVALID_ARG;
    else if (w >= c.V) err = ORC_E_VOCAB;
    else if (dead[s]) err = ORC_E_CAPACITY;                    // reading 9: reset required
    else if (p >= limit[s]) err = ORC_E_HISTORY;               // S:272, reading 17
    else if (!(c.cache_enabled && o->sess[s].qcache.count({p, w})) &&
             o->sess[s].rec.size() >= c.max_histories)
      err = ORC_E_CAPACITY;                                     // no room for a new history
    if (err != ORC_OK) {
      score[q] = NAN;
      child[q] = 0xFFFFFFFFu;
      if (outcome) outcome[q] = ORC_INVALID;
      if (s < c.num_sessions && o->sess[s].sticky == ORC_OK) o->sess[s].sticky = err;
      if (err == ORC_E_CAPACITY) o->sess[s].poisoned = true;
      if (first_err == ORC_OK) first_err = err;
      continue;
    }
    Session &S = o->sess[s];
    S.total++;
    const Record &pr = S.rec[p];
    uint32_t slot;
    uint8_t oc;
    if (c.cache_enabled) {
      auto qit = S.qcache.find({p, w});
      if (qit != S.qcache.end()) {                              // QHIT
        S.query_hits++;
        auto fq = first_q.find({s, {p, w}});
        if (fq != first_q.end()) dup_of.push_back({q, fq->second});   // score known after the pass
        else score[q] = qit->second.first;
        child[q] = qit->second.second;
        if (outcome) outcome[q] = ORC_QHIT;
        continue;
      }
      S.hidden_lookups++;
      orc_compress(c.key_mode, c.round_digits, c.H, S.state[pr.slot].data(),
                   reinterpret_cast<uint8_t *>(&code[0]));
      auto key = std::make_pair(w, code);
      auto hit = S.hcache.find(key);
      if (hit != S.hcache.end()) {                              // SHIT
        S.hidden_hits++;
        slot = hit->second;
        oc = ORC_SHIT;
      } else {                                                  // MISS
        slot = (uint32_t)S.state.size();
        S.state.emplace_back(c.H, 0.0f);
        S.hcache.emplace(key, slot);
        pending.push_back({s, slot, w, pr.slot});
        S.gru++;
        oc = ORC_MISS;
      }
    } else {                                                    // cache off: plain definition
      slot = (uint32_t)S.state.size();
      S.state.emplace_back(c.H, 0.0f);
      pending.push_back({s, slot, w, pr.slot});
      S.gru++;
      oc = ORC_MISS;
    }
    pscore.push_back({q, s, pr.slot, p, w});
    Record nr;
    nr.slot = slot;
    nr.ctx = pr.ctx;
    nr.ctx.push_back(w);
    while (nr.ctx.size() > c.N - 1) nr.ctx.erase(nr.ctx.begin());   // last N-1 words
    const uint32_t h = (uint32_t)S.rec.size();
    S.rec.push_back(nr);
    if (c.cache_enabled) {
      S.qcache[{p, w}] = {NAN, h};                              // score filled after the pass
      first_q[{s, {p, w}}] = q;
    }
    child[q] = h;
    if (outcome) outcome[q] = oc;
  }
  // The frame's scores and owed GRU evaluations are independent of each other
  // (they read only states of earlier frames and write distinct outputs), so
  // they may run on several host threads (bench.py's cpu_baseline: all
  // cores); each is the same sequential function call, so the results do not
  // depend on the thread count.
  const long ns = (long)pscore.size(), ng = (long)pending.size();
#pragma omp parallel for schedule(dynamic, 4)
  for (long i = 0; i < ns; ++i) {
    const PendingScore &ps = pscore[i];
    const Session &S = o->sess[ps.s];
    const Record &pr = S.rec[ps.p];
    score[ps.q] = orc_score(&c, &o->w, S.state[ps.slot].data(), pr.ctx.data(), (uint32_t)pr.ctx.size(), ps.w);
  }
  for (const PendingScore &ps : pscore) {
    if (!c.cache_enabled) continue;
    Session &S = o->sess[ps.s];
    S.qcache[{ps.p, ps.w}].first = score[ps.q];
  }
  for (const auto &d : dup_of) score[d.first] = score[d.second];
#pragma omp parallel for schedule(dynamic, 1)
  for (long i = 0; i < ng; ++i) {
    const Pending &pd = pending[i];
    Session &S = o->sess[pd.session];
    orc_gru(&c, &o->w, o->w.emb + (size_t)pd.word * c.E, S.state[pd.parent_slot].data(),
            nullptr, S.state[pd.slot].data());
  }
  return first_err;
}

int orc_stats(orc_t *o, uint32_t s, uint64_t *out) {
  if (!o || !out) return ORC_E_INVALID_ARG;
  uint64_t t[5] = {0, 0, 0, 0, 0};
  int sticky = ORC_OK;
  for (uint32_t i = 0; i < o->cfg.num_sessions; ++i) {
    if (s != 0xFFFFFFFFu && s != i) continue;
    const Session &S = o->sess[i];
    t[0] += S.total; t[1] += S.query_hits; t[2] += S.hidden_lookups;
    t[3] += S.hidden_hits; t[4] += S.gru;
    if (sticky == ORC_OK) sticky = S.sticky;
  }
  std::memcpy(out, t, sizeof t);
  return sticky;
}

int orc_num_handles(orc_t *o, uint32_t s, uint32_t *handles, uint32_t *slots) {
  if (!o || s >= o->cfg.num_sessions) return ORC_E_INVALID_ARG;
  if (handles) *handles = (uint32_t)o->sess[s].rec.size();
  if (slots) *slots = (uint32_t)o->sess[s].state.size();
  return ORC_OK;
}

int orc_read_slots(orc_t *o, uint32_t s, uint32_t n, const uint32_t *handles, uint32_t *slots) {
  if (!o || s >= o->cfg.num_sessions) return ORC_E_INVALID_ARG;
  const Session &S = o->sess[s];
  for (uint32_t i = 0; i < n; ++i)
    slots[i] = handles[i] < S.rec.size() ? S.rec[handles[i]].slot : 0xFFFFFFFFu;
  return ORC_OK;
}

int orc_read_states(orc_t *o, uint32_t s, uint32_t n, const uint32_t *handles, float *states) {
  if (!o || s >= o->cfg.num_sessions) return ORC_E_INVALID_ARG;
  const Session &S = o->sess[s];
  const uint32_t H = o->cfg.H;
  for (uint32_t i = 0; i < n; ++i) {
    if (handles[i] >= S.rec.size()) {
      for (uint32_t j = 0; j < H; ++j) states[(size_t)i * H + j] = NAN;
      continue;
    }
    const std::vector<float> &v = S.state[S.rec[handles[i]].slot];
    std::memcpy(states + (size_t)i * H, v.data(), 4 * (size_t)H);
  }
  return ORC_OK;
}

int orc_read_ctx(orc_t *o, uint32_t s, uint32_t n, const uint32_t *handles, uint32_t *ctx7,
                 uint32_t *ctx_len) {
  if (!o || s >= o->cfg.num_sessions) return ORC_E_INVALID_ARG;
  const Session &S = o->sess[s];
  for (uint32_t i = 0; i < n; ++i) {
    for (int j = 0; j < 7; ++j) ctx7[7 * i + j] = 0xFFFFFFFFu;
    ctx_len[i] = 0;
    if (handles[i] >= S.rec.size()) continue;
    const Record &r = S.rec[handles[i]];
    ctx_len[i] = (uint32_t)r.ctx.size();
    for (size_t j = 0; j < r.ctx.size(); ++j) ctx7[7 * i + j] = r.ctx[j];
  }
  return ORC_OK;
}

// log Z of each history handle of session s (its stored state and context);
// NaN for a handle that does not exist.
int orc_log_normalizer_handles(orc_t *o, uint32_t s, uint32_t n, const uint32_t *handles, double *out) {
  if (!o || s >= o->cfg.num_sessions) return ORC_E_INVALID_ARG;
  const Session &S = o->sess[s];
  for (uint32_t i = 0; i < n; ++i) {
    if (handles[i] >= S.rec.size()) {
      out[i] = NAN;
      continue;
    }
    const Record &r = S.rec[handles[i]];
    out[i] = orc_log_normalizer(&o->cfg, &o->w, S.state[r.slot].data(), r.ctx.data(),
                                (uint32_t)r.ctx.size());
  }
  return ORC_OK;
}

int orc_overwrite_state(orc_t *o, uint32_t s, uint32_t handle, const float *h) {
  if (!o || s >= o->cfg.num_sessions) return ORC_E_INVALID_ARG;
  Session &S = o->sess[s];
  if (handle >= S.rec.size()) return ORC_E_HISTORY;
  std::memcpy(S.state[S.rec[handle].slot].data(), h, 4 * (size_t)o->cfg.H);
  return ORC_OK;
}

}  // extern "C"

// Host threads the frame's independent scores / GRU evaluations use
// (OpenMP; 1 without it).  n > 0 sets the count, n == 0 only queries it.
int orc_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}
