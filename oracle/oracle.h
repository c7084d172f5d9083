/* oracle.h -- CPU oracle of the frame-batched GRU-RNNLM query step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * path under paper_1801_09866_b200/ (see DESIGN.md "Oracle").
 *
 * Plain, slow, obviously correct: fp64 accumulation in ascending index order,
 * one rounding to fp32 at the end; std::map caches; one query at a time in
 * stream order.  Every function cites the passage of the paper (P:n =
 * /root/reference/PAPER.md line n) or the SURVEY 8(c) reading it follows.
 */
#ifndef RNNLM_ORACLE_H
#define RNNLM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_KEY_OFF = 0, ORC_KEY_ROUND = 1, ORC_KEY_SIGN = 2 };
enum { ORC_CELL_GRU = 0, ORC_CELL_GRU_LBR = 1, ORC_CELL_RNN = 2 };   /* Chung GRU / linear-before-reset / Elman */
enum { ORC_QHIT = 0, ORC_SHIT = 1, ORC_MISS = 2, ORC_INVALID = 255 };
enum { ORC_OK = 0, ORC_E_INVALID_ARG = 1, ORC_E_DIMENSION = 2, ORC_E_NONFINITE = 3,
       ORC_E_VOCAB = 4, ORC_E_HISTORY = 5, ORC_E_CAPACITY = 6 };

typedef struct {
  uint32_t V, E, H;
  uint32_t maxent_log2, N;
  uint32_t key_mode, round_digits;
  uint32_t cache_enabled;
  uint32_t num_sessions;
  uint32_t max_histories;
  uint32_t cell;                /* ORC_CELL_* */
} orc_config;

/* Row-major fp32 arrays; the oracle keeps the POINTERS (no copy): the caller
 * keeps them alive for the oracle's lifetime. */
typedef struct {
  const float *emb;                                   /* V x E */
  const float *Wz, *Uz, *bz, *Wr, *Ur, *br, *Wh, *Uh, *bh;   /* H x E, H x H, H */
  const float *nce_w, *nce_b;                         /* V x H, V */
  const float *maxent;                                /* 2^maxent_log2 */
} orc_weights;

typedef struct orc orc_t;

/* Number of code bytes for (mode, k, H): sign ceil(H/8); round k<=2 H; k=3,4 2H; off 4H. */
uint32_t orc_code_bytes(uint32_t mode, uint32_t k, uint32_t H);
/* compress(h, mode) -- P:119-120, SURVEY 8(c) readings 3-6. Returns 0, or
 * ORC_E_NONFINITE / ORC_E_INVALID_ARG. */
int orc_compress(uint32_t mode, uint32_t k, uint32_t H, const float *h, uint8_t *code);
/* MaxEnt feature indices (SPEC S:177 recurrence). ctx is MOST RECENT LAST.
 * Writes min(N, ctx_len+1) indices; returns that count. */
uint32_t orc_maxent_indices(const uint32_t *ctx, uint32_t ctx_len, uint32_t w, uint32_t N,
                            uint64_t M, uint64_t *idx);
/* h' = GRU(x, h), Chung form (SURVEY 8(c) reading 1); fp64 throughout.
 * out64 and/or out32 may be NULL. */
void orc_gru(const orc_config *cfg, const orc_weights *w, const float *x, const float *h,
             double *out64, float *out32);
/* score = Theta[w].h + b[w] + sum_k T[idx_k] (readings 2, 12, 13). */
float orc_score(const orc_config *cfg, const orc_weights *wt, const float *h,
                const uint32_t *ctx, uint32_t ctx_len, uint32_t w);

orc_t *orc_create(const orc_config *cfg, const orc_weights *w, int *status);
void orc_destroy(orc_t *o);
int orc_reset_session(orc_t *o, uint32_t s);
/* One frame (one query_batch call): queries in index order. */
int orc_query_frame(orc_t *o, uint32_t n, const uint32_t *session, const uint32_t *parent,
                    const uint32_t *word, float *score, uint32_t *child, uint8_t *outcome);
/* out[0..4] = total, query_hits, hidden_lookups, hidden_hits, gru; returns sticky error. */
int orc_stats(orc_t *o, uint32_t s, uint64_t *out);
int orc_num_handles(orc_t *o, uint32_t s, uint32_t *handles, uint32_t *slots);
/* Per handle: slot, context (most recent LAST, padded with 0xFFFFFFFF to 7), state. */
int orc_read_slots(orc_t *o, uint32_t s, uint32_t n, const uint32_t *handles, uint32_t *slots);
int orc_read_states(orc_t *o, uint32_t s, uint32_t n, const uint32_t *handles, float *states);
int orc_read_ctx(orc_t *o, uint32_t s, uint32_t n, const uint32_t *handles, uint32_t *ctx7,
                 uint32_t *ctx_len);
/* Replay protocol: overwrite the state owned by handle's slot. */
int orc_overwrite_state(orc_t *o, uint32_t s, uint32_t handle, const float *h);
/* Exact log-normaliser log sum_v exp(score_v) over the vocabulary, fp64
 * (S:201-209), of a state + context, or of stored handles. */
double orc_log_normalizer(const orc_config *cfg, const orc_weights *wt, const float *h,
                          const uint32_t *ctx, uint32_t ctx_len);
int orc_log_normalizer_handles(orc_t *o, uint32_t s, uint32_t n, const uint32_t *handles, double *out);

/* Host threads for the frame's independent score / GRU evaluations (n > 0
 * sets, 0 queries); results do not depend on it. */
int orc_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
