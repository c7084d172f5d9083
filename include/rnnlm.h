/* rnnlm.h -- C ABI of the B200-native frame-batched GRU-RNNLM query step.
 *
 * The operation (PAPER.md, arXiv 1801.09866; P:n = line n of PAPER.md):
 *   An online ASR decoder emits, at every 10 ms frame, LM queries
 *   (history, next word) for the hypotheses that reached a word boundary
 *   (P:45-47).  Each query is answered with an unnormalised log-score
 *   (NCE inner product of the history's GRU output with the word's output row
 *   plus bias, plus the hashed n-gram MaxEnt bypass) and a
 *   handle for the extended history, whose state is the GRU update
 *   h' = GRU(x_word, h).  Redundant work is removed by an exact
 *   LM-query cache on (history, word) (Fig. 1) and by a cache of GRU
 *   outputs keyed on (word, lossily compressed history vector), where the
 *   compression rounds each element to k decimals or keeps only its sign
 *   (Table 1).  All queries of one decoder frame are one batch
 *   (frame-wise batching).
 *
 *   On B200 the whole step stays resident in HBM: one rnnlm_query_batch call
 *   = one frame for any number of sessions, executed as a short sequence of
 *   sm_100a kernels on the caller's stream.  Semantics
 *   are those of SURVEY.md 8(c) / DESIGN.md "Readings", which the CPU oracle
 *   (oracle/, test infrastructure) implements one query at a time.
 *
 * Conventions
 *   - One rnnlm_t per CUDA device; one host thread per handle at a time.
 *   - Every call that takes a cudaStream_t is stream-ordered and asynchronous
 *     and allocates nothing (so a caller may capture it in a CUDA graph).
 *     rnnlm_query_batch forks part of its work onto an internal stream and
 *     joins it back into the caller's stream before returning.
 *     rnnlm_cache_stats, rnnlm_get_timing and rnnlm_create/destroy synchronise.
 *   - Pointers named d_* are DEVICE pointers owned by the caller; they must
 *     stay valid until the work on the given stream completes.  Pointers
 *     without the prefix are host pointers, read/written before return.
 *   - History handles are dense u32 per session.  Handle 0 is the utterance
 *     root: zero state, word context [0] (<s>).  A query's parent must be a
 *     handle created by an EARLIER rnnlm_query_batch call of that session
 *     (reading 17).  New handles are numbered densely, in stream
 *     (index) order, over the non-QHIT queries of the session; state slots
 *     densely over the MISS queries (reading 20).
 *   - Errors: argument errors are returned synchronously.  Per-query errors
 *     (session >= num_sessions, word >= V, unknown/unborn parent, batch not
 *     sorted by session, capacity exhausted) are detected on the device: the
 *     query gets score = NaN, child = 0xFFFFFFFF, outcome = RNNLM_INVALID, the
 *     rest of the batch proceeds, and the first such error is latched into a
 *     sticky word returned by rnnlm_cache_stats.  After RNNLM_E_CAPACITY the
 *     affected session must be reset.
 */
#ifndef RNNLM_H
#define RNNLM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RNNLM_ABI_VERSION 3

typedef struct rnnlm rnnlm_t;          /* opaque; one per CUDA device */
typedef struct rnnlm_graph rnnlm_graph_t;   /* opaque; a captured rnnlm_query_batch (rnnlm_graph_create) */
typedef struct CUstream_st *rnnlm_stream_t;   /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  RNNLM_OK = 0,
  RNNLM_E_INVALID_ARG = 1,  /* null pointer, bad enum, n > max_queries_per_call, unsorted batch */
  RNNLM_E_DIMENSION = 2,    /* V < 2, E/H not multiples of 8, N outside 1..8, ... */
  RNNLM_E_NONFINITE = 3,    /* a weight is NaN or Inf */
  RNNLM_E_VOCAB = 4,        /* query word >= V (per query, sticky) */
  RNNLM_E_HISTORY = 5,      /* parent handle not created in an earlier call (per query, sticky) */
  RNNLM_E_CAPACITY = 6,     /* session ran out of history handles (per query, sticky) */
  RNNLM_E_CUDA = 7,         /* a CUDA runtime call failed */
  RNNLM_E_OOM = 8           /* device allocation failed at create */
} rnnlm_status;

/* History-vector compression used as the hidden-state cache key. */
typedef enum {
  RNNLM_KEY_OFF = 0,        /* exact fp32 bit pattern */
  RNNLM_KEY_ROUND = 1,      /* q_i = roundf(h_i * 10^k) (fp32 product, half away from zero), k = round_digits */
  RNNLM_KEY_SIGN = 2        /* bit_i = (h_i >= 0.0f) */
} rnnlm_key_mode;

/* Arithmetic of the GRU gate contraction (a5).  States are always fp32. */
typedef enum {
  RNNLM_MATH_FP32 = 0,      /* FP32 FFMA (SIMT) */
  RNNLM_MATH_TF32 = 1,      /* fp32 operands read as TF32, fp32 accumulation on tcgen05 tensor cores */
  RNNLM_MATH_BF16 = 2,      /* bf16 operands, fp32 accumulation on tcgen05 tensor cores */
  RNNLM_MATH_TF32X3 = 3,    /* fp32-accurate on tcgen05: a = a_hi + a_lo, w = w_hi + w_lo (TF32 parts),
                             * a.w ~ a_hi.w_hi + a_hi.w_lo + a_lo.w_hi (three TF32 products, fp32
                             * accumulation; the 1e-5 path of the FP32 mode at tensor-core rate).
                             * Products that are identically zero are not computed: a_hi.w_lo when
                             * every gate weight is TF32-exact (w_lo == 0), a_lo.w_hi over the
                             * embedding part of K when every embedding entry is (x_lo == 0);
                             * rnnlm_tf32x3_products reports what remains. */
  RNNLM_MATH_BF16X3 = 4     /* fp32-accurate on tcgen05 bf16 tensor cores: every fp32 operand is split
                             * into three bf16 parts v = hi + mid + lo (|v - hi - mid - lo| <= 2^-27 |v|;
                             * each part times a bf16 weight part is exact in fp32), and the
                             * contraction sums a_i.w_j over i + j <= 2 (six bf16 products, fp32
                             * accumulation), held to the FP32 mode's 1e-5 like TF32X3.  Identically
                             * zero products are skipped: with bf16-exact gate weights only
                             * a_hi.w + a_mid.w + a_lo.w remain, and over the embedding part of K
                             * only x_hi.w when every embedding entry is bf16-exact (2 bf16 products
                             * per useful multiply-add at E = H; rnnlm_tf32x3_products reports it).
                             * Scores use the fp32 output weights (like TF32 / TF32X3). */
  /* The tensor-core modes need E % 64 == 0 and H % 128 == 0 (else
   * rnnlm_create returns RNNLM_E_DIMENSION).  BF16 stores bf16 copies of E
   * and the gate weights (and of nce_w when every entry is bf16-exact); TF32
   * keeps every parameter fp32. */
} rnnlm_math;

typedef enum { RNNLM_QHIT = 0, RNNLM_SHIT = 1, RNNLM_MISS = 2, RNNLM_INVALID = 255 } rnnlm_outcome;

/* Recurrent cell of step (a5).  GRU: the cited GRU (Chung
 * 2014, reading 1), c = tanh(Wh x + Uh (r . h) + bh).
 * GRU_LBR: "linear before reset", c = tanh(Wh x + bh + r . (Uh h)) (the
 * torch.nn.GRUCell form with no inner bias); z, r, the update
 * h' = (1 - z) h + z c and everything else are identical.
 * RNN: the paper's comparison "vanilla-RNNLM" as an Elman layer with
 * the logistic activation of the RNNLM it cites, h' = sigma(Wh x + Uh h + bh)
 * (Wz, Uz, bz, Wr, Ur, br are not used). */
typedef enum { RNNLM_CELL_GRU = 0, RNNLM_CELL_GRU_LBR = 1, RNNLM_CELL_RNN = 2 } rnnlm_cell;

/* Kernels of step (a5) per call (north_star "a vectorised
 * memory-bound GEMV path where [the batch] does not [fill tiles]").
 * TILES: the gather + tile kernels (tcgen05 for BF16 / TF32 / 3xTF32, FFMA
 * tiles for FP32).  GEMV: two small-frame kernels that cut the work by output
 * units across all SMs (same operand rounding as the engine's math mode;
 * FP32 and 3xTF32 engines use plain fp32 FFMA).  AUTO: GEMV for calls of at
 * most RNNLM_GEMV_AUTO_MAX_QUERIES queries, tiles otherwise.  Results of the
 * two kinds agree within the math mode's tolerance, not bitwise (summation
 * order).  On the AUTO path a call of at most RNNLM_GEMV_AUTO_MAX_QUERIES
 * queries runs as ONE cooperative kernel (k_small: every step of the call,
 * grid barriers instead of kernel boundaries; results bitwise those of the
 * GEMV path). */
typedef enum { RNNLM_GRU_AUTO = 0, RNNLM_GRU_TILES = 1, RNNLM_GRU_GEMV = 2 } rnnlm_gru_path;
#define RNNLM_GEMV_AUTO_MAX_QUERIES 512u

typedef struct {
  uint32_t vocab, embed, hidden;        /* 2 <= V < 2^31 (word 0 = <s>), E, H; E and H multiples of 8 */
  uint32_t maxent_log2, maxent_order;   /* MaxEnt table M = 2^maxent_log2 floats (<= 2^31); order N in 1..8 */
  uint32_t key_mode, round_digits;      /* rnnlm_key_mode; round_digits in 1..4 when ROUND */
  uint32_t math;                        /* rnnlm_math */
  uint32_t cache_enabled;               /* 0: no cache at all, every valid query is a MISS */
  uint32_t num_sessions;                /* utterance streams owned by this handle */
  uint32_t max_queries_per_call;        /* B_max: fixes scratch sizes */
  uint32_t max_histories_per_session;   /* handle/state capacity per session (>= 2); no eviction */
  int32_t device;                       /* CUDA device ordinal */
  uint32_t cell;                        /* rnnlm_cell (0 = GRU) */
  uint32_t max_queries_per_session_call;  /* most queries ONE session has in one call (0 = max_queries_per_call);
                                         * sizes each session's two hash tables at 2 x (this + max_histories)
                                         * entries (load <= 0.5).  A call exceeding it stays memory-safe but
                                         * may fail its queries with RNNLM_E_CAPACITY. */
  uint32_t gru_path;                    /* rnnlm_gru_path (0 = AUTO) */
} rnnlm_config;

/* Host fp32 row-major weights, copied at create (caller may free on return).
 * Shapes: emb V x E; Wz, Wr, Wh H x E; Uz, Ur, Uh H x H; bz, br, bh H;
 * nce_w V x H (row per word, the paper's H x V matrix transposed);
 * nce_b V; maxent 2^maxent_log2. */
typedef struct {
  const float *emb;
  const float *Wz, *Uz, *bz, *Wr, *Ur, *br, *Wh, *Uh, *bh;
  const float *nce_w, *nce_b;
  const float *maxent;
} rnnlm_weights;

typedef struct {
  uint64_t total_queries, query_hits, hidden_lookups, hidden_hits, gru_computations;
  int32_t sticky_error;                 /* rnnlm_status of the first per-query error, else 0 */
  int32_t pad_;
} rnnlm_stats;

/* Per-kernel-group device time accumulated while timing is enabled (CUDA
 * events around each group, on the stream the group runs on; scoring and the
 * result write run on an internal side stream concurrently with the GRU). */
typedef struct {
  double ms_cache;      /* key/probe/claim/scan/commit kernels (a1-a4) */
  double ms_score;      /* NCE + MaxEnt scoring (a6), side stream */
  double ms_gru;        /* gather + gate contraction + gates, both phases (a5) */
  double ms_encode;     /* code + code hash of new states (a1; FP32 SIMT path only) */
  double ms_final;      /* result write + counters (a7), side stream */
  uint64_t calls;       /* timed query_batch calls */
  uint64_t launches;    /* kernels launched by those calls */
  /* timing level 2, tensor-core paths only: split of ms_gru (gather, fused GEMM) */
  double ms_gru_gather, ms_gru_phase1, ms_gru_phase2;
  double ms_fused;      /* calls that ran the fused small-frame kernel (k_small): the whole step */
} rnnlm_timing;

/* Create an engine on cfg->device: validates dims and weights, copies the
 * weights into kernel layouts, allocates every pool once, resets all
 * sessions.  On failure *out = NULL and the status says why. */
rnnlm_status rnnlm_create(const rnnlm_config *cfg, const rnnlm_weights *w, rnnlm_t **out);
void rnnlm_destroy(rnnlm_t *h);

/* Utterance start for one session (UINT32_MAX = all): clears both caches,
 * counters, histories; handle 0 becomes the root again. */
rnnlm_status rnnlm_reset_session(rnnlm_t *h, uint32_t session, rnnlm_stream_t stream);

/* One decoder frame of n LM queries (frame-wise batching).
 *   d_session, d_parent, d_word: n u32 each.  Queries must be sorted by
 *     session (non-decreasing); within a session, index order is stream order.
 *   d_score (n f32), d_child (n u32): results; d_outcome (n u8) may be NULL.
 * Steps: (a1) key of the parent state, (a2) LM-query cache,
 * (a3) hidden-state cache, (a4) miss compaction + handle/slot allocation,
 * (a5) embedding gather + GRU for the misses, (a6) NCE + MaxEnt score of every
 * non-QHIT query, (a7) result write + cache inserts + counters. */
rnnlm_status rnnlm_query_batch(rnnlm_t *h, uint32_t n, const uint32_t *d_session,
                               const uint32_t *d_parent, const uint32_t *d_word, float *d_score,
                               uint32_t *d_child, uint8_t *d_outcome, rnnlm_stream_t stream);

/* CUDA-graph form of rnnlm_query_batch for decoder loops (SURVEY 3.2, 7 step
 * 9): captures ONE call on fixed device buffers into an instantiated graph;
 * every rnnlm_graph_launch replays it on `stream` (one graph launch instead of
 * ~10 kernel launches; no host work per frame).  The caller rewrites the
 * CONTENTS of d_session / d_parent / d_word (and *d_n) before each launch.
 *   max_n: queries the graph is sized for (<= max_queries_per_call).
 *   d_n: nullable device u32, the query count of each replay (read on the
 *     device; values above max_n are clamped); NULL = always max_n.
 * Same semantics, results and errors as rnnlm_query_batch with those inputs.
 * rnnlm_results_ready does not apply to graph launches (the stream itself
 * orders them).  The graph references the engine: destroy it first. */
rnnlm_status rnnlm_graph_create(rnnlm_t *h, uint32_t max_n, const uint32_t *d_n, const uint32_t *d_session,
                                const uint32_t *d_parent, const uint32_t *d_word, float *d_score,
                                uint32_t *d_child, uint8_t *d_outcome, rnnlm_graph_t **out);
rnnlm_status rnnlm_graph_launch(rnnlm_graph_t *g, rnnlm_stream_t stream);
void rnnlm_graph_destroy(rnnlm_graph_t *g);

/* Makes `stream` wait until the per-query results of the most recent
 * rnnlm_query_batch (d_score, d_child, d_outcome) are written.  They are final
 * before that call's GRU (a5) finishes -- the GRU only produces the new
 * states later calls read -- so a caller can copy the results out and
 * prepare the next frame while the state update still runs; the next
 * rnnlm_query_batch on the same stream is ordered after it as usual. */
rnnlm_status rnnlm_results_ready(rnnlm_t *h, rnnlm_stream_t stream);

/* Counters of one session (UINT32_MAX = sum over all).  Synchronises the
 * device.  Returns the sticky error (also stored in out->sticky_error). */
rnnlm_status rnnlm_cache_stats(rnnlm_t *h, uint32_t session, rnnlm_stats *out);

/* States (n x H fp32) of n handles of one session; unknown handles -> NaN rows. */
rnnlm_status rnnlm_read_states(rnnlm_t *h, uint32_t session, uint32_t n, const uint32_t *d_handles,
                               float *d_states, rnnlm_stream_t stream);
/* State slot of each handle (0xFFFFFFFF if unknown). */
rnnlm_status rnnlm_read_slots(rnnlm_t *h, uint32_t session, uint32_t n, const uint32_t *d_handles,
                              uint32_t *d_slots, rnnlm_stream_t stream);
/* Stored compression code of each handle's state, rnnlm_code_bytes() bytes per
 * row (sign: bit i in byte i/8 at bit i%8; round: int8 (k<=2) / LE int16;
 * off: the fp32 bit patterns).  Unknown handles -> 0xFF bytes. */
rnnlm_status rnnlm_read_codes(rnnlm_t *h, uint32_t session, uint32_t n, const uint32_t *d_handles,
                              uint8_t *d_codes, rnnlm_stream_t stream);
/* The same compression applied to n arbitrary fp32 rows d_states (n x H),
 * with the handle's key mode (inspection/testing of step a1). */
rnnlm_status rnnlm_encode_states(rnnlm_t *h, uint32_t n, const float *d_states, uint8_t *d_codes,
                                 rnnlm_stream_t stream);
/* MaxEnt feature indices of queries (session, parent, word), n x maxent_order
 * u64, unused orders = UINT64_MAX (inspection/testing of step a6). */
rnnlm_status rnnlm_maxent_indices(rnnlm_t *h, uint32_t n, const uint32_t *d_session,
                                  const uint32_t *d_parent, const uint32_t *d_word, uint64_t *d_idx,
                                  rnnlm_stream_t stream);
uint32_t rnnlm_code_bytes(const rnnlm_t *h);

/* Exact log-normaliser of n stored histories: the
 * normalisation over the vocabulary that NCE avoids ("they need to be
 * normalized ... a highly computationally intensive task considering the
 * vocabulary size"; SPEC exact_log_prob S:201-209):
 *   d_log_z[i] = log sum_{v < V} exp(s_v),  s_v = the step-(a6) score of word v
 *   for history d_history[i] of session d_session[i] (NCE + all MaxEnt orders),
 * so score - log Z is the exact log-probability.  n <= max_queries_per_call;
 * d_session, d_history: n u32 (device); d_log_z: n f32 (device), NaN for a
 * history that does not exist.  Tensor-core contraction in every math mode
 * (state split into two bf16 halves against bf16 output rows; engines whose
 * output rows are not bf16-exact use a rounded bf16 copy made at the first
 * call).  The first call allocates its scratch (synchronous).  Requires
 * hidden % 64 == 0 (else RNNLM_E_DIMENSION). */
rnnlm_status rnnlm_log_normalizer(rnnlm_t *h, uint32_t n, const uint32_t *d_session,
                                  const uint32_t *d_history, float *d_log_z, rnnlm_stream_t stream);

/* Workload plumbing (not part of the method): d_parent[i] = d_ref[i] < 0 ? 0
 * : d_log[d_ref[i]], i.e. map "child of earlier query j" references to the
 * handles the engine returned for those queries. */
rnnlm_status rnnlm_resolve_parents(uint32_t n, const int64_t *d_ref, const uint32_t *d_log,
                                   uint32_t *d_parent, rnnlm_stream_t stream);

/* level 0: off; 1: per kernel group; 2: also per GRU kernel (adds events inside
 * the GRU group, which serialise those launches). */
rnnlm_status rnnlm_set_timing(rnnlm_t *h, int level);
rnnlm_status rnnlm_get_timing(rnnlm_t *h, rnnlm_timing *out, int reset);
/* Kernels launched by this handle since create (host-side count). */
uint64_t rnnlm_launch_count(const rnnlm_t *h);
/* Split (fp32-accurate) engines: tensor-core products per useful multiply-add
 * of the gate contraction, in the mode's own MMA kind (RNNLM_MATH_TF32X3: TF32
 * products, 3 less the skipped zero products, e.g. 1.5 with TF32-exact weights
 * and embeddings at E = H; RNNLM_MATH_BF16X3: bf16 products, 6 less the skipped
 * ones, e.g. 2 with bf16-exact weights and embeddings at E = H); else 0. */
double rnnlm_tf32x3_products(const rnnlm_t *h);
const char *rnnlm_status_string(rnnlm_status s);
int rnnlm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RNNLM_H */
