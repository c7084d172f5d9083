// rnnlm_impl.cuh -- internal data layout shared by the engine's kernels.
//
// Layout in HBM: all pools are allocated once at
// rnnlm_create with fixed capacity, indexed [session * cap + local].
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rnnlm.h"

namespace rnnlm_dev {

constexpr unsigned long long TAG_EMPTY = ~0ull;
constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr int MAX_CTX = 7;            // maxent_order <= 8

// LM-query cache entry (a2): key (parent handle << 32 | word), value (score, child).
// Bit 31 of the word field marks an entry inserted by the running call (so V < 2^31).
struct __align__(16) QEntry {
  unsigned long long tag;
  float score;
  uint32_t child;
};
// Hidden-state cache entry (a3): key reference (ref_slot << 32 | word) -- the
// key is (word, code(state[ref_slot])) -- and the value: the child state slot.
struct __align__(16) HEntry {
  unsigned long long tag;
  uint32_t slot;
  uint32_t pad;
};
// History record: state slot + word context, MOST RECENT FIRST, NONE = absent.
struct __align__(32) Rec {
  uint32_t slot;
  uint32_t ctx[MAX_CTX];
};
// Scoring work item of a non-QHIT query, written by k_commit: the parent's
// record (state slot + word context) and the query's session / word, so the
// scorer needs no further lookups before its row loads.  pr.slot == NONE: the
// query failed in k_commit (out of handles) and is not scored.
struct __align__(32) ScoreItem {
  Rec pr;
  uint32_t q, s, w, pad;
};
// Per-session counters and allocation cursors.
struct __align__(64) SessCtr {
  uint32_t next_handle, next_slot;
  uint32_t poisoned;                // a capacity failure happened: every later query is INVALID
  uint32_t pad1;
  unsigned long long total, qhits, hlookups, hhits, gru;
  unsigned long long pad2[1];
};

// Per-query classification carried between the kernels of one call.
enum : uint32_t {
  ST_INVALID = 0,
  ST_QHIT_OLD = 1,   // (parent, word) cached by an earlier call
  ST_QNEED = 2,      // not cached before this call: claims a query-cache entry
  ST_QHIT_NEW = 3,   // duplicate of a lower-index query of this call
  ST_SHIT_OLD = 4,   // hidden key cached by an earlier call
  ST_HNEED = 5,      // hidden key not cached before this call: claims an entry
  ST_SHIT_NEW = 6,   // hidden key first claimed by a lower-index query of this call
  ST_MISS = 7,       // owes a GRU evaluation
  ST_MISS_NC = 8,    // cache disabled: every valid query owes a GRU evaluation
};

// Everything a kernel needs, passed by value.
struct Params {
  uint32_t V, E, H, N, S, cap;
  uint32_t qmask, hmask;          // table capacity - 1 (power of two)
  uint32_t key_mode, round_digits, cache, math;
  uint32_t cell;                  // rnnlm_cell
  unsigned long long M_mask;
  uint32_t cstride;               // bytes per stored code row (multiple of 16)
  uint32_t code_bytes, code_words;
  uint32_t Hp;                    // H rounded up to 64 (SIMT weight layouts)
  float round_scale;              // 10^round_digits in fp32
  // weights (device, kernel layouts)
  const float *emb;               // V x E fp32
  const __nv_bfloat16 *emb16;     // V x E bf16 (MATH_BF16)
  const float *nce_w;             // V x H fp32 (or NULL when nce_w16 is used)
  const __nv_bfloat16 *nce_w16;   // V x H bf16 (only when every entry is bf16-exact)
  const float *nce_b;             // V
  const float *maxent;            // M
  const float *w1x;               // SIMT phase 1, x part: [E][Hp/64][3][64] (z, r, h gates)
  const float *w1h;               // SIMT phase 1, h part: [H][Hp/64][2][64] (z, r gates)
  const float *b1;                // [Hp/64][3][64] (bz, br, bh)
  const float *w2;                // SIMT phase 2: Uh^T [H][Hp]
  // pools
  Rec *rec;                       // S*cap
  float *state;                   // S*cap x H fp32
  uint8_t *codes;                 // S*cap x cstride (key modes sign/round)
  unsigned long long *codehash;   // S*cap
  QEntry *qtab;                   // S*(qmask+1)
  uint32_t *qowner;
  HEntry *htab;                   // S*(hmask+1)
  uint32_t *howner;
  SessCtr *ctr;                   // S
  int *sticky;
  // per-call scratch (B_max)
  uint32_t *st, *qent, *aux, *hent, *pslot, *cslot, *excl_nonq, *excl_miss;
  unsigned long long *phash;      // code hash of the parent's state (cache on; k_qcache -> k_hcache)
  ScoreItem *score_items;         // [non-QHIT index] (k_commit -> k_score)
  uint32_t *dup_list;             // QHIT_NEW queries of this call (count in counts[3])
  uint8_t *claimed;               // bit 0: claimed a query-cache entry, bit 1: a hidden-cache entry
  uint32_t *row_src, *row_dst, *row_word;   // GRU rows: global state rows + word
  uint32_t *seg_excl_nonq, *seg_excl_miss, *seg_cnt_nonq, *seg_cnt_miss;  // per session
  unsigned long long *tile_status;
  uint32_t *tile_ticket;
  uint32_t *counts;               // [0] non-QHIT total, [1] GRU rows, [2] bad-batch flag (cleared by the call's last kernel), [3] duplicates
  // GRU intermediates (rows x H)
  float *g_z, *g_rh, *g_wxb;
  __nv_bfloat16 *g_rh16;
};

struct CallArgs {
  uint32_t n;                     // queries of the call (the grids' size); with d_n: the maximum
  const uint32_t *d_n;            // nullable: the call's query count, read on the device (graph replay, <= n)
  const uint32_t *session, *parent, *word;
  float *score;
  uint32_t *child;
  uint8_t *outcome;
};

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

__device__ __forceinline__ void latch(int *sticky, int err) { atomicCAS(sticky, 0, err); }

// The call's query count: host-given, or read from device memory (a replayed
// CUDA graph sized for A.n queries serves any count up to A.n).
__device__ __forceinline__ uint32_t call_n(const CallArgs &A) {
  if (!A.d_n) return A.n;
  const uint32_t n = *A.d_n;
  return n < A.n ? n : A.n;
}

// Programmatic dependent launch (PDL): every kernel of the step is launched
// with programmatic stream serialisation, so its launch and CTA rasterisation
// overlap the tail of the previous kernel; griddepcontrol.wait then blocks
// until the previous grid has completed and its memory is visible.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace rnnlm_dev

// ---- host launchers (one per kernel family) --------------------------------
namespace rnnlm_host {
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                      cudaStream_t s, unsigned cluster_x, Args... args) {
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = cluster_x;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
using rnnlm_dev::CallArgs;
using rnnlm_dev::Params;
#ifndef RNNLM_SCAN_ITEMS
#define RNNLM_SCAN_ITEMS 2
#endif
constexpr int SCAN_TILE = 256 * RNNLM_SCAN_ITEMS;    // queries per look-back tile (256 threads)
int launch_cache_front(const Params &P, const CallArgs &A, cudaStream_t s);   // returns #launches
int launch_commit(const Params &P, const CallArgs &A, cudaStream_t s);
int launch_score(const Params &P, const CallArgs &A, int num_sms, cudaStream_t s);
int launch_final(const Params &P, const CallArgs &A, cudaStream_t s);
int launch_dup_scores(const Params &P, const CallArgs &A, int num_sms, cudaStream_t s);
int launch_gru_simt(const Params &P, uint32_t max_rows, int num_sms, cudaStream_t s);
int launch_encode_rows(const Params &P, uint32_t max_rows, int num_sms, cudaStream_t s);
int launch_reset_root(const Params &P, uint32_t s_lo, uint32_t s_hi, cudaStream_t s);
int launch_read_states(const Params &P, uint32_t sess, uint32_t n, const uint32_t *h, float *out,
                       cudaStream_t s);
int launch_read_slots(const Params &P, uint32_t sess, uint32_t n, const uint32_t *h, uint32_t *out,
                      cudaStream_t s);
int launch_read_codes(const Params &P, uint32_t sess, uint32_t n, const uint32_t *h, uint8_t *out,
                      cudaStream_t s);
int launch_encode_states(const Params &P, uint32_t n, const float *states, uint8_t *out,
                         cudaStream_t s);
int launch_maxent_indices(const Params &P, uint32_t n, const uint32_t *sess, const uint32_t *par,
                          const uint32_t *word, unsigned long long *out, cudaStream_t s);
int launch_resolve_parents(uint32_t n, const int64_t *ref, const uint32_t *log, uint32_t *out,
                           cudaStream_t s);
}  // namespace rnnlm_host
