// cache.cuh -- per-query device functions of steps (a2) LM-query cache,
// (a3) hidden-state cache, (a4) miss compaction + handle/slot allocation and
// (a7) result write + counters.  The multi-kernel path (k_cache.cu: one
// kernel per step, kernel boundaries between claim and owner read) and the
// fused small-frame kernel (k_small.cu: grid barriers instead) both run
// these, so the two paths share every decision rule.  See k_cache.cu for the
// semantics (first occupant = lowest query index).
#pragma once

#include "rnnlm_impl.cuh"

namespace rnnlm_dev {

__device__ __forceinline__ unsigned long long vload64(const unsigned long long *p) {
  return *reinterpret_cast<const volatile unsigned long long *>(p);
}

__device__ __forceinline__ uint32_t hhome(unsigned long long codehash, uint32_t w, uint32_t mask) {
  return (uint32_t)(mix64(codehash ^ ((unsigned long long)w * 0x9E3779B97F4A7C15ull)) & mask);
}

// Full code equality of the states in global rows a and b (never a hash).
// Loads are issued four 16-byte words at a time before any compare, so a
// 128-byte sign code costs two dependent round trips instead of eight.
static __device__ bool code_equal(const Params &P, size_t a, size_t b) {
  if (a == b) return true;
  const uint4 *pa, *pb;
  uint32_t n16;
  if (P.key_mode == RNNLM_KEY_OFF) {
    pa = reinterpret_cast<const uint4 *>(P.state + a * P.H);
    pb = reinterpret_cast<const uint4 *>(P.state + b * P.H);
    n16 = P.H / 4;
  } else {
    pa = reinterpret_cast<const uint4 *>(P.codes + a * P.cstride);
    pb = reinterpret_cast<const uint4 *>(P.codes + b * P.cstride);
    n16 = P.cstride / 16;
  }
  for (uint32_t i = 0; i < n16; i += 4) {
    uint4 x[4], y[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x[j] = y[j] = make_uint4(0u, 0u, 0u, 0u);
      if (i + j < n16) { x[j] = pa[i + j]; y[j] = pb[i + j]; }
    }
    uint32_t d = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) d |= (x[j].x ^ y[j].x) | (x[j].y ^ y[j].y) | (x[j].z ^ y[j].z) | (x[j].w ^ y[j].w);
    if (d) return false;
  }
  return true;
}

// Hidden-cache key match: same word and equal code of the reference state
// (an entry whose reference IS the probing row matches without reading it).
__device__ __forceinline__ bool hkey_match(const Params &P, unsigned long long tag, uint32_t s,
                                           uint32_t w, uint32_t ps, unsigned long long hh) {
  if ((uint32_t)tag != w) return false;
  const uint32_t ref = (uint32_t)(tag >> 32);
  if (ref == ps) return true;
  const size_t base = (size_t)s * P.cap;
  if (P.codehash[base + ref] != hh) return false;
  return code_equal(P, base + ref, base + ps);
}

// Entries inserted during the current call carry NEW_BIT in their word field;
// entries of earlier calls never do (k_commit clears the bit).  A probe that
// meets its key without the bit is a hit on an earlier call; with the bit, a
// key claimed concurrently in this call.  Chains are never shortened, so an
// earlier-call entry of a key always precedes every slot filled in this call.
constexpr unsigned long long NEW_BIT = 1ull << 31;

// ---- (a2) LM-query cache: probe + claim ---------------------------------------
// The loads of the session counters, the parent's record, the first probe and
// the parent's code hash are issued before the validation that decides whether
// they are needed (indices clamped in bounds), so the chain is inputs ->
// {counters, record, probe} -> {code hash, CAS}.  The parent's state slot and
// code hash are handed to k_hcache (pslot, phash).
__device__ __forceinline__ void qcache_query(const Params &P, const CallArgs &A, uint32_t q) {
  const uint32_t s = A.session[q], w = A.word[q], p = A.parent[q];
  const uint32_t sprev = q > 0 ? A.session[q - 1] : 0u;
  const uint32_t sc = s < P.S ? s : 0u, pc = p < P.cap ? p : 0u;
  const size_t cb = (size_t)sc * P.cap;
  const uint32_t poisoned = P.ctr[sc].poisoned, nh = P.ctr[sc].next_handle;
  const uint32_t ps = P.rec[cb + pc].slot;
  const unsigned long long key = ((unsigned long long)p << 32) | w, nkey = key | NEW_BIT;
  const size_t base = (size_t)sc * (P.qmask + 1);
  uint32_t idx = (uint32_t)(mix64(key) & P.qmask);
  unsigned long long t = P.cache ? vload64(&P.qtab[base + idx].tag) : 0ull;
  P.claimed[q] = 0;
  int err = 0;
  if (s >= P.S) err = RNNLM_E_INVALID_ARG;
  else if (q > 0 && sprev > s) err = RNNLM_E_INVALID_ARG;
  else if (w >= P.V) err = RNNLM_E_VOCAB;
  else if (poisoned) err = RNNLM_E_CAPACITY;
  else if (p >= nh) err = RNNLM_E_HISTORY;
  if (q > 0 && sprev > s) P.counts[2] = 1u;            // batch not sorted by session
  if (err) {
    P.st[q] = ST_INVALID;
    latch(P.sticky, err);
    return;
  }
  P.pslot[q] = ps;
  if (!P.cache) {
    P.st[q] = ST_MISS_NC;
    return;
  }
  const unsigned long long hh = P.codehash[cb + (ps < P.cap ? ps : 0u)];
  for (uint32_t probes = 0; probes <= P.qmask; ++probes) {
    if (probes) t = vload64(&P.qtab[base + idx].tag);
    if (t == key) { P.st[q] = ST_QHIT_OLD; P.qent[q] = idx; return; }
    if (t == TAG_EMPTY) t = atomicCAS(&P.qtab[base + idx].tag, TAG_EMPTY, nkey);
    if (t == TAG_EMPTY || t == nkey) {                  // claimed (or joined) in this call
      atomicMin(&P.qowner[base + idx], q);
      P.st[q] = ST_QNEED;
      P.qent[q] = idx;
      P.phash[q] = hh;
      P.claimed[q] = 1;
      return;
    }
    idx = (idx + 1) & P.qmask;
  }
  // table full: tables hold >= cap + B_max keys, so this needs exhausted handles
  P.st[q] = ST_INVALID;
  latch(P.sticky, RNNLM_E_CAPACITY);
}

// ---- (a3) hidden-state cache: owner resolution + probe + claim -----------------
// Chain: per-query scratch -> {query-cache owner, first probe} -> CAS.
__device__ __forceinline__ void hcache_query(const Params &P, const CallArgs &A, uint32_t q) {
  const uint32_t st = P.st[q];
  const bool bad = P.counts[2] != 0u;
  const uint32_t s = A.session[q], w = A.word[q], qe = P.qent[q], ps = P.pslot[q];
  const unsigned long long hh = P.phash[q];
  if (st != ST_QNEED || bad) return;
  const uint32_t o = P.qowner[(size_t)s * (P.qmask + 1) + qe];
  const size_t base = (size_t)s * (P.hmask + 1);
  uint32_t idx = hhome(hh, w, P.hmask);
  unsigned long long t = vload64(&P.htab[base + idx].tag);
  if (o != q) { P.st[q] = ST_QHIT_NEW; P.aux[q] = o; return; }
  const unsigned long long mine = (((unsigned long long)ps << 32) | w) | NEW_BIT;
  for (uint32_t probes = 0; probes <= P.hmask; ++probes) {
    if (probes) t = vload64(&P.htab[base + idx].tag);
    if (t == TAG_EMPTY) {
      t = atomicCAS(&P.htab[base + idx].tag, TAG_EMPTY, mine);
      if (t == TAG_EMPTY) t = mine;                     // inserted: falls into the claim below
    }
    if (hkey_match(P, t & ~NEW_BIT, s, w, ps, hh)) {
      if (!(t & NEW_BIT)) {                             // cached by an earlier call
        P.st[q] = ST_SHIT_OLD;
        P.hent[q] = idx;
        P.cslot[q] = P.htab[base + idx].slot;
        return;
      }
      atomicMin(&P.howner[base + idx], q);
      P.st[q] = ST_HNEED;
      P.hent[q] = idx;
      P.claimed[q] |= 2;
      return;
    }
    idx = (idx + 1) & P.hmask;
  }
  P.st[q] = ST_INVALID;                                 // table full -> capacity failure
  latch(P.sticky, RNNLM_E_CAPACITY);
}

// Final outcome of query q (a pending hidden-cache claim resolves to MISS for
// its owner, SHIT_NEW for the others) as (non-QHIT << 32 | MISS) flags.
__device__ __forceinline__ unsigned long long scan_flag(const Params &P, const CallArgs &A, uint32_t q, bool bad) {
  uint32_t st = P.st[q];
  const uint32_t sq = A.session[q], he = P.hent[q];
  if (bad) {
    if (st != ST_INVALID) latch(P.sticky, RNNLM_E_INVALID_ARG);
    st = ST_INVALID;
  } else if (st == ST_HNEED) {
    const uint32_t o = P.howner[(size_t)sq * (P.hmask + 1) + he];
    st = (o == q) ? ST_MISS : ST_SHIT_NEW;
    P.aux[q] = o;
  }
  P.st[q] = st;
  const uint32_t nonq = (st == ST_SHIT_OLD || st == ST_SHIT_NEW || st == ST_MISS || st == ST_MISS_NC);
  const uint32_t miss = (st == ST_MISS || st == ST_MISS_NC);
  return ((unsigned long long)nonq << 32) | miss;
}

// The scan's results for query q: exclusive prefixes, the session's segment
// start (first query of a session), the call totals (last query).
__device__ __forceinline__ void scan_store(const Params &P, const CallArgs &A, uint32_t q, uint32_t n, bool bad,
                                           unsigned long long run, unsigned long long v) {
  P.excl_nonq[q] = (uint32_t)(run >> 32);
  P.excl_miss[q] = (uint32_t)run;
  const uint32_t s = A.session[q];
  if (!bad && s < P.S && (q == 0 || A.session[q - 1] != s)) {
    P.seg_excl_nonq[s] = (uint32_t)(run >> 32);
    P.seg_excl_miss[s] = (uint32_t)run;
  }
  if (q == n - 1) {
    const unsigned long long tot = run + v;
    P.counts[0] = (uint32_t)(tot >> 32);
    P.counts[1] = (uint32_t)tot;
  }
}

// ---- (a4) commit: handles, slots, records, cache values, work lists -------
// Every load is issued before the first store (the compiler cannot move a load
// above a store it cannot prove disjoint), so the chain is per-query scratch ->
// {session segments and cursors, owners, parent record, owner's miss index}.
__device__ __forceinline__ void commit_query(const Params &P, const CallArgs &A, uint32_t q, uint32_t n) {
  const uint32_t st = P.st[q];
  const uint32_t s = A.session[q];
  const uint32_t snext = q + 1 < n ? A.session[q + 1] : NONE;
  const uint32_t w = A.word[q], p = A.parent[q];
  const uint32_t en = P.excl_nonq[q], r = P.excl_miss[q];
  const uint32_t qe = P.qent[q], he = P.hent[q], cs = P.cslot[q], ax = P.aux[q], ps = P.pslot[q];
  const uint8_t cl = P.claimed[q];
  const bool bad = P.counts[2] != 0u;
  const bool nonq = (st == ST_SHIT_OLD || st == ST_SHIT_NEW || st == ST_MISS || st == ST_MISS_NC);
  const bool miss = (st == ST_MISS || st == ST_MISS_NC);
  // second round trip (indices clamped in bounds; unused values are discarded)
  const uint32_t sc = s < P.S ? s : 0u;
  const size_t cb = (size_t)sc * P.cap;
  const size_t qb0 = (size_t)sc * (P.qmask + 1), hb0 = (size_t)sc * (P.hmask + 1);
  const uint32_t sen = P.seg_excl_nonq[sc], sem = P.seg_excl_miss[sc];
  const uint32_t nh0 = P.ctr[sc].next_handle, ns0 = P.ctr[sc].next_slot;
  const uint32_t qo = (cl & 1) ? P.qowner[qb0 + qe] : NONE;
  const uint32_t ho = (cl & 2) ? P.howner[hb0 + he] : NONE;
  const Rec pr = nonq ? P.rec[cb + (p < P.cap ? p : 0u)] : Rec{};
  const uint32_t eo = (nonq && st == ST_SHIT_NEW) ? P.excl_miss[ax] : 0u;
  if (!bad && s < P.S && snext != s) {                 // last of the session
    P.seg_cnt_nonq[s] = en + (nonq ? 1u : 0u) - sen;
    P.seg_cnt_miss[s] = r + (miss ? 1u : 0u) - sem;
  }
  // entries this query claimed AND owns: clear NEW_BIT (good batch) or remove
  // them again (rejected batch: every entry of this call goes, chains return
  // to their state before the call)
  if (qo == q) {
    QEntry *e = &P.qtab[qb0 + qe];
    if (bad) { e->tag = TAG_EMPTY; P.qowner[qb0 + qe] = NONE; }
    else e->tag &= ~NEW_BIT;
  }
  if (ho == q) {
    HEntry *e = &P.htab[hb0 + he];
    if (bad) { e->tag = TAG_EMPTY; P.howner[hb0 + he] = NONE; }
    else e->tag &= ~NEW_BIT;
  }
  if (!nonq) return;
  const uint32_t h = nh0 + (en - sen);
  ScoreItem it;
  it.pr = pr;
  it.q = q; it.s = s; it.w = w; it.pad = 0u;
  if (h >= P.cap) {                                    // out of history handles
    it.pr.slot = NONE;
    P.score_items[en] = it;
    P.st[q] = ST_INVALID;
    latch(P.sticky, RNNLM_E_CAPACITY);
    P.ctr[s].poisoned = 1u;                            // read from the next call on
    A.score[q] = __int_as_float(0x7fc00000);
    A.child[q] = NONE;
    if (P.cache) { P.qtab[qb0 + qe].child = NONE; P.qtab[qb0 + qe].score = __int_as_float(0x7fc00000); }
    if (miss) {                                        // a GRU row that is computed and discarded:
      P.row_src[r] = (uint32_t)cb;                     // in-range gather indices (the session's root)
      P.row_word[r] = 0u;
      P.row_dst[r] = NONE;
    }
    return;
  }
  uint32_t sl;
  if (miss) {
    sl = ns0 + (r - sem);
    P.row_src[r] = (uint32_t)(cb + ps);
    P.row_dst[r] = (uint32_t)(cb + sl);
    P.row_word[r] = w;
    if (P.cache) {
      P.htab[hb0 + he].slot = sl;
      P.codehash[cb + sl] = 0ull;                      // accumulated by the GRU epilogue
    }
  } else if (st == ST_SHIT_OLD) {
    sl = cs;
  } else {                                             // SHIT_NEW: the owner's new slot
    sl = ns0 + (eo - sem);
  }
  P.cslot[q] = sl;
  Rec nr;                                              // last N-1 words of (ctx o w)
  nr.slot = sl;
  nr.ctx[0] = P.N > 1 ? w : NONE;
#pragma unroll
  for (int j = 1; j < MAX_CTX; ++j) nr.ctx[j] = (uint32_t)j + 1 < P.N ? pr.ctx[j - 1] : NONE;   // static indices: registers
  P.rec[cb + h] = nr;
  P.score_items[en] = it;
  A.child[q] = h;
  if (P.cache) P.qtab[qb0 + qe].child = h;
}

// ---- (a7) final: QHIT results, outcomes, counters, cursors -----------------
// Warp-collective: all 32 lanes of a warp call it (q >= n: inactive lane).
__device__ __forceinline__ void final_query(const Params &P, const CallArgs &A, uint32_t q, uint32_t n) {
  const bool active = q < n;
  uint32_t st = active ? P.st[q] : ST_INVALID;
  const uint32_t s = active ? A.session[q] : NONE;
  uint8_t oc = RNNLM_INVALID;
  if (active) {
    if (st == ST_QHIT_OLD) {
      const rnnlm_dev::QEntry e = P.qtab[(size_t)s * (P.qmask + 1) + P.qent[q]];
      A.score[q] = e.score;
      A.child[q] = e.child;
      if (e.child == NONE) st = ST_INVALID; else oc = RNNLM_QHIT;   // entry of a failed query
    } else if (st == ST_QHIT_NEW) {
      // the owner's handle is final after k_commit; its score is copied by
      // k_dup_scores once k_score has run
      const uint32_t o = P.aux[q];
      const uint32_t c = A.child[o];
      A.child[q] = c;
      if (c == NONE) {
        st = ST_INVALID;
      } else {
        oc = RNNLM_QHIT;
        P.dup_list[atomicAdd(&P.counts[3], 1u)] = q;
      }
    } else if (st == ST_SHIT_OLD || st == ST_SHIT_NEW) {
      oc = RNNLM_SHIT;
    } else if (st == ST_MISS || st == ST_MISS_NC) {
      oc = RNNLM_MISS;
    }
    if (st == ST_INVALID) {
      A.score[q] = __int_as_float(0x7fc00000);
      A.child[q] = NONE;
    }
    if (A.outcome) A.outcome[q] = oc;
  }
  const bool valid = st != ST_INVALID;
  const uint32_t key = valid ? s : NONE;
  const uint32_t mask = __match_any_sync(0xffffffffu, key);
  const uint32_t c_tot = valid;
  const uint32_t c_qh = valid && (st == ST_QHIT_OLD || st == ST_QHIT_NEW);
  const uint32_t c_hl = valid && P.cache && !c_qh;
  const uint32_t c_hh = valid && (st == ST_SHIT_OLD || st == ST_SHIT_NEW);
  const uint32_t c_gru = valid && (st == ST_MISS || st == ST_MISS_NC);
  const uint32_t t_tot = __reduce_add_sync(mask, c_tot), t_qh = __reduce_add_sync(mask, c_qh);
  const uint32_t t_hl = __reduce_add_sync(mask, c_hl), t_hh = __reduce_add_sync(mask, c_hh);
  const uint32_t t_gru = __reduce_add_sync(mask, c_gru);
  if (key != NONE && (threadIdx.x & 31) == (uint32_t)(__ffs(mask) - 1)) {
    SessCtr *c = &P.ctr[key];
    if (t_tot) atomicAdd(&c->total, (unsigned long long)t_tot);
    if (t_qh) atomicAdd(&c->qhits, (unsigned long long)t_qh);
    if (t_hl) atomicAdd(&c->hlookups, (unsigned long long)t_hl);
    if (t_hh) atomicAdd(&c->hhits, (unsigned long long)t_hh);
    if (t_gru) atomicAdd(&c->gru, (unsigned long long)t_gru);
  }
  if (active && P.counts[2] == 0u && s < P.S && (q == n - 1 || A.session[q + 1] != s)) {
    SessCtr *c = &P.ctr[s];
    const uint32_t nh = c->next_handle + P.seg_cnt_nonq[s];
    const uint32_t ns = c->next_slot + P.seg_cnt_miss[s];
    c->next_handle = nh < P.cap ? nh : P.cap;
    c->next_slot = ns < P.cap ? ns : P.cap;
  }
}

}  // namespace rnnlm_dev
