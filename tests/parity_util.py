"""Replay-protocol parity driver: CUDA path vs CPU oracle.

Per frame: both sides get the same queries (parents resolved from their own
returned handles), then
  * outcomes, child handles and state slots must be bit-exact,
  * scores within ``tol_score`` (absolute),
  * every new state (MISS) within ``tol_state`` of the oracle's fp64 GRU,
  * the stored compression codes of new states bit-exact vs the oracle's
    compress() of the SAME (GPU) vector,
and finally the oracle's new states are overwritten with the GPU's, so the
next frame's keys on both sides are computed from identical vectors
("computed from identical input vectors", BASELINE.json north_star).

Used by tests/ and by __graft_entry__.smoke() only.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle as O


def _dev(a, device="cuda"):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32), device=device)


def replay_compare(eng, orc, wl, frames=None, tol_score=1e-5, tol_state=1e-5, check_codes=True,
                   batches=None, only_session=None):
    """``batches``: the calls to make, as index arrays into the workload's
    query stream (default: one call per frame, the first ``frames`` frames);
    e.g. one call per query or the offline level schedule
    (8(f)-4).  Both sides get the same calls.  ``only_session``: the engine
    runs every session of each call (the full-size launch), the oracle (a
    one-session engine) replays that session's queries only, and everything
    is compared for that session (sessions are independent)."""
    if batches is None:
        F = wl.frames if frames is None else frames
        batches = [np.arange(wl.frame_slice(t).start, wl.frame_slice(t).stop) for t in range(F)]
    child_g = np.zeros(wl.n_total, np.uint32)
    child_o = np.zeros(wl.n_total, np.uint32)
    rep = dict(max_score_err=0.0, max_state_err=0.0, frames=len(batches), queries=0, miss=0, shit=0,
               qhit=0, invalid=0)
    for t, sl in enumerate(batches):
        pg = O.resolve_parents(wl.parent_ref[sl], child_g)
        po = O.resolve_parents(wl.parent_ref[sl], child_o)
        sess = wl.session[sl]
        mine = slice(None) if only_session is None else sess == only_session
        assert np.array_equal(pg[mine], po[mine]), f"frame {t}: parent handles diverged"
        sc, ch, oc = eng.query_batch(_dev(sess), _dev(pg), _dev(wl.word[sl]))
        gsc = sc.cpu().numpy()
        gch = ch.cpu().numpy().view(np.uint32)
        goc = oc.cpu().numpy()
        if only_session is not None:                   # keep this session's queries, oracle session 0
            keep = sess == only_session
            child_g[sl] = gch
            sl = np.asarray(sl)[keep] if not isinstance(sl, slice) else np.arange(sl.start, sl.stop)[keep]
            sess, pg, po = sess[keep], pg[keep], po[keep]
            gsc, gch, goc = gsc[keep], gch[keep], goc[keep]
            osc, och, ooc = orc.query_frame(np.zeros_like(sess), po, wl.word[sl])
        else:
            osc, och, ooc = orc.query_frame(sess, po, wl.word[sl])
        bad = np.nonzero(goc != ooc)[0]
        assert len(bad) == 0, (f"frame {t}: outcome mismatch at {bad[:8]}: gpu {goc[bad[:8]]} "
                               f"oracle {ooc[bad[:8]]}")
        assert np.array_equal(gch, och), f"frame {t}: child handles differ"
        valid = ooc != O.INVALID
        assert np.array_equal(np.isnan(gsc), np.isnan(osc))
        if valid.any():
            err = float(np.max(np.abs(gsc[valid] - osc[valid])))
            rep["max_score_err"] = max(rep["max_score_err"], err)
            assert err <= tol_score, f"frame {t}: score error {err}"
        child_g[sl] = gch
        child_o[sl] = och
        rep["queries"] += len(sess)
        rep["miss"] += int(np.sum(ooc == O.MISS))
        rep["shit"] += int(np.sum(ooc == O.SHIT))
        rep["qhit"] += int(np.sum(ooc == O.QHIT))
        rep["invalid"] += int(np.sum(ooc == O.INVALID))
        for s in np.unique(sess):
            so = 0 if only_session is not None else int(s)          # the oracle's session
            m = (sess == s) & valid & (ooc != O.QHIT)
            if not m.any():
                continue
            hs = gch[m]
            gs = eng.read_slots(int(s), hs).cpu().numpy().view(np.uint32)
            assert np.array_equal(gs, orc.read_slots(so, hs)), f"frame {t}: slots differ"
            mm = (sess == s) & (ooc == O.MISS)
            if not mm.any():
                continue
            hm = gch[mm]
            gst = eng.read_states(int(s), hm).cpu().numpy()
            ost = orc.read_states(so, hm)
            err = float(np.max(np.abs(gst - ost)))
            rep["max_state_err"] = max(rep["max_state_err"], err)
            assert err <= tol_state, f"frame {t}: state error {err}"
            if check_codes and eng.cfg.cache_enabled:
                gcode = eng.read_codes(int(s), hm).cpu().numpy()
                for i in range(len(hm)):
                    ref = O.compress(gst[i], eng.cfg.key_mode, eng.cfg.round_digits)
                    assert np.array_equal(gcode[i], ref), f"frame {t}: code of handle {hm[i]} differs"
            for i, hd in enumerate(hm):
                orc.overwrite_state(so, int(hd), gst[i])
    gst = eng.cache_stats() if only_session is None else eng.cache_stats(only_session)
    ost = orc.stats()
    for k in ("total_queries", "query_hits", "hidden_lookups", "hidden_hits", "gru_computations",
              "sticky_error"):
        assert gst[k] == ost[k], f"stat {k}: gpu {gst[k]} oracle {ost[k]}"
    rep["stats"] = gst
    return rep
