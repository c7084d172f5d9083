"""World-size-2 gloo test of the multi-GPU host path on CPU.

Each rank owns a contiguous block of sessions (paper_1801_09866_b200.parallel),
runs them on its own engine (here the CPU oracle stands in for the per-GPU
engine, injected explicitly), and the per-frame (score, child) results are
all-gathered.  Rank 0 checks that the gathered results equal a single-process
run over all sessions bitwise (configuration invariance).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1801_09866_b200.parallel import all_gather_results, session_range, unpack_results


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_rank(rank, world, port, S, frames, B_s, result_q):
    import oracle as O
    from synth import generate_workload
    from synth.model import ModelDims, generate_model
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d = ModelDims(V=64, E=16, H=16, maxent_log2=10, N=4)
        m = generate_model(d, seed=5, scale=1.5)
        wl = generate_workload(S, frames, B_s, d.V, seed=3)
        lo, hi = session_range(S, world, rank)
        mine = wl.select_sessions(lo, hi)
        cap = wl.max_histories_hint()
        eng = O.Oracle(O.make_config(d.V, d.E, d.H, d.maxent_log2, d.N, O.KEY_SIGN, 0, 1,
                                     hi - lo, cap), m)
        child = np.zeros(mine.n_total, np.uint32)
        gathered = []
        for t in range(frames):
            sl = mine.frame_slice(t)
            par = O.resolve_parents(mine.parent_ref[sl], child)
            sc, ch, _ = eng.query_frame(mine.session[sl], par, mine.word[sl])
            child[sl] = ch
            out = all_gather_results(torch.from_numpy(sc), torch.from_numpy(ch.view(np.int32)))
            g_sc, g_ch = unpack_results(out)
            gathered.append((g_sc.numpy().copy(), g_ch.numpy().view(np.uint32).copy()))
        if rank == 0:
            result_q.put(gathered)
    finally:
        dist.destroy_process_group()


def test_sharded_gather_equals_single_process():
    import oracle as O
    from synth import generate_workload
    from synth.model import ModelDims, generate_model
    S, frames, B_s, world = 4, 12, 48, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_rank, args=(r, world, port, S, frames, B_s, q))
             for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    d = ModelDims(V=64, E=16, H=16, maxent_log2=10, N=4)
    m = generate_model(d, seed=5, scale=1.5)
    wl = generate_workload(S, frames, B_s, d.V, seed=3)
    ref = O.Oracle(O.make_config(d.V, d.E, d.H, d.maxent_log2, d.N, O.KEY_SIGN, 0, 1, S,
                                 wl.max_histories_hint()), m)
    sc, ch, _ = O.run_workload(ref, wl)
    for t in range(frames):
        sl = wl.frame_slice(t)
        g_sc, g_ch = gathered[t]
        # rank-major blocks of contiguous sessions == global session-major order
        assert np.array_equal(g_sc.view(np.uint32), sc[sl].view(np.uint32))
        assert np.array_equal(g_ch, ch[sl])


@pytest.mark.parametrize("total,world", [(64, 1), (64, 8), (10, 4), (3, 4)])
def test_session_range_even_split(total, world):
    sizes = [session_range(total, world, r) for r in range(world)]
    assert sizes[0][0] == 0 and sizes[-1][1] == total
    for (a, b), (c, _) in zip(sizes, sizes[1:]):
        assert b == c
    lens = [b - a for a, b in sizes]
    assert max(lens) - min(lens) <= 1 and lens == sorted(lens, reverse=True)
