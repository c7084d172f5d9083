#!/usr/bin/env python
"""Benchmark of the frame-batched GRU-RNNLM query step (BASELINE.json metric).

    python bench.py --gpus N --steps K --warmup W [--workload multi] [--math bf16]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference ...        (the CPU oracle arm)

A step = one decoder frame of every session this rank owns: one
rnnlm_query_batch call that runs the whole hot path (keys, both caches,
compaction, gather + GRU, NCE + MaxEnt scoring, result write) over that
frame's queries.  Workload: BASELINE.json configs[4] ("multi": 64 utterance
streams x 2,048 queries/frame on the large model, V=200k, H=E=1024, 2^27
4-gram MaxEnt) per GPU (weak scaling: sessions are independent units,
DESIGN.md "Multi-GPU"); synthetic, seeded (synth/).  The per-query results
(score, child) of every step are all-gathered over NCCL on a side stream when
N > 1.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import CONFIGS, generate_model, generate_workload, model_dims  # noqa: E402

METRIC = "RNNLM queries/sec (frame-batched, cache on)"
UNIT = "queries/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="multi", choices=list(CONFIGS))
    ap.add_argument("--sessions", type=int, default=None, help="sessions per rank (default: config)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--math", default="bf16", choices=["bf16", "tf32", "fp32", "tf32x3"])
    ap.add_argument("--key", default="sign", help="off | sign | round:K")
    ap.add_argument("--cell", default="gru", choices=["gru", "lbr", "rnn"],
                    help="recurrent cell (SURVEY 8(f)-3): gru = Chung GRU (the paper's), lbr = linear before "
                         "reset, rnn = the paper's comparison vanilla RNN (Elman, logistic)")
    ap.add_argument("--no-cache", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--prefill", type=int, default=40,
                    help="untimed frames run before warm-up so timed frames are mid-utterance")
    ap.add_argument("--uniform-words", action="store_true", help="(ncu evidence) no Zipf reuse")
    ap.add_argument("--timing-level", type=int, default=1, help="1: kernel groups, 2: + GRU kernels")
    ap.add_argument("--normalizer", action="store_true",
                    help="SURVEY 8(f)-2 workload: exact log-normalisers/s instead of the query step")
    ap.add_argument("--histories", type=int, default=2048, help="(--normalizer) histories per call")
    ap.add_argument("--offline", action="store_true",
                    help="SURVEY 8(f)-4 workload: whole utterances rescored level by level (2-pass) vs frame by frame")
    ap.add_argument("--frames", type=int, default=None, help="(--offline) frames per utterance (default: config)")
    ap.add_argument("--trace", default=None,
                    help="(diagnostics) write a CUPTI kernel timeline of the timed steps (chrome trace JSON); "
                         "the printed numbers of such a run are not bench values")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def sessions_for(args, world):
    S = args.sessions or CONFIGS[args.workload]["S"]
    if args.scaling == "strong":
        assert S % world == 0, "strong scaling needs sessions divisible by world size"
        return S // world
    return S


def key_mode(name):
    from paper_1801_09866_b200 import KEY_MODES
    return KEY_MODES[name]


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- oracle timing
def time_oracle(dims, model, wl, mode, k, cache, budget_s, max_steps=None, cell=0):
    """The CPU oracle as it stands (single thread), on a bounded prefix of the
    workload's first session.  Returns (queries, seconds, frames)."""
    import oracle as O
    one = wl.select_sessions(0, 1)
    cfg = O.make_config(dims.V, dims.E, dims.H, dims.maxent_log2, dims.N, mode, k,
                        1 if cache else 0, 1,
                        one.max_histories_hint() if cache else one.frames * one.B_s + 2, cell=cell)
    orc = O.Oracle(cfg, model)
    child = np.zeros(one.n_total, np.uint32)
    done_q, t_total, f = 0, 0.0, 0
    per_step = []
    while f < one.frames and t_total < budget_s and (max_steps is None or f < max_steps):
        sl = one.frame_slice(f)
        par = O.resolve_parents(one.parent_ref[sl], child)
        t0 = time.perf_counter()
        _, ch, _ = orc.query_frame(one.session[sl], par, one.word[sl])
        dt = time.perf_counter() - t0
        child[sl] = ch
        done_q += len(par)
        t_total += dt
        per_step.append(dt)
        f += 1
    return done_q, t_total, f, per_step


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    c = CONFIGS[args.workload]
    dims = model_dims(args.workload)
    model = generate_model(dims, seed=1234)
    mode, k = key_mode(args.key)
    steps = args.warmup + args.steps
    wl = generate_workload(1, steps, c["B_s"], dims.V, seed=7)
    # each step = one frame of one utterance stream (bounded sample of the workload)
    q, secs, frames, per = time_oracle(dims, model, wl, mode, k, not args.no_cache, 1e30,
                                       max_steps=steps, cell={"gru": 0, "lbr": 1, "rnn": 2}[args.cell])
    timed = per[args.warmup:]
    tq = c["B_s"] * len(timed)
    value = tq / sum(timed)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(timed) / len(timed), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "key": args.key,
                   "sample": f"1 session x {c['B_s']} queries per step (frames {args.warmup}.."
                             f"{steps - 1} of utterance 0)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{len(timed)} frames x {c['B_s']} queries, session 0",
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.p = None
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out = ""
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1801_09866_b200 as R
    from paper_1801_09866_b200.parallel import all_gather_results

    rank, world, local = dist_env()
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    # One rank per GPU.  RNNLM_BENCH_SHARED_GPU=1 (code-path check on a one-GPU
    # box only: ranks share device 0 and the collectives go through gloo) --
    # numbers of such a run are not bench values.
    shared = os.environ.get("RNNLM_BENCH_SHARED_GPU") == "1"
    local = local % torch.cuda.device_count() if shared else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    c = CONFIGS[args.workload]
    dims = model_dims(args.workload)
    S = sessions_for(args, world)
    B_s = c["B_s"]
    F0 = args.prefill
    # two timed passes of K frames each: A (the bench value, no library timing
    # events) then B (per-kernel CUDA events inside the library: roofline)
    frames = F0 + args.warmup + 2 * args.steps
    model = generate_model(dims, seed=1234)
    V_draw = dims.V
    wl = generate_workload(S, frames, B_s, V_draw, seed=7 + rank * S,
                           zipf_s=0.0 if args.uniform_words else 1.0)
    mode, k = key_mode(args.key)
    math = {"bf16": R.MATH_BF16, "tf32": R.MATH_TF32, "fp32": R.MATH_FP32, "tf32x3": R.MATH_TF32X3}[args.math]
    n = wl.n_per_frame
    # cache off: every valid query makes a new history (reading 23), so the
    # per-session pool must hold one per query of the run
    cap = wl.max_histories_hint() if not args.no_cache else frames * B_s + 2
    eng = R.RNNLM.from_dims(dims, model, key_mode=mode, round_digits=k, math=math,
                            cell={"gru": R.CELL_GRU, "lbr": R.CELL_GRU_LBR, "rnn": R.CELL_RNN}[args.cell],
                            cache_enabled=not args.no_cache, num_sessions=S,
                            max_queries_per_call=n, max_histories_per_session=cap, device=local)

    d_sess = torch.as_tensor(wl.session.view(np.int32), device=dev)
    d_word = torch.as_tensor(wl.word.view(np.int32), device=dev)
    d_ref = torch.as_tensor(wl.parent_ref, device=dev)
    d_child = torch.zeros(wl.n_total, dtype=torch.int32, device=dev)
    d_score = torch.zeros(wl.n_total, dtype=torch.float32, device=dev)
    d_par = torch.zeros(n, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)        # > 126 MB L2
    side = torch.cuda.Stream(device=dev)
    gathered = torch.empty((world * n, 2), dtype=torch.int32, device=dev) if world > 1 else None
    main = torch.cuda.current_stream()

    def step(t, timed_events=None):
        sl = wl.frame_slice(t)
        R.resolve_parents(d_ref[sl], d_child, d_par)
        if timed_events is not None:
            timed_events[0].record()
        eng.query_batch(d_sess[sl], d_par, d_word[sl], score=d_score[sl], child=d_child[sl],
                        want_outcome=False)
        if timed_events is not None:
            timed_events[1].record()
        if world > 1:
            ev = torch.cuda.Event()
            ev.record(main)
            side.wait_event(ev)
            with torch.cuda.stream(side):
                all_gather_results(d_score[sl], d_child[sl], out=gathered)

    # ---- prefill (utterance start, untimed) + warm-up
    for t in range(F0 + args.warmup):
        step(t)
    torch.cuda.synchronize()

    def timed_pass(t_lo, t_hi, level, trace=None):
        """Frames [t_lo, t_hi), one event pair per step (resolve kernel + step;
        the L2 flush is between pairs).  Returns (ms over ranks: max, library
        timing, cache-stat deltas, our launches, clocks)."""
        st0 = eng.cache_stats()
        eng.set_timing(level)
        eng.get_timing(reset=True)
        l0 = eng.launch_count()
        clocks = ClockSampler(local)
        time.sleep(0.3)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(t_hi - t_lo)]
        prof = None
        if trace:
            from torch.profiler import ProfilerActivity, profile
            prof = profile(activities=[ProfilerActivity.CUDA])
            prof.__enter__()
        for i, t in enumerate(range(t_lo, t_hi)):
            flush.zero_()
            sl = wl.frame_slice(t)
            evs[i][0].record()
            R.resolve_parents(d_ref[sl], d_child, d_par)
            eng.query_batch(d_sess[sl], d_par, d_word[sl], score=d_score[sl], child=d_child[sl],
                            want_outcome=False)
            if world > 1:
                ev = torch.cuda.Event()
                ev.record(main)
                side.wait_event(ev)
                with torch.cuda.stream(side):
                    all_gather_results(d_score[sl], d_child[sl], out=gathered)
            evs[i][1].record()
        torch.cuda.synchronize()
        if prof is not None:
            prof.__exit__(None, None, None)
            prof.export_chrome_trace(trace)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk = clocks.stop()
        timing = eng.get_timing(reset=True)
        eng.set_timing(0)
        launches = eng.launch_count() - l0 + (t_hi - t_lo)      # + resolve_parents kernels
        st1 = eng.cache_stats()
        total_ms = float(sum(a.elapsed_time(b) for a, b in evs))
        gru_ms = timing["ms_gru"]
        if world > 1:
            tt = torch.tensor([total_ms, gru_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            total_ms = float(tt[0])
        d = {kk: st1[kk] - st0[kk] for kk in ("total_queries", "query_hits", "hidden_lookups",
                                              "hidden_hits", "gru_computations")}
        return total_ms, timing, d, launches, clk

    tA = F0 + args.warmup
    tB = tA + args.steps
    total_ms, _, d_stats, launches, clk = timed_pass(tA, tB, 0, args.trace)
    # level 2: events around the fused GRU kernel itself (k_gru_tc), after the A1 gather
    ms_B, timing, d_B, _, _ = timed_pass(tB, tB + args.steps, max(2, args.timing_level))
    queries_rank = n * args.steps
    total_queries = queries_rank * world
    value = total_queries / (total_ms / 1e3)
    rows = d_B["gru_computations"]
    gates = 1 if args.cell == "rnn" else 3                 # vanilla RNN: one gate
    flops = 2.0 * gates * dims.H * (dims.E + dims.H) * rows   # [Q, E+H] x [E+H, gates*H], 2 flop/MAC
    # the dominant kernel's own time: the fused GRU kernel (tensor-core paths) or
    # the two SIMT GRU kernels (FP32), without the A1 gather / cache front
    k_ms = timing["ms_gru_phase1"] + timing["ms_gru_phase2"] if math != R.MATH_FP32 else timing["ms_gru"]
    gru_s = k_ms / 1e3
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    if math == R.MATH_BF16:
        peak = peaks.get("bf16_tflops_sustained", 1400.0)
        bound, peak_src = "tensor", ("measured bf16_tflops_sustained" if peaks else "fallback")
    elif math == R.MATH_TF32X3:
        # three TF32 products per useful multiply-add: useful-flop peak = TF32 peak / 3
        peak = 0.5 * peaks.get("bf16_tflops_sustained", 1400.0) / 3.0
        bound, peak_src = "tensor", ("measured bf16_tflops_sustained x 0.5 (tf32/bf16 dense ratio) / 3 "
                                     "(three TF32 products per useful MAC)")
    elif math == R.MATH_TF32:
        # no measured TF32 peak: the measured bf16 peak x the nominal dense ratio (1.125 / 2.25 PF)
        peak = 0.5 * peaks.get("bf16_tflops_sustained", 1400.0)
        bound, peak_src = "tensor", "measured bf16_tflops_sustained x 0.5 (nominal tf32/bf16 dense ratio)"
    else:
        sm_max = peaks.get("sm_max_mhz", 1965.0)
        peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12     # FP32 FFMA lanes x 2 flop x clock
        bound, peak_src = "alu", "derived: 148 SMs x 128 FP32 lanes x 2 x sm_max_mhz"
    achieved = flops / gru_s / 1e12 if gru_s > 0 else 0.0
    # the library runs the CTA-pair kernel for the bf16 GRU when H % 256 == 0
    # (gru_tc_prepare; RNNLM_TC_PAIR=0 selects one CTA per tile)
    pair = (math == R.MATH_BF16 and args.cell == "gru" and dims.H % 256 == 0
            and os.environ.get("RNNLM_TC_PAIR", "1") != "0")
    gru_kernel = "k_gru_tc2" if pair else "k_gru_tc"
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        # captured for the paper's cell only; other cells report no traffic figure
        ent = prof.get(args.workload, {}).get(args.math, {}) if args.cell == "gru" else {}
        traffic = ent.get("kernels", {}).get(gru_kernel, ent.get("gru_dram_bytes_per_step"))
    except Exception:
        pass
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None,
        "dtype": {"bf16": "bf16", "tf32": "tf32", "fp32": "f32", "tf32x3": "f32 (3xTF32)"}[args.math], "data": "synthetic",
        "config": {"workload": args.workload, "sessions_per_gpu": S, "queries_per_session_frame": B_s,
                   "queries_per_step": total_queries // args.steps, "V": dims.V, "E": dims.E,
                   "H": dims.H, "maxent": f"2^{dims.maxent_log2} {dims.N}-gram", "key": args.key,
                   "cache": not args.no_cache, "math": args.math, "cell": args.cell,
                   "l2": "flushed between timed steps (256 MiB write outside the event pair)",
                   "timed_frames": f"value: frames {tA}..{tB - 1}; roofline pass (library kernel events on): frames {tB}..{frames - 1} ({F0} prefill + {args.warmup} warm-up frames untimed)",
                   "parallelism": f"dp{world} (sessions sharded, weights replicated, NCCL all-gather of (score, child))"},
        "roofline": {"kernel": ((f"{gru_kernel} (fused tcgen05 GRU, both phases"
                                 + (", CTA pair)" if pair else ")")) if math != R.MATH_FP32
                                else "k_gru1_f32 + k_gru2_f32 (+ gather, FP32 SIMT)"), "bound": bound,
                     "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                     "traffic": traffic, "peak_source": peak_src,
                     "algorithmic": f"{2 * gates}*H*(E+H) flop x {rows} GRU rows over {args.steps} steps",
                     "kernel_ms_per_step": k_ms / args.steps,
                     "gather_plus_kernel_ms_per_step": timing["ms_gru"] / args.steps,
                     "share_of_step": (k_ms / ms_B) if ms_B else None},
        "kernel_ms_per_step": {kk: timing[kk] / args.steps for kk in
                               ("ms_cache", "ms_score", "ms_gru", "ms_encode", "ms_final",
                                "ms_gru_gather", "ms_gru_phase1", "ms_gru_phase2")},
        "hit_rates": {"query_cache": d_stats["query_hits"] / max(1, d_stats["total_queries"]),
                      "hidden_cache": d_stats["hidden_hits"] / max(1, d_stats["hidden_lookups"]),
                      "gru_rows_per_step": d_stats["gru_computations"] / args.steps},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    # ---- e2e: same metric through the C ABI with host buffers, copies inside the timed region
    if not args.no_e2e:
        e2e = run_e2e(args, eng, wl, dev, world)
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        q, secs, f, _ = time_oracle(dims, model, wl, mode, k, not args.no_cache, args.cpu_seconds,
                                    cell={"gru": 0, "lbr": 1, "rnn": 2}[args.cell])
        line["cpu_baseline"] = {"value": q / secs, "unit": UNIT, "cores": 1, "kind": "oracle",
                                "sample": f"session 0, frames 0..{f - 1} ({q} queries, {secs:.1f} s)",
                                "cpu": cpu_model(), "host_cores": host_cores()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, eng, wl, dev, world):
    """Host-buffer path through the public C ABI: per step H2D of the decoder's
    queries (session, parent reference = index of the earlier query whose child
    is the parent, word) from pinned memory, rnnlm_resolve_parents (reference
    -> handle, on the device, from the children the engine returned),
    rnnlm_query_batch, D2H of (score, child) into pinned memory, synchronise."""
    import torch
    import torch.distributed as dist
    n = wl.n_per_frame
    eng.reset_session()
    import paper_1801_09866_b200 as R
    # per frame one contiguous pinned record block [ref i64 | session u32 | word u32] x n
    # (16 B per query), so each step's inputs are ONE host->device copy
    F = wl.frames
    blk = np.empty((F, 4 * n), dtype=np.int32)
    for t in range(F):
        sl = wl.frame_slice(t)
        blk[t, :2 * n] = np.ascontiguousarray(wl.parent_ref[sl], dtype=np.int64).view(np.int32)
        blk[t, 2 * n:3 * n] = wl.session[sl].view(np.int32)
        blk[t, 3 * n:] = wl.word[sl].view(np.int32)
    h_in_all = torch.from_numpy(blk).pin_memory()
    h_out = torch.empty(2 * n, dtype=torch.int32).pin_memory()      # [score bits | child]
    d_in = torch.empty(4 * n, dtype=torch.int32, device=dev)
    d_ref = d_in[:2 * n].view(torch.int64)
    d_sess, d_word = d_in[2 * n:3 * n], d_in[3 * n:]
    d_par = torch.empty(n, dtype=torch.int32, device=dev)
    d_out = torch.empty(2 * n, dtype=torch.int32, device=dev)
    d_score = d_out[:n].view(torch.float32)
    d_child_log = torch.zeros(wl.n_total, dtype=torch.int32, device=dev)

    def host_step(t):
        sl = wl.frame_slice(t)
        d_in.copy_(h_in_all[t], non_blocking=True)
        R.resolve_parents(d_ref, d_child_log, d_par)
        eng.query_batch(d_sess, d_par, d_word, score=d_score, child=d_child_log[sl], want_outcome=False)
        d_out[n:].copy_(d_child_log[sl])
        h_out.copy_(d_out, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    F0 = args.prefill
    for t in range(F0 + args.warmup):
        host_step(t)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t in range(F0 + args.warmup, F0 + args.warmup + args.steps):
        host_step(t)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([secs], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        secs = float(tt[0])
    return {"value": n * args.steps * world / secs, "unit": UNIT,
            "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 8 * n,
            "note": "wall clock per step: H2D (session u32, parent reference i64, word u32) from pinned "
                    "memory, device-side reference -> handle resolution, the step, D2H (score, child), "
                    "synchronise; per rank, max over ranks"}


def run_normalizer(args):
    """throughput of the exact log-normaliser (rnnlm_log_normalizer)
    on the large model (V = 200k, H = 1024, 4-gram MaxEnt 2^27): log Z of
    --histories distinct stored histories per call (the 2,048 queries/frame of
    BASELINE configs[2]), device-timed with CUDA events; one JSON line.
    Roofline of the dominant kernel (k_norm_tc): its algorithmic traffic is
    the MaxEnt gathers, (K - 1) random 4-byte reads = 32-byte sectors per
    (history, word) (order 1 is a per-word bias), plus one pass over the bf16
    output rows per 128-history tile; the contraction (two bf16 MMAs per
    element pair) is reported beside it."""
    import torch

    import paper_1801_09866_b200 as R
    from synth import generate_model, generate_workload, model_dims

    d = model_dims("large")
    m = generate_model(d, seed=1234)
    n = args.histories
    # distinct histories: one utterance, cache off, 2 frames of n/2 queries
    # each -> every query makes a new history (depth 1 and 2)
    wl = generate_workload(1, 2, n // 2, d.V, seed=5)
    math = {"bf16": R.MATH_BF16, "tf32": R.MATH_TF32, "fp32": R.MATH_FP32, "tf32x3": R.MATH_TF32X3}[args.math]
    eng = R.RNNLM.from_dims(d, m, key_mode=R.KEY_SIGN, math=math, cache_enabled=False, num_sessions=1,
                            max_queries_per_call=n, max_histories_per_session=n + 2)
    dev = torch.device("cuda", 0)
    child = torch.zeros(wl.n_total, dtype=torch.int32, device=dev)
    ref = torch.as_tensor(wl.parent_ref, device=dev)
    par = torch.zeros(wl.n_per_frame, dtype=torch.int32, device=dev)
    for t in range(wl.frames):
        sl = wl.frame_slice(t)
        R.resolve_parents(ref[sl], child, par)
        s_ = torch.as_tensor(wl.session[sl].view(np.int32), device=dev)
        w_ = torch.as_tensor(wl.word[sl].view(np.int32), device=dev)
        eng.query_batch(s_, par, w_, score=torch.empty(wl.n_per_frame, device=dev), child=child[sl],
                        want_outcome=False)
    torch.cuda.synchronize()
    hist = torch.arange(1, n + 1, dtype=torch.int32, device=dev)       # handles 1..n (0 = root)
    sess = torch.zeros(n, dtype=torch.int32, device=dev)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        eng.log_normalizer(sess, hist, out=out)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in evs:
        a.record()
        eng.log_normalizer(sess, hist, out=out)
        b.record()
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    assert torch.isfinite(out).all()
    K = d.N
    sectors = n * d.V * (K - 1) * 32.0
    theta = -(-n // 128) * d.V * d.H * 2.0
    flops = 2.0 * 2.0 * n * d.V * d.H
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs", 6458.1)
    gbs = (sectors + theta) / (ms * 1e-3) / 1e9
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))["normalizer"]["bf16"][
            "k_norm_tc_dram_bytes_per_launch"]
    except Exception:
        pass
    line = {
        "metric": "exact log-normalisers/sec (large model, V=200k, 4-gram MaxEnt)", "value": n / (ms * 1e-3),
        "unit": "histories/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "dtype": "bf16x2", "data": "synthetic",
        "config": {"workload": "normalizer", "histories_per_call": n, "V": d.V, "H": d.H,
                   "maxent": f"2^{d.maxent_log2} {d.N}-gram", "engine_math": args.math,
                   "l2": "inputs (1.6 GB of gathers + 6.5 GB of output rows per call) exceed L2"},
        "roofline": {"kernel": "k_norm_tc (contraction + MaxEnt gathers + online log-sum-exp)", "bound": "hbm",
                     "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                     "algorithmic": f"{n} x {d.V} x {K - 1} random 32-B MaxEnt sectors + {-(-n // 128)} passes "
                                    f"over the bf16 output rows",
                     "traffic": traffic, "contraction_tflops": flops / (ms * 1e-3) / 1e12},
    }
    if not args.no_cpu_baseline:
        import oracle as O
        orc = O.Oracle(O.make_config(d.V, d.E, d.H, d.maxent_log2, d.N, O.KEY_OFF, 0, 0, 1, n + 2), m)
        st = eng.read_states(0, np.arange(1, 3, dtype=np.uint32)).cpu().numpy()
        t0 = time.perf_counter()
        cfg = O.make_config(d.V, d.E, d.H, d.maxent_log2, d.N)
        for i in range(2):
            O.log_normalizer(cfg, m, st[i], [int(wl.word[i])])
        secs = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": 2 / secs, "unit": "histories/s", "cores": 1, "kind": "oracle",
                                "sample": f"2 histories ({secs:.1f} s)"}
        del orc
    print(json.dumps(line), flush=True)


def run_offline(args):
    """whole utterances known in advance (2-pass lattice
    rescoring) scheduled level by level (paper_1801_09866_b200.offline)
    instead of one call per frame.  Both schedules run the same synthetic
    utterances on the same engine settings; each is device-timed with CUDA
    events around the whole stream (after one untimed warm-up pass)."""
    import torch

    import paper_1801_09866_b200 as R
    from paper_1801_09866_b200.offline import OfflineRunner

    c = CONFIGS[args.workload]
    dims = model_dims(args.workload)
    S = args.sessions or c["S"]
    frames = args.frames or c["frames"]
    model = generate_model(dims, seed=1234)
    wl = generate_workload(S, frames, c["B_s"], dims.V, seed=7)
    mode, k = key_mode(args.key)
    math = {"bf16": R.MATH_BF16, "tf32": R.MATH_TF32, "fp32": R.MATH_FP32, "tf32x3": R.MATH_TF32X3}[args.math]
    dev = torch.device("cuda", 0)
    Bmax = 32768
    cap = wl.max_histories_hint()

    def engine(B):
        return R.RNNLM.from_dims(dims, model, key_mode=mode, round_digits=k, math=math, num_sessions=S,
                                 max_queries_per_call=B, max_histories_per_session=cap)

    d_sess = torch.as_tensor(wl.session.view(np.int32), device=dev)
    d_word = torch.as_tensor(wl.word.view(np.int32), device=dev)
    d_ref = torch.as_tensor(wl.parent_ref, device=dev)
    on = engine(wl.n_per_frame)
    d_child = torch.zeros(wl.n_total, dtype=torch.int32, device=dev)
    d_score = torch.zeros(wl.n_total, dtype=torch.float32, device=dev)
    d_par = torch.zeros(wl.n_per_frame, dtype=torch.int32, device=dev)

    def online():
        on.reset_session()
        for t in range(wl.frames):
            sl = wl.frame_slice(t)
            R.resolve_parents(d_ref[sl], d_child, d_par)
            on.query_batch(d_sess[sl], d_par, d_word[sl], score=d_score[sl], child=d_child[sl], want_outcome=False)

    off = engine(Bmax)
    runner = OfflineRunner(off, wl, max_batch=Bmax)

    def offline():
        off.reset_session()
        runner.run()

    def timed(fn):
        fn()                                                     # warm-up pass
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    ms_on = timed(online)
    ms_off = timed(offline)
    same = bool(torch.equal(d_score, runner.score)) if mode == R.KEY_OFF else None
    nb = len(runner.batches)
    line = {
        "metric": "RNNLM queries/sec (offline level-batched rescoring of whole utterances)",
        "value": wl.n_total / (ms_off * 1e-3), "unit": "queries/s", "n_gpus": 1, "steps": 1, "warmup": 1,
        "ms_per_step": ms_off, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": {"bf16": "bf16", "tf32": "tf32", "fp32": "f32", "tf32x3": "f32 (3xTF32)"}[args.math], "data": "synthetic",
        "config": {"workload": args.workload, "sessions": S, "frames": frames, "queries": int(wl.n_total),
                   "key": args.key, "math": args.math, "offline_calls": nb, "online_calls": frames,
                   "mean_queries_per_offline_call": wl.n_total / max(1, nb),
                   "step": "one pass over the whole query stream"},
        "online": {"value": wl.n_total / (ms_on * 1e-3), "ms": ms_on},
        "speedup_vs_online": ms_on / ms_off,
        "scores_bitwise_equal_online": same,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.offline:
        if args.impl == "reference" or dist_env()[1] > 1:
            raise SystemExit("--offline: one GPU, our implementation only")
        run_offline(args)
    elif args.normalizer:
        if args.impl == "reference" or dist_env()[1] > 1:
            raise SystemExit("--normalizer: one GPU, our implementation only")
        run_normalizer(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
