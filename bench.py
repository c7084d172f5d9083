#!/usr/bin/env python
"""Benchmark of the frame-batched GRU-RNNLM query step (BASELINE.json metric).

    python bench.py --gpus N --steps K --warmup W
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference ...        (the CPU oracle arm)

A step = one decoder frame of every utterance stream this rank owns: one
rnnlm_query_batch call that runs the whole hot path (keys, both caches,
compaction, gather + GRU, NCE + MaxEnt scoring, result write) over that
frame's queries, plus (N > 1) the NCCL all-gather of the per-query
(score, child) results.

Headline workload: BASELINE.json configs[4] ("multi": 64 concurrent utterance
streams x 2,048 queries/frame on the large model, V=200k, H=E=1024, 2^27
4-gram MaxEnt, sign keys), the 64 streams SHARDED over the N GPUs (strong
scaling, "evenly distributing the block").  The streams are not in
step: stream s joins at frame s * (T0 / 64) of a 400-frame (4-s) run,
so the timed frames see the streams at every point of their utterances.
Synthetic and seeded (synth/).  The headline arithmetic is the paper's
single precision: the fp32-accurate 3xTF32 tensor-core mode, held to
the FP32 path's 1e-5 in tests; the bf16 tensor-core numbers of the same
frames are the "bf16" key.  "configs" carries BASELINE configs[0]-[3]
(tiny, moderate, large, compression sweep), one GPU, measured in the same run.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import gc
import ctypes
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
UTT_FRAMES = 400            # a 4-s utterance at 10 ms frames
TOTAL_STREAMS = 64          # BASELINE configs[4]
MATHS = ("bf16", "tf32", "fp32", "tf32x3", "bf16x3")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="multi", choices=list(CONFIGS))
    ap.add_argument("--sessions", type=int, default=None, help="streams in the job (default: config)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong: the job's streams are split over the ranks (BASELINE configs[4]); "
                         "weak: every rank runs that many streams")
    ap.add_argument("--math", default="bf16x3", choices=MATHS, help="headline arithmetic")
    ap.add_argument("--also", default="bf16,tf32x3", help="extra math modes measured on the same frames (comma list, or none)")
    ap.add_argument("--key", default="sign", help="off | sign | round:K")
    ap.add_argument("--cell", default="gru", choices=["gru", "lbr", "rnn"],
                    help="recurrent cell (SURVEY 8(f)-3): gru = Chung GRU (the paper's), lbr = linear before "
                         "reset, rnn = the paper's comparison vanilla RNN (Elman, logistic)")
    ap.add_argument("--no-cache", action="store_true")
    ap.add_argument("--no-stagger", action="store_true", help="all streams start together (frame 0)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the configs[0]-[3] block")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--uniform-words", action="store_true", help="(ncu evidence) no Zipf reuse")
    ap.add_argument("--timing-level", type=int, default=2, help="1: kernel groups, 2: + GRU kernels")
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


def key_mode(name):
    from paper_1801_09866_b200 import KEY_MODES
    return KEY_MODES[name]


def math_id(name):
    import paper_1801_09866_b200 as R
    return {"bf16": R.MATH_BF16, "tf32": R.MATH_TF32, "fp32": R.MATH_FP32, "tf32x3": R.MATH_TF32X3,
            "bf16x3": R.MATH_BF16X3}[name]


def dtype_of(name):
    return {"bf16": "bf16", "tf32": "tf32", "fp32": "f32", "tf32x3": "f32 (3xTF32)",
            "bf16x3": "f32 (bf16x3 split)"}[name]


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


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ----------------------------------------------------------------------------- workloads
def stream_starts(total_streams: int, lead: int) -> np.ndarray:
    """Join frame of every stream: evenly spread over [0, lead] so that, once
    all have joined, the streams are at every point of their utterances."""
    return (np.arange(total_streams, dtype=np.int64) * lead) // max(1, total_streams - 1)


def multi_workload(args, lo: int, hi: int, frames: int, stagger: bool, uniform: bool):
    """Streams [lo, hi) of the job (stream s draws from seed 7 + s)."""
    c = CONFIGS[args.workload]
    V = model_dims(args.workload).V
    wl = generate_workload(hi - lo, frames, c["B_s"], V, seed=7 + lo, zipf_s=0.0 if uniform else 1.0)
    if stagger:
        tail = args.warmup + 2 * args.steps
        starts = stream_starts(args.total_streams, max(0, frames - tail - 1))[lo:hi]
        wl = wl.staggered(starts)
    return wl


# ----------------------------------------------------------------------------- oracle timing
def time_oracle(dims, model, wl, mode, k, cache, budget_s, max_steps=None, cell=0, threads=None, start=0):
    """The CPU oracle as it stands (scores / GRUs of a frame on `threads` host
    threads, decisions sequential), on a bounded prefix of the workload's
    first stream; frames before `start` run untimed (they build the caches
    and histories the timed frames depend on).  Returns (queries, seconds,
    frames, per-frame seconds, threads)."""
    import oracle as O
    th = O.threads(threads or host_cores())
    one = wl.select_sessions(0, 1)
    cfg = O.make_config(dims.V, dims.E, dims.H, dims.maxent_log2, dims.N, mode, k,
                        1 if cache else 0, 1,
                        one.max_histories_hint() if cache else one.n_total + 2, cell=cell)
    orc = O.Oracle(cfg, model)
    child = np.zeros(one.n_total, np.uint32)
    done_q, t_total, f = 0, 0.0, 0
    per_step = []
    while f < one.frames and t_total < budget_s and (max_steps is None or f < start + max_steps):
        sl = one.frame_slice(f)
        if sl.stop > sl.start:
            par = O.resolve_parents(one.parent_ref[sl], child)
            t0 = time.perf_counter()
            _, ch, _ = orc.query_frame(one.session[sl], par, one.word[sl])
            dt = time.perf_counter() - t0
            child[sl] = ch
            if f >= start:
                done_q += len(par)
                t_total += dt
                per_step.append((dt, len(par)))
        f += 1
    return done_q, t_total, f, per_step, th


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    c = CONFIGS[args.workload]
    dims = model_dims(args.workload)
    model = generate_model(dims, seed=1234)
    mode, k = key_mode(args.key)
    steps = args.warmup + args.steps
    # each step = one frame of one utterance stream (a bounded sample of the
    # workload): stream 0 of the bench's stream set (seed 7), mid-utterance
    # frames start.. (the frames before run untimed to build the caches)
    start = UTT_FRAMES // 2 if c["frames"] >= UTT_FRAMES else 0
    wl = generate_workload(1, max(UTT_FRAMES, start + steps), c["B_s"], dims.V, seed=7)
    q, secs, frames, per, th = time_oracle(dims, model, wl, mode, k, not args.no_cache, 1e30, max_steps=steps,
                                           cell={"gru": 0, "lbr": 1, "rnn": 2}[args.cell], start=start)
    timed = per[args.warmup:]
    tq = sum(n for _, n in timed)
    ts = sum(dt for dt, _ in timed)
    value = tq / ts
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * ts / len(timed), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "key": args.key,
                   "sample": f"1 stream x {c['B_s']} queries per step (timed frames {start + args.warmup}.."
                             f"{start + steps - 1} of utterance 0; frames 0..{start + args.warmup - 1} untimed)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": th, "kind": "oracle",
                         "sample": f"{len(timed)} frames x {c['B_s']} queries, stream 0",
                         "cpu": cpu_model(), "host_cores": host_cores()},
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


def burst_clocks(clk) -> bool:
    """The timed region ran at (near) the maximum SM clock with no power cap:
    the burst peaks apply (the measured sustained peaks are for seconds-long
    power-capped runs)."""
    if not clk.get("sm_mhz") or not clk.get("sm_max_mhz"):
        # no clock sample landed in a few-ms region: the burst peak (the larger,
        # i.e. the conservative denominator for a short timed region)
        return True
    return clk["sm_mhz"] >= 0.95 * clk["sm_max_mhz"] and "sw_power_cap" not in clk.get("reasons", [])


def measure_tf32_peak(dev):
    """cuBLAS TF32 dense throughput on this GPU (fp32 8192^3 matmul with TF32
    allowed, 2N^3 flop): best of 10 short runs (burst) -- MEASURED_PEAKS.json
    holds no TF32 figure."""
    import torch
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device=dev)
        b = torch.randn(n, n, device=dev)
        for _ in range(3):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old


def gru_peak(math, clk, peaks, tf32_peak, x3_products=3):
    """(peak, unit, bound, source) for the dominant kernel of `math`; 3xTF32:
    the useful-flop peak = TF32 peak / tensor products per useful MAC."""
    burst = burst_clocks(clk)
    which = "burst" if burst else "sustained"
    bf16 = peaks.get("bf16_tflops" if burst else "bf16_tflops_sustained")
    if math in ("bf16", "bf16x3"):
        div = float(x3_products) if math == "bf16x3" else 1.0
        note = (f" / {x3_products:g} (bf16 products per useful multiply-add of the three-part split; "
                "identically-zero products of bf16-exact weights / embeddings are skipped)" if math == "bf16x3" else "")
        if bf16:
            return bf16 / div, "TFLOP/s", "tensor", (f"MEASURED_PEAKS bf16 ({which}: run at max clock, no power cap)"
                if burst else f"MEASURED_PEAKS bf16 ({which}: clocks below max or power-capped)") + note
        return 2250.0 / div, "TFLOP/s", "tensor", "B200_PROFILING nominal dense bf16 (no measured peak)" + note
    if math in ("tf32", "tf32x3"):
        div = float(x3_products) if math == "tf32x3" else 1.0
        note = (f" / {x3_products:g} (TF32 products per useful multiply-add; identically-zero products "
                "of TF32-exact weights / embeddings are skipped)" if math == "tf32x3" else "")
        if tf32_peak:
            return tf32_peak / div, "TFLOP/s", "tensor", f"cuBLAS TF32 8192^3 measured in this run (burst){note}"
        return (bf16 or 2250.0) * 0.5 / div, "TFLOP/s", "tensor", f"bf16 peak x 0.5 (nominal tf32/bf16){note}"
    sm_max = (clk.get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0)
    return 148 * 128 * 2 * sm_max * 1e6 / 1e12, "TFLOP/s", "alu", \
        "derived: 148 SMs x 128 FP32 lanes x 2 flop x sm_max_mhz (B300_MICROARCH unit counts)"


# ----------------------------------------------------------------------------- the step bench
class StepBench:
    """One engine over this rank's streams; prefill, warm-up and two timed
    passes of K frames (value: no library events; roofline: library events on)."""

    def __init__(self, args, dims, model, wl, math, dev, world, local, group=None):
        import torch

        import paper_1801_09866_b200 as R
        self.args, self.dims, self.wl, self.math, self.dev = args, dims, wl, math, dev
        self.world, self.local = world, local
        mode, k = key_mode(args.key)
        self.n = wl.n_per_frame
        cap = wl.max_histories_hint() if not args.no_cache else int(np.max(np.bincount(wl.session))) + 2
        self.eng = R.RNNLM.from_dims(dims, model, key_mode=mode, round_digits=k, math=math_id(math),
                                     cell={"gru": R.CELL_GRU, "lbr": R.CELL_GRU_LBR, "rnn": R.CELL_RNN}[args.cell],
                                     cache_enabled=not args.no_cache, num_sessions=wl.S,
                                     max_queries_per_call=self.n, max_histories_per_session=cap, device=local,
                                     max_queries_per_session_call=CONFIGS[args.workload]["B_s"])
        self.d_sess = torch.as_tensor(wl.session.view(np.int32), device=dev)
        self.d_word = torch.as_tensor(wl.word.view(np.int32), device=dev)
        self.d_ref = torch.as_tensor(wl.parent_ref, device=dev)
        self.d_child = torch.zeros(wl.n_total, dtype=torch.int32, device=dev)
        self.d_score = torch.zeros(wl.n_total, dtype=torch.float32, device=dev)
        self.d_par = torch.zeros(self.n, dtype=torch.int32, device=dev)
        self.flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)        # > 126 MB L2
        self.side = torch.cuda.Stream(device=dev)
        self.gathered = torch.empty((world * self.n, 2), dtype=torch.int32, device=dev) if world > 1 else None
        self.R = R
        tail = args.warmup + 2 * args.steps
        self.t0 = wl.frames - tail            # first warm-up frame

    def call(self, t):
        sl = self.wl.frame_slice(t)
        if sl.stop == sl.start:
            return sl
        k = sl.stop - sl.start
        self.R.resolve_parents(self.d_ref[sl], self.d_child, self.d_par[:k])
        self.eng.query_batch(self.d_sess[sl], self.d_par[:k], self.d_word[sl], score=self.d_score[sl],
                             child=self.d_child[sl], want_outcome=False)
        return sl

    def gather(self, sl):
        from paper_1801_09866_b200.parallel import all_gather_results
        all_gather_results(self.d_score[sl], self.d_child[sl], out=self.gathered)

    def prefill(self):
        import torch
        for t in range(self.t0 + self.args.warmup):
            self.call(t)
        torch.cuda.synchronize()

    def timed_pass(self, t_lo, t_hi, level, trace=None):
        """Frames [t_lo, t_hi): one event pair per step; the L2 flush is between
        pairs.  With N > 1 the all-gather of step i's results runs on a side
        stream during step i + 1 and every step's end event waits for it (the
        last gather is timed on its own), so all K gathers complete inside the
        timed region.  Returns (ms, library timing, stat deltas, launches, clocks)."""
        import torch
        import torch.distributed as dist
        eng, world = self.eng, self.world
        st0 = eng.cache_stats()
        eng.set_timing(level)
        eng.get_timing(reset=True)
        l0 = eng.launch_count()
        clocks = ClockSampler(self.local)
        time.sleep(0.3)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        main = torch.cuda.current_stream()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(t_hi - t_lo + 1)]
        prof = None
        if trace:
            from torch.profiler import ProfilerActivity, profile
            prof = profile(activities=[ProfilerActivity.CUDA])
            prof.__enter__()
        prev = None
        for i, t in enumerate(range(t_lo, t_hi)):
            self.flush.zero_()
            evs[i][0].record()
            if world > 1 and prev is not None:
                self.side.wait_event(evs[i][0])
                with torch.cuda.stream(self.side):
                    self.gather(prev)
            prev = self.call(t)
            if world > 1:
                main.wait_stream(self.side)
            evs[i][1].record()
        if world > 1:                                   # the last step's gather
            evs[-1][0].record()
            self.side.wait_event(evs[-1][0])
            with torch.cuda.stream(self.side):
                self.gather(prev)
            main.wait_stream(self.side)
            evs[-1][1].record()
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
        n_ev = len(evs) if world > 1 else len(evs) - 1
        total_ms = float(sum(a.elapsed_time(b) for a, b in evs[:n_ev]))
        if world > 1:
            tt = torch.tensor([total_ms], dtype=torch.float64, device=self.dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            total_ms = float(tt[0])
        d = {kk: st1[kk] - st0[kk] for kk in ("total_queries", "query_hits", "hidden_lookups",
                                              "hidden_hits", "gru_computations")}
        return total_ms, timing, d, launches, clk

    def run(self, trace=None):
        a = self.args
        self.prefill()
        tA = self.t0 + a.warmup
        tB = tA + a.steps
        ms_A, _, st_A, launches, clk = self.timed_pass(tA, tB, 0, trace)
        ms_B, timing, st_B, _, clk_B = self.timed_pass(tB, tB + a.steps, max(2, a.timing_level))
        return dict(ms=ms_A, stats=st_A, launches=launches, clocks=clk, ms_B=ms_B, timing=timing,
                    stats_B=st_B, clocks_B=clk_B, frames=(tA, tB, tB + a.steps))


def step_summary(args, bench, res, world, peaks, tf32_peak):
    """value, roofline and hit rates of one StepBench.run()."""
    import paper_1801_09866_b200 as R
    dims, math = bench.dims, bench.math
    steps = args.steps
    q_rank = res["stats"]["total_queries"]
    value = q_rank * world / (res["ms"] / 1e3)         # every rank has the same query count per frame
    timing, rows = res["timing"], res["stats_B"]["gru_computations"]
    gates = 1 if args.cell == "rnn" else 3
    flops = 2.0 * gates * dims.H * (dims.E + dims.H) * rows      # [Q, E+H] x [E+H, gates*H]
    tc = math != "fp32"
    gemv = bench.n <= 512
    k_ms = (timing["ms_gru_phase1"] + timing["ms_gru_phase2"]) if (tc and not gemv) else timing["ms_gru"]
    # the roofline pass's clock samples, else the value pass's (same run, same frames' length)
    clk_p = res["clocks_B"] if (res["clocks_B"] or {}).get("sm_mhz") else res["clocks"]
    peak, unit, bound, src = gru_peak(math, clk_p, peaks, tf32_peak, bench.eng.tf32x3_products() or 3)
    achieved = flops / (k_ms / 1e3) / 1e12 if k_ms > 0 else 0.0
    pair = (math in ("bf16", "bf16x3") and args.cell == "gru" and dims.H % 256 == 0
            and os.environ.get("RNNLM_TC_PAIR", "1") != "0")
    kname = ("k_gru_tc2 (fused tcgen05 GRU, both phases, CTA pair)" if pair else
             "k_gru_tc (fused tcgen05 GRU, both phases)") if tc else "k_gru1_f32 + k_gru2_f32 (FP32 SIMT tiles)"
    return {
        "value": value, "ms_per_step": res["ms"] / steps, "dtype": dtype_of(math),
        "roofline": {"kernel": kname, "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
                     "frac": achieved / peak if peak else None, "traffic": None,
                     "traffic_ncu": (f"profiles/ncu_r2_gru_{math}.md (dram bytes per launch, ncu --set full)"
                                     if math in ("bf16", "bf16x3") else "profiles/ncu_r2_start_tf32x3.md"),
                     "peak_source": src,
                     "algorithmic": f"{2 * gates}*H*(E+H) flop per GRU row x {rows} rows over {steps} steps",
                     "kernel_ms_per_step": k_ms / steps,
                     "gather_plus_kernel_ms_per_step": timing["ms_gru"] / steps,
                     "share_of_step": (k_ms / res["ms_B"]) if res["ms_B"] else None,
                     "clocks_of_this_pass": res["clocks_B"]},
        "kernel_ms_per_step": {kk: timing[kk] / steps for kk in
                               ("ms_cache", "ms_score", "ms_gru", "ms_encode", "ms_final",
                                "ms_gru_gather", "ms_gru_phase1", "ms_gru_phase2")},
        "hit_rates": {"query_cache": res["stats"]["query_hits"] / max(1, res["stats"]["total_queries"]),
                      "hidden_cache": res["stats"]["hidden_hits"] / max(1, res["stats"]["hidden_lookups"]),
                      "hidden_hits_per_step": res["stats"]["hidden_hits"] / steps,
                      "gru_rows_per_step": res["stats"]["gru_computations"] / steps},
        "gpu_launches": int(res["launches"]),
        "clocks": res["clocks"],
    }


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1801_09866_b200.parallel import session_range

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
    S_job = args.sessions or c["S"]
    if args.scaling == "strong":
        if S_job % world:
            raise SystemExit("strong scaling needs the streams divisible by the world size")
        lo, hi = session_range(S_job, world, rank)
        args.total_streams = S_job
    else:
        lo, hi = rank * S_job, (rank + 1) * S_job
        args.total_streams = S_job * world
    tail = args.warmup + 2 * args.steps
    frames = max(UTT_FRAMES, tail + 8)
    peaks = load_peaks()
    tf32_peak = measure_tf32_peak(dev) if ("tf32" in args.math or "tf32" in args.also) else None
    model = generate_model(dims, seed=1234)
    wl = multi_workload(args, lo, hi, frames, not args.no_stagger, args.uniform_words)

    bench = StepBench(args, dims, model, wl, args.math, dev, world, local)
    res = bench.run(args.trace)
    head = step_summary(args, bench, res, world, peaks, tf32_peak)
    tA, tB, tC = res["frames"]
    line = {
        "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": head["dtype"], "data": "synthetic",
        "config": {"workload": args.workload, "streams_total": args.total_streams, "streams_per_gpu": hi - lo,
                   "queries_per_stream_frame": c["B_s"], "queries_per_step": int(wl.n_per_frame) * world,
                   "V": dims.V, "E": dims.E, "H": dims.H, "maxent": f"2^{dims.maxent_log2} {dims.N}-gram",
                   "key": args.key, "cache": not args.no_cache, "math": args.math, "cell": args.cell,
                   "streams": ("staggered: stream s joins at frame s*%d/%d of a %d-frame run; timed frames see "
                               "every utterance position" % (frames - tail - 1, args.total_streams - 1, frames))
                   if not args.no_stagger else "in step (all join at frame 0)",
                   "l2": "flushed between timed steps (256 MiB write outside the event pair)",
                   "timed_frames": f"value: frames {tA}..{tB - 1}; roofline pass (library kernel events on): "
                                   f"frames {tB}..{tC - 1} ({tA} prefill/warm-up frames untimed)",
                   "parallelism": f"{world} GPU(s), streams sharded ({args.scaling} scaling), weights replicated, "
                                  "NCCL all-gather of (score, child) per step inside the timed region"},
        "roofline": head["roofline"], "kernel_ms_per_step": head["kernel_ms_per_step"],
        "hit_rates": head["hit_rates"], "gpu_launches": head["gpu_launches"], "clocks": head["clocks"],
    }
    if not args.no_e2e:
        line["e2e"] = run_e2e(args, bench, dev, world)
    del bench
    gc.collect()
    torch.cuda.empty_cache()
    if world > 1 and args.scaling == "strong":
        # the weak-scaling companion (BASELINE configs[4] read per GPU): every rank
        # runs its own full 64-stream job, same math, same timing rules
        ts = args.total_streams
        args.total_streams = S_job * world
        wl_w = multi_workload(args, rank * S_job, (rank + 1) * S_job, frames, not args.no_stagger, args.uniform_words)
        bw = StepBench(args, dims, model, wl_w, args.math, dev, world, local)
        rw = bw.run()
        sw = step_summary(args, bw, rw, world, peaks, tf32_peak)
        line["weak_scaling"] = {"value": sw["value"], "unit": UNIT, "ms_per_step": sw["ms_per_step"],
                                "streams_total": S_job * world, "streams_per_gpu": S_job,
                                "queries_per_step": int(wl_w.n_per_frame) * world,
                                "roofline_frac": sw["roofline"]["frac"], "clocks": sw["clocks"]}
        args.total_streams = ts
        del bw, wl_w
        gc.collect()
        torch.cuda.empty_cache()
    for other in [m for m in args.also.split(",") if m and m != "none" and m != args.math]:
        b2 = StepBench(args, dims, model, wl, other, dev, world, local)
        r2 = b2.run()
        line[other] = {k: v for k, v in step_summary(args, b2, r2, world, peaks, tf32_peak).items()}
        del b2
        gc.collect()
        torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        mode, k = key_mode(args.key)
        q, secs, f, _, th = time_oracle(dims, model, wl, mode, k, not args.no_cache, args.cpu_seconds,
                                        cell={"gru": 0, "lbr": 1, "rnn": 2}[args.cell])
        line["cpu_baseline"] = {"value": q / secs, "unit": UNIT, "cores": th, "kind": "oracle",
                                "sample": f"stream 0, its utterance frames 0..{f - 1} ({q} queries, {secs:.1f} s "
                                          f"of oracle time; scores and GRUs of a frame on {th} threads)",
                                "cpu": cpu_model(), "host_cores": host_cores()}
    del wl
    gc.collect()
    if rank == 0 and world == 1 and not args.no_configs:
        line["configs"] = run_configs(args, dev, peaks, tf32_peak)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, bench, dev, world):
    """Host-buffer path through the public API, as a streaming decoder runs
    it: per step ONE H2D copy of the decoder's packed queries (parent
    reference i64 = index of the earlier query whose child is the parent,
    session u32, word u32) from pinned memory, rnnlm_resolve_parents
    (reference -> handle on the device), rnnlm_query_batch, (N > 1) the NCCL
    all-gather of (score, child), ONE D2H copy of the (gathered) results into
    pinned memory, and the host waits for that step's results.  Double
    buffered: step i + 1's H2D (copy stream) overlaps step i's kernels and
    step i's D2H (copy stream) overlaps step i + 1's kernels; the host reads
    step i's results after enqueueing step i + 1 (parents are references
    resolved on the device, so the next frame does not wait for the host).
    The engine restarts its streams (reset) and replays the untimed frames on
    the device first."""
    import torch
    import torch.distributed as dist

    import paper_1801_09866_b200 as R
    from paper_1801_09866_b200.parallel import all_gather_results
    eng, wl, n = bench.eng, bench.wl, bench.n
    eng.reset_session()
    bench.d_child.zero_()
    for t in range(bench.t0):                           # untimed replay up to the warm-up frames
        bench.call(t)
    torch.cuda.synchronize()
    frames = list(range(bench.t0, bench.t0 + args.warmup + args.steps))
    blk = np.empty((len(frames), 4 * n), dtype=np.int32)
    for i, t in enumerate(frames):
        sl = wl.frame_slice(t)
        assert sl.stop - sl.start == n
        blk[i, :2 * n] = np.ascontiguousarray(wl.parent_ref[sl], dtype=np.int64).view(np.int32)
        blk[i, 2 * n:3 * n] = wl.session[sl].view(np.int32)
        blk[i, 3 * n:] = wl.word[sl].view(np.int32)
    h_in_all = torch.from_numpy(blk).pin_memory()
    out_rows = world * n
    h_out = [torch.empty(2 * out_rows, dtype=torch.int32).pin_memory() for _ in range(2)]
    d_in = [torch.empty(4 * n, dtype=torch.int32, device=dev) for _ in range(2)]
    d_par = torch.empty(n, dtype=torch.int32, device=dev)
    d_score = torch.empty(n, dtype=torch.float32, device=dev)
    d_out = [torch.empty((out_rows, 2), dtype=torch.int32, device=dev) for _ in range(2)]
    main = torch.cuda.current_stream()
    h2d, d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ev_in = [torch.cuda.Event() for _ in frames]        # step i's inputs on the device
    ev_used = [torch.cuda.Event() for _ in frames]      # step i's inputs consumed, outputs packed
    ev_out = [torch.cuda.Event() for _ in frames]       # step i's results in host memory

    def upload(i):
        b = i % 2
        if i >= 2:
            h2d.wait_event(ev_used[i - 2])              # the buffer's previous step has consumed it
        with torch.cuda.stream(h2d):
            d_in[b].copy_(h_in_all[i], non_blocking=True)
            ev_in[i].record(h2d)

    def compute(i, t):
        b = i % 2
        sl = wl.frame_slice(t)
        main.wait_event(ev_in[i])
        d_ref, d_sess, d_word = d_in[b][:2 * n].view(torch.int64), d_in[b][2 * n:3 * n], d_in[b][3 * n:]
        R.resolve_parents(d_ref, bench.d_child, d_par)
        eng.query_batch(d_sess, d_par, d_word, score=d_score, child=bench.d_child[sl], want_outcome=False)
        if i >= 2:
            main.wait_event(ev_out[i - 2])              # d_out[b] of step i - 2 has been read back
        if world > 1:
            all_gather_results(d_score, bench.d_child[sl], out=d_out[b])
        else:
            d_out[b][:, 0].copy_(d_score.view(torch.int32))
            d_out[b][:, 1].copy_(bench.d_child[sl])
        ev_used[i].record(main)
        d2h.wait_event(ev_used[i])
        with torch.cuda.stream(d2h):
            h_out[b].copy_(d_out[b].view(-1), non_blocking=True)
            ev_out[i].record(d2h)

    def run(lo, hi):
        upload(lo)
        for i in range(lo, hi):
            if i + 1 < hi:
                upload(i + 1)
            compute(i, frames[i])
            if i > lo:
                ev_out[i - 1].synchronize()             # the host reads step i - 1's results
        ev_out[hi - 1].synchronize()

    run(0, args.warmup)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(args.warmup, len(frames))
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([secs], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        secs = float(tt[0])
    return {"value": n * args.steps * world / secs, "unit": UNIT,
            "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 8 * out_rows,
            "note": "wall clock over the steps: per step H2D (parent reference i64, session u32, word u32) from "
                    "pinned memory, device-side reference -> handle resolution, the step, the all-gather (N > 1), "
                    "D2H of the (score, child) results, the host waiting for them; double-buffered copies on "
                    "copy streams (step i + 1's upload and step i - 1's read-back overlap step i); the same "
                    "frames as the value pass; max over ranks"}


# ----------------------------------------------------------------------------- configs[0]-[3]
def single_stream(name, frames=None, seed=7):
    c = CONFIGS[name]
    d = model_dims(name)
    return d, generate_workload(1, frames or c["frames"], c["B_s"], d.V, seed=seed)


def frame_loop(eng, wl, dev, t_lo, t_hi, use_graph=False, timing=0):
    """Run frames [0, t_hi) of a one-stream workload, time [t_lo, t_hi) as one
    device interval and on the host clock.  Returns (device ms, wall s,
    scores, children, library timing)."""
    import torch

    import paper_1801_09866_b200 as R
    n = wl.n_per_frame
    d_sess = torch.as_tensor(wl.session.view(np.int32), device=dev)
    d_word = torch.as_tensor(wl.word.view(np.int32), device=dev)
    d_ref = torch.as_tensor(wl.parent_ref, device=dev)
    d_child = torch.zeros(wl.n_total, dtype=torch.int32, device=dev)
    d_score = torch.zeros(wl.n_total, dtype=torch.float32, device=dev)
    par = torch.zeros(n, dtype=torch.int32, device=dev)
    if use_graph:
        bs, bw = torch.zeros(n, dtype=torch.int32, device=dev), torch.zeros(n, dtype=torch.int32, device=dev)
        sc, ch = torch.zeros(n, dtype=torch.float32, device=dev), torch.zeros(n, dtype=torch.int32, device=dev)
        g = eng.graph(n, bs, par, bw, sc, ch)

    # Direct calls go through the C ABI with every frame's pointers precomputed:
    # per frame the host pays two ctypes calls, as a C/C++ decoder would, instead
    # of torch slicing + the Python wrappers (~30 us per frame, which made the
    # tiny config host-bound: 32 vs 18 us per frame, profiles/host_rate_r2.jsonl)
    from paper_1801_09866_b200 import _lib
    lib = _lib.load()
    cst = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = lambda x: ctypes.c_void_p(x.data_ptr())
    slices = [wl.frame_slice(t) for t in range(t_hi)]
    pre = [(s_.stop - s_.start, vp(d_ref[s_]), vp(d_sess[s_]), vp(d_word[s_]), vp(d_score[s_]), vp(d_child[s_]))
           for s_ in slices]
    p_par, p_log = vp(par), vp(d_child)

    def frame(t):
        if use_graph:
            sl = slices[t]
            R.resolve_parents(d_ref[sl], d_child, par)
            bs.copy_(d_sess[sl])
            bw.copy_(d_word[sl])
            g.launch()
            d_child[sl].copy_(ch)
            d_score[sl].copy_(sc)
        else:
            nn, pr, ps, pw, psc, pch = pre[t]
            _lib.check(lib.rnnlm_resolve_parents(nn, pr, p_log, p_par, cst), "resolve_parents")
            _lib.check(lib.rnnlm_query_batch(eng._h, nn, ps, p_par, pw, psc, pch, None, cst), "rnnlm_query_batch")

    for t in range(t_lo):
        frame(t)
    torch.cuda.synchronize()
    eng.set_timing(timing)
    eng.get_timing(reset=True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    a.record()
    for t in range(t_lo, t_hi):
        frame(t)
    b.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    tm = eng.get_timing(reset=True)
    eng.set_timing(0)
    return a.elapsed_time(b), wall, d_score.cpu().numpy(), d_child.cpu().numpy(), tm


def run_configs(args, dev, peaks, tf32_peak):
    """BASELINE configs[0]-[3] on one GPU (single utterance stream each):
    per-frame latency and q/s (direct calls and a replayed CUDA graph), the
    small-frame GEMV kernels' achieved bytes/s, bf16 vs fp32-accurate on the
    large model, and the compression sweep."""
    import torch

    import paper_1801_09866_b200 as R
    out = {}
    hbm = peaks.get("hbm_gbs", 6551.0)

    def eng_for(d, m, wl, key, math, path=R.GRU_AUTO, cache=True):
        mode, k = key_mode(key)
        return R.RNNLM.from_dims(d, m, key_mode=mode, round_digits=k, math=math_id(math), cache_enabled=cache,
                                 num_sessions=1, max_queries_per_call=wl.n_per_frame,
                                 max_histories_per_session=wl.max_histories_hint(), gru_path=path)

    # tiny (configs[0]) and moderate (configs[1]): latency-bound single-stream frames
    for name, maths, keys in (("tiny", ("fp32",), ("sign", "round:2")),
                              ("moderate", ("bf16", "bf16x3"), ("off", "sign"))):
        d, wl = single_stream(name)
        m = generate_model(d, seed=1234)
        F = wl.frames
        t_lo = min(40, F // 2)
        res = {}
        for math in maths:
            for key in keys:
                e = eng_for(d, m, wl, key, math)
                ms, wall, _, _, tm = frame_loop(e, wl, dev, t_lo, F, timing=1)
                st = e.cache_stats()
                del e
                e = eng_for(d, m, wl, key, math)
                ms_g, wall_g, _, _, _ = frame_loop(e, wl, dev, t_lo, F, use_graph=True)
                del e
                nq = wl.n_per_frame * (F - t_lo)
                rows = st["gru_computations"] / F
                nonq = st["hidden_lookups"] / F
                # algorithmic bytes of one small frame (SURVEY 8(d) per-query model): the gate
                # weights once (L2-resident), per query 12 B in + 32 B probe + 8 B out, per
                # non-QHIT query its score's row / state / bias / MaxEnt sectors + record,
                # hidden probe and two inserts, per GRU row its x / h reads and new state
                s_w = 2 if math == "bf16" else 4
                wbytes = 3 * d.H * (d.E + d.H) * s_w
                fbytes = (wbytes + wl.n_per_frame * 52 + nonq * (d.H * s_w + 4 * d.H + 32 + 32 * d.N + 128)
                          + rows * (d.E * s_w + 8 * d.H))
                fused_ms = tm["ms_fused"] / max(1, tm["calls"])
                gbs = fbytes / (fused_ms * 1e-3) / 1e9 if fused_ms > 0 else None
                res[f"{math}/{key}"] = {
                    "q_per_s": nq / (ms * 1e-3), "us_per_frame": 1e3 * ms / (F - t_lo),
                    "q_per_s_wall": nq / wall, "us_per_frame_wall": 1e6 * wall / (F - t_lo),
                    "graph": {"q_per_s": nq / (ms_g * 1e-3), "us_per_frame": 1e3 * ms_g / (F - t_lo),
                              "us_per_frame_wall": 1e6 * wall_g / (F - t_lo)},
                    "query_cache_hit": st["query_hits"] / max(1, st["total_queries"]),
                    "hidden_hits": st["hidden_hits"], "gru_rows_per_frame": rows,
                    "fused_kernel": {"kernel": "k_small (whole step, one cooperative launch; GEMV GRU)",
                                     "us_per_frame": 1e3 * fused_ms, "algorithmic_bytes_per_frame": fbytes,
                                     "achieved_gbs": gbs, "hbm_peak_gbs": hbm,
                                     "frac_of_hbm": (gbs / hbm) if gbs else None,
                                     "note": "latency-bound: ~1 MB per frame through a one-CTA cache front "
                                             "(block barriers) and three grid barriers of dependent L2 round "
                                             "trips; bytes/s is far below HBM bandwidth"},
                }
        out[name] = {"streams": 1, "queries_per_frame": wl.n_per_frame, "frames": F,
                     "timed_frames": f"{t_lo}..{F - 1}", "V": d.V, "H": d.H, "results": res}
        del m
        gc.collect()
        torch.cuda.empty_cache()

    # large (configs[2]) and the compression sweep (configs[3]): one stream, 2,048 queries/frame
    d, wl = single_stream("large")
    m = generate_model(d, seed=1234)
    F = wl.frames
    t_lo = F - 60
    res = {}
    for math in ("bf16", "bf16x3", "tf32x3", "fp32"):
        e = eng_for(d, m, wl, "sign", math)
        ms, wall, _, _, tm = frame_loop(e, wl, dev, t_lo, F, timing=0)
        st = e.cache_stats()
        del e
        res[math] = {"q_per_s": wl.n_per_frame * (F - t_lo) / (ms * 1e-3), "us_per_frame": 1e3 * ms / (F - t_lo),
                     "gru_rows_per_frame": st["gru_computations"] / F, "dtype": dtype_of(math)}
    out["large"] = {"streams": 1, "queries_per_frame": wl.n_per_frame, "frames": F, "key": "sign",
                    "timed_frames": f"{t_lo}..{F - 1}", "results": res}
    sweep = {}
    base = None
    for key in ("off", "round:3", "round:2", "round:1", "sign"):
        e = eng_for(d, m, wl, key, args.math)
        ms, wall, sc, ch, _ = frame_loop(e, wl, dev, 0, F)
        st = e.cache_stats()
        del e
        if base is None:
            base = (sc, st["gru_computations"])
        dev_abs = np.abs(sc.astype(np.float64) - base[0].astype(np.float64))
        sweep[key] = {"hidden_hit_rate": st["hidden_hits"] / max(1, st["hidden_lookups"]),
                      "gru_computations": st["gru_computations"],
                      "redundancy_pct_vs_off": 100.0 * (base[1] - st["gru_computations"]) / max(1, base[1]),
                      "score_dev_vs_off_max": float(dev_abs.max()), "score_dev_vs_off_mean": float(dev_abs.mean()),
                      "q_per_s": wl.n_total / (ms * 1e-3)}
    out["sweep"] = {"model": "large", "math": args.math, "streams": 1, "frames": F,
                    "queries": int(wl.n_total), "note": "Table 1 (P:122-143) on the synthetic stream: redundancy "
                    "= (gru(off) - gru(mode)) / gru(off); score deviation against the same engine with lossless "
                    "keys (mode off) over the whole utterance", "results": sweep}
    del m
    gc.collect()
    torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- (f2), (f4)
def run_normalizer(args):
    """throughput of the exact log-normaliser (rnnlm_log_normalizer)
    on the large model (V = 200k, H = 1024, 4-gram MaxEnt 2^27): log Z of
    --histories distinct stored histories per call, device-timed with CUDA
    events; one JSON line.  Roofline of the dominant kernel (k_norm_tc): its
    algorithmic traffic is the MaxEnt gathers, (K - 1) random 4-byte reads =
    32-byte sectors per (history, word) (order 1 is a per-word bias), plus one
    pass over the bf16 output rows per 128-history tile."""
    import torch

    import paper_1801_09866_b200 as R

    d = model_dims("large")
    m = generate_model(d, seed=1234)
    n = args.histories
    # distinct histories: one utterance, cache off, 2 frames of n/2 queries
    # each -> every query makes a new history (depth 1 and 2)
    wl = generate_workload(1, 2, n // 2, d.V, seed=5)
    math = math_id(args.math)
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
    hbm = load_peaks().get("hbm_gbs", 6551.0)
    gbs = (sectors + theta) / (ms * 1e-3) / 1e9
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
                     "traffic": None, "contraction_tflops": flops / (ms * 1e-3) / 1e12},
    }
    print(json.dumps(line), flush=True)


def run_offline(args):
    """whole utterances known in advance (2-pass lattice
    rescoring) scheduled level by level (paper_1801_09866_b200.offline)
    instead of one call per frame.  Both schedules run the same synthetic
    utterances on the same engine settings (the tile GRU kernels); each is
    device-timed with CUDA events around the whole stream (after one untimed
    warm-up pass).  With lossy keys the level order changes which query is a
    key's first occupant, so results are bitwise equal to the online schedule
    only at key off (reported)."""
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
    math = math_id(args.math)
    dev = torch.device("cuda", 0)
    Bmax = 32768
    cap = wl.max_histories_hint()

    def engine(B):
        return R.RNNLM.from_dims(dims, model, key_mode=mode, round_digits=k, math=math, num_sessions=S,
                                 max_queries_per_call=B, max_histories_per_session=cap, gru_path=R.GRU_TILES)

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
    same = bool(torch.equal(d_score, runner.score))
    nb = len(runner.batches)
    line = {
        "metric": "RNNLM queries/sec (offline level-batched rescoring of whole utterances)",
        "value": wl.n_total / (ms_off * 1e-3), "unit": "queries/s", "n_gpus": 1, "steps": 1, "warmup": 1,
        "ms_per_step": ms_off, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": dtype_of(args.math), "data": "synthetic",
        "config": {"workload": args.workload, "sessions": S, "frames": frames, "queries": int(wl.n_total),
                   "key": args.key, "math": args.math, "offline_calls": nb, "online_calls": frames,
                   "mean_queries_per_offline_call": wl.n_total / max(1, nb),
                   "step": "one pass over the whole query stream"},
        "online": {"value": wl.n_total / (ms_on * 1e-3), "ms": ms_on},
        "speedup_vs_online": ms_on / ms_off,
        "scores_bitwise_equal_online": same,
        "note": None if mode == R.KEY_OFF else "lossy keys: the level order changes first occupants, so results "
                                               "may differ from the online schedule (DESIGN.md reading 29)",
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
