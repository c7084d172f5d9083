"""Summarise a chrome trace written by `bench.py --trace`: per timed step, each
GPU kernel's start / end relative to the step's first kernel (us) and stream."""
import json
import sys

tr = json.load(open(sys.argv[1]))
ev = [e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
ev.sort(key=lambda e: e["ts"])
steps, cur = [], []
for e in ev:
    n = e["name"]
    if "k_resolve_parents" in n and cur:
        steps.append(cur)
        cur = []
    cur.append(e)
if cur:
    steps.append(cur)
want = int(sys.argv[2]) if len(sys.argv) > 2 else len(steps) // 2
for si in ([want] if want >= 0 else range(len(steps))):
    st = steps[si]
    t0 = st[0]["ts"]
    print(f"--- step {si}: span {max(e['ts'] + e['dur'] for e in st if 'FillFunctor' not in e['name']) - t0:.1f} us")
    for e in st:
        name = e["name"].split("(")[0].replace("void ", "")[:40]
        print(f"{name:40s} stream {e['args'].get('stream', '?'):>4} start {e['ts'] - t0:8.1f} end {e['ts'] + e['dur'] - t0:8.1f} dur {e['dur']:7.1f}")
