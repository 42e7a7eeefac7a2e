"""Device timeline of config-4 RK4 steps (CUPTI through torch.profiler): every
kernel of the library with its real start/end on the GPU (concurrent streams
included, nothing serialised), then per-kernel busy time, the union of busy
time, and the idle gaps between kernels — the exposed latency ncu's
serialised launch list cannot show.

    python tools/timeline.py [steps] [--config c4|c4eval|c3|c5|...] [--json out]
"""
import argparse
import collections
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("steps", type=int, nargs="?", default=2)
ap.add_argument("--config", default="c4")
ap.add_argument("--json", default=None)
ap.add_argument("--gaps", type=int, default=25, help="largest idle gaps listed")
args = ap.parse_args()

import paper_2401_07361_b200 as ss  # noqa: E402

bench.use_config(args.config)
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
xyz, zeta, area = bench.fixture_product()
st = bench.Stepper(ss, torch, dev, xyz, zeta, area, 1, 0)
for _ in range(3):
    st.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(args.steps):
        st.step()
    torch.cuda.synchronize()
def short_name(n):
    n = n.replace("(anonymous namespace)::", "").replace("void ", "").replace("CUB_200802_SM_1000::", "")
    depth, out = 0, []
    for ch in n:  # drop the argument list, keep template arguments
        if ch == "(" and depth == 0:
            break
        depth += ch == "<"
        depth -= ch == ">"
        out.append(ch)
    return "".join(out)[:80]


ev = []
trace_path = "/tmp/ssum_timeline_trace.json"
prof.export_chrome_trace(trace_path)
for e in json.load(open(trace_path))["traceEvents"]:
    if e.get("ph") != "X" or e.get("cat") not in ("kernel", "gpu_memcpy", "gpu_memset"):
        continue
    t0 = float(e["ts"])
    t1 = t0 + float(e["dur"])
    stream = e.get("args", {}).get("stream", -1)
    ev.append((t0, t1, short_name(e["name"]), stream))
ev.sort()
if not ev:
    sys.exit("no device events")
t_begin, t_end = ev[0][0], max(e[1] for e in ev)
span = t_end - t_begin
busy = collections.defaultdict(float)
cnt = collections.Counter()
for t0, t1, n, _ in ev:
    short = n
    busy[short] += t1 - t0
    cnt[short] += 1
# union of busy intervals and the gaps between them
gaps = []
cur0, cur1 = ev[0][0], ev[0][1]
union = 0.0
prev_name = ev[0][2]
for t0, t1, n, _ in ev[1:]:
    if t0 > cur1:
        union += cur1 - cur0
        gaps.append((t0 - cur1, prev_name, n, cur1 - t_begin))
        cur0, cur1 = t0, t1
    else:
        cur1 = max(cur1, t1)
    if t1 >= cur1:
        prev_name = n
union += cur1 - cur0
per = args.steps
out = {
    "config": args.config, "steps": args.steps,
    "span_ms_per_step": span / per / 1e3, "busy_union_ms_per_step": union / per / 1e3,
    "idle_ms_per_step": (span - union) / per / 1e3, "n_gaps": len(gaps),
    # host round trips (read-backs) leave long gaps; back-to-back dependent
    # launches short ones
    "idle_by_gap_size_ms_per_step": {
        lbl: sum(g[0] for g in gaps if lo <= g[0] < hi) / per / 1e3
        for lbl, lo, hi in (("<5us", 0, 5), ("5-10us", 5, 10), ("10-30us", 10, 30), (">=30us", 30, 1e18))},
    "kernels": sorted(({"kernel": k, "ms_per_step": v / per / 1e3, "launches_per_step": cnt[k] / per}
                       for k, v in busy.items()), key=lambda d: -d["ms_per_step"]),
    "largest_gaps_us": [{"us": g, "after": a, "before": b, "at_ms": t / 1e3}
                        for g, a, b, t in sorted(gaps, reverse=True)[:args.gaps]],
}
print(f"span {out['span_ms_per_step']:.3f} ms/step, busy union {out['busy_union_ms_per_step']:.3f}, "
      f"idle {out['idle_ms_per_step']:.3f} in {len(gaps)} gaps")
print("idle by gap size (ms/step):", {k: round(v, 3) for k, v in out["idle_by_gap_size_ms_per_step"].items()})
for d in out["kernels"][:40]:
    print(f"  {d['ms_per_step']:8.3f} ms  x{d['launches_per_step']:5.1f}  {d['kernel']}")
print("largest gaps:")
for d in out["largest_gaps_us"]:
    print(f"  {d['us']:8.1f} us at {d['at_ms']:8.3f} ms  {d['after']} -> {d['before']}")
# the ordered kernel sequence of the last step (start offset, duration, name)
last = [e for e in ev if e[0] >= t_begin + span * (per - 1) / per]
out["last_step_sequence"] = [{"t_us": round(t0 - last[0][0], 1), "us": round(t1 - t0, 1), "stream": sm, "k": n}
                             for t0, t1, n, sm in last]
if args.json:
    with open(args.json, "w") as f:
        json.dump(out, f, indent=1)
