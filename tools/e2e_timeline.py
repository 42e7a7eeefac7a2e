"""Device timeline of the end-to-end RK4 call (ss.rk4 -> ssum_rk4 on pinned
host arrays, one step per call; CUPTI through torch.profiler): where the
copies sit relative to the kernels, and what is exposed beyond the
device-resident step.

    python tools/e2e_timeline.py [calls]
"""
import json
import os
import sys
import time

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import bench  # noqa: E402
import paper_2401_07361_b200 as ss  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 2
bench.use_config("c4")
xyz, zeta, area = bench.fixture_product()
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
hx, hz, ha = pin(xyz), pin(zeta), pin(area)
cfg = ss.TraversalConfig(**bench.C["cfg"])
tree = ss.FaceTree(0)
rk = bench.C["rk4"]
for _ in range(2):
    ss.rk4(hx, hz, ha, cfg, dt=rk["dt"], steps=1, omega=bench.OMEGA, tree=tree, inplace=True)
walls = []
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(calls):
        t0 = time.perf_counter()
        ss.rk4(hx, hz, ha, cfg, dt=rk["dt"], steps=1, omega=bench.OMEGA, tree=tree, inplace=True)
        walls.append((time.perf_counter() - t0) * 1e3)
    torch.cuda.synchronize()
path = "/tmp/ssum_e2e_trace.json"
prof.export_chrome_trace(path)
ev = []
for e in json.load(open(path))["traceEvents"]:
    if e.get("ph") != "X" or e.get("cat") not in ("kernel", "gpu_memcpy", "gpu_memset"):
        continue
    ev.append((e["ts"], e["dur"], e["args"].get("stream", -1), e["name"][:60], e["args"].get("bytes", 0)))
ev.sort()
print("wall ms per call (under the profiler):", ["%.2f" % w for w in walls])
# split into calls at the big H2D copies' first event after a long pause
t0 = ev[0][0]
big = [e for e in ev if e[3].startswith("Memcpy") and e[1] > 50]
print("large copies (start ms, dur ms, stream, name):")
for e in big:
    print("  %9.3f %7.3f  s%-3d %s" % ((e[0] - t0) / 1e3, e[1] / 1e3, e[2], e[3]))
walks = [e for e in ev if "k_walk" in e[3]]
fin = [e for e in ev if "k_rk4_final" in e[3]]
tiles = [e for e in ev if "k_tiles" in e[3]]
print("k_walk starts (ms):", ["%.3f" % ((e[0] - t0) / 1e3) for e in walks])
print("k_tiles ends (ms):", ["%.3f" % ((e[0] + e[1] - t0) / 1e3) for e in tiles])
print("k_rk4_final (ms):", ["%.3f+%.3f" % ((e[0] - t0) / 1e3, e[1] / 1e3) for e in fin])
print("last event end (ms): %.3f" % ((ev[-1][0] + ev[-1][1] - t0) / 1e3))
