"""Warp-stall samples and executed instructions per innermost loop of one
kernel in an `ncu --set full --import-source on` report (the source page).

    python tools/source_loops.py <report.ncu-rep> <kernel template args, e.g. "(int)0, (int)0"> [launch-skip]
"""
import csv
import io
import re
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:k_tiles|k_finish|k_bfs",
                      "--launch-skip", skip, "--launch-count", "2"], capture_output=True, text=True).stdout
blocks, cur = [], None
for r in csv.reader(io.StringIO(raw)):
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
b = [x for x in blocks if pat in x["name"]][0]
hdr, data = b["rows"][0], b["rows"][1:]
ia, isrc, isamp, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("# Samples"), hdr.index("Instructions Executed")
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
ins = []
for r in data:
    try:
        ins.append((int(r[ia], 16), r[isrc], int(r[isamp] or 0), int(r[iex] or 0),
                    {hdr[i]: int(r[i] or 0) for i in st}))
    except ValueError:
        pass
tot_s, tot_i = sum(x[2] for x in ins), sum(x[3] for x in ins)
print(b["name"][:70])
print("instructions", len(ins), "samples", tot_s, "warp instructions executed", tot_i)
idx = {a: i for i, (a, *_rest) in enumerate(ins)}
loops = []
for a, s, *_ in ins:
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w*,\s*)?0x([0-9a-f]+)", s)
    if m:
        t = int(m.group(1), 16)
        if t < a and t in idx:
            loops.append((t, a))
inner = [l for l in loops if not any(o != l and o[0] >= l[0] and o[1] <= l[1] for o in loops)]
covered = set()
base = ins[0][0]
isf64 = lambda s: re.match(r"\s*(@!?U?P\d+\s+)?D(FMA|MUL|ADD|SETP)", s) is not None  # noqa: E731
for t, e in sorted(inner):
    seg = ins[idx[t]:idx[e] + 1]
    covered.update(range(idx[t], idx[e] + 1))
    s, ex = sum(x[2] for x in seg), sum(x[3] for x in seg)
    if 100 * s / tot_s < 0.8:
        continue
    f64 = sum(x[3] for x in seg if isf64(x[1]))
    agg = {}
    for x in seg:
        for k, v in x[4].items():
            agg[k] = agg.get(k, 0) + v
    top = sorted(agg.items(), key=lambda kv: -kv[1])[:5]
    print("loop %#07x-%#07x: %4d instr  samples %5.1f%%  executed %5.1f%%  fp64 %3.0f%% of executed  %s" % (
        t - base, e - base, len(seg), 100 * s / tot_s, 100 * ex / tot_i, 100 * f64 / max(ex, 1),
        [(k[6:], round(100 * v / tot_s, 1)) for k, v in top]))
rest = [x for i, x in enumerate(ins) if i not in covered]
print("outside innermost loops: samples %.1f%%  executed %.1f%%" % (
    100 * sum(x[2] for x in rest) / tot_s, 100 * sum(x[3] for x in rest) / tot_i))
for x in sorted(rest, key=lambda x: -x[2])[:14]:
    top = sorted(x[4].items(), key=lambda kv: -kv[1])[:2]
    print("  %#07x %5.2f%%  %-58s %s" % (x[0] - base, 100 * x[2] / tot_s, x[1][:58], [(k[6:], v) for k, v in top]))
# executed share of the code outside the innermost loops, in address order (runs of ~64 instructions)
print("outside-loop code by address (executed %, samples %):")
run = []
def flush():
    if not run:
        return
    ex, s = sum(x[3] for x in run), sum(x[2] for x in run)
    if 100 * ex / tot_i >= 0.3 or 100 * s / tot_s >= 0.3:
        per = ex / len(run) / max(ins[0][3], 1)
        print("  %#07x-%#07x  %4d instr  executed %5.2f%%  samples %5.2f%%  (avg executions per instr / kernel-entry executions: %.1f)" % (
            run[0][0] - base, run[-1][0] - base, len(run), 100 * ex / tot_i, 100 * s / tot_s, per))
for i, x in enumerate(ins):
    if i in covered:
        flush()
        run = []
        continue
    run.append(x)
    if len(run) >= 64:
        flush()
        run = []
flush()
