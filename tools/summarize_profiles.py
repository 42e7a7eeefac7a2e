"""Summaries for profiles/README.md from ncu output.

    python tools/summarize_profiles.py launches <launches.csv>
        launch table of the last treecode call on device-resident inputs in a
        `ncu --metrics gpu__time_duration.sum` launch list.
    python tools/summarize_profiles.py full <report.ncu-rep> [out.json]
        key metrics of every kernel in an `ncu --set full` capture.
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr, data = rows[0], rows[1:]
    ik, iname, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    unit = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    seq = []
    for d in data:
        if d[iname] != "gpu__time_duration.sum":
            continue
        v = float(d[iv].replace(",", ""))
        u = d[unit] if unit is not None else "ns"
        ms = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(u, 1e-6)
        name = d[ik].split("(")[0].replace("void ", "").replace("ssum::<unnamed>::", "").replace("<unnamed>::", "")
        seq.append((name, ms))
    # one step = one treecode call, which starts with the binning (k_walk on
    # a reused tree, k_bin_roots on a new one); report the last call on
    # device-resident inputs (one k_finish: host-pointer calls finish in pieces)
    starts = [i for i, (n, _) in enumerate(seq) if n in ("k_walk", "k_bin_roots")] + [len(seq)]
    calls = [seq[a:b] for a, b in zip(starts[:-1], starts[1:])]
    device_calls = [c for c in calls if sum(1 for n, _ in c if n.startswith("k_finish")) == 1]
    # the capture's last calls may be a list-builder trial (k_sub_lists timed
    # against k_bfs every 512 calls): report the last call on the chosen
    # builder, i.e. the kind the majority of the device calls used
    pool = device_calls or calls
    sub = [c for c in pool if any(n == "k_sub_lists" for n, _ in c)]
    glob = [c for c in pool if not any(n == "k_sub_lists" for n, _ in c)]
    step = (glob if len(glob) >= len(sub) else sub)[-1]
    ends = calls
    agg = OrderedDict()
    for name, ms in step:
        c, t = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, t + ms)
    tot = sum(t for c, t in agg.values())
    print(f"{len(ends)} treecode calls in the capture; the last on device-resident inputs: {len(step)} launches, "
          f"{tot:.3f} ms serialised cold-cache device time\n")
    print("| kernel | ms | launches | share |\n|---|---|---|---|")
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{name[:60]}` | {t:.3f} | {c} | {100 * t / tot:.1f}% |")


FULL_KEYS = OrderedDict(
    [
        ("duration_ms", "gpu__time_duration.sum"),
        ("fp64_pipe_active_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("xu_pipe_pct", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
        ("lsu_wavefronts_pct", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        ("registers", "launch__registers_per_thread"),
        ("dram_read_bytes", "dram__bytes_read.sum"),
        ("dram_write_bytes", "dram__bytes_write.sum"),
    ]
)


def full(rep, out=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        rec = OrderedDict(kernel=d[hdr.index("Kernel Name")].split("(")[0].replace("void ", ""))
        for k, m in FULL_KEYS.items():
            if m not in hdr:
                continue
            v = float(d[hdr.index(m)].replace(",", "") or 0)
            u = units[hdr.index(m)]
            if k == "duration_ms":
                v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(u, 1.0)
            if k.startswith("dram") and u in ("Mbyte", "MB"):
                v *= 1e6
            if k.startswith("dram") and u in ("Kbyte", "KB"):
                v *= 1e3
            if k.startswith("dram") and u in ("Gbyte", "GB"):
                v *= 1e9
            rec[k] = v
        stalls = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[i].replace(",", "") or 0))
                  for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
        tot = sum(v for _, v in stalls) or 1.0
        rec["top_stalls_pct"] = OrderedDict((h, round(100 * v / tot, 1)) for h, v in sorted(stalls, key=lambda x: -x[1])[:5])
        res.append(rec)
    print("| kernel | ms | FP64 pipe | issue | warps | XU | LSU wavefronts | regs | DRAM MB |\n|---|---|---|---|---|---|---|---|---|")
    for r in res:
        print(f"| `{r['kernel'][:40]}` | {r['duration_ms']:.3f} | {r['fp64_pipe_active_pct']:.1f}% | "
              f"{r['issue_active_pct']:.1f}% | {r['warps_active_pct']:.1f}% | {r.get('xu_pipe_pct', 0):.1f}% | "
              f"{r.get('lsu_wavefronts_pct', 0):.1f}% | {r['registers']:.0f} | "
              f"{(r['dram_read_bytes'] + r['dram_write_bytes']) / 1e6:.0f} |")
    if out:
        json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
