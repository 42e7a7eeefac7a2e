"""The DESIGN.md §6 table rows from a directory of bench lines
(bench_<config>.json as tools/profile_round2c.sh writes them).

    python tools/bench_table.py gpurun_out/prof2e
"""
import json
import os
import sys

d = sys.argv[1]


def line(name):
    p = os.path.join(d, f"bench_{name}.json")
    if not os.path.exists(p):
        p = os.path.join(d, f"r2d_bench_{name}.json")
    for l in open(p):
        if l.startswith("{"):
            return json.loads(l)


ref = line("reference_arm")
print("| config | N | ms/step | evals/s | e2e evals/s | roofline | reference CPU evals/s (16 thr) | parity vs reference | E mine (reference E) |")
print("|---|---|---|---|---|---|---|---|---|")
for name in ("config4", "c4eval", "c1", "c2", "c2pc", "c2log", "c3", "c5"):
    b = line(name)
    n = b["config"]["n"]
    cpu = b.get("cpu_baseline") or {}
    cpus = "%.3e" % cpu["value"] if cpu.get("value") else "-"
    if name == "config4":
        cpus = "%.3e (reference arm)" % ref["value"]
        par = "%.1e after 1 step" % b["parity_rel_l2_vs_reference"]
        ms = "%.2f, %.2f/eval" % (b["ms_per_step"], b["ms_per_step"] / 4)
    else:
        par = "%.1e" % b["parity_rel_l2_vs_reference"]
        ms = "%.2f" % b["ms_per_step"]
        if cpu.get("kind") == "port":
            cpus += " (port, %d thr)" % cpu.get("cores", 1)
    e = b.get("error_vs_direct") or {}
    es = "%.3e" % e["value"] if e.get("value") else "-"
    if e.get("reference_same_targets"):
        es += " (%.3e)" % e["reference_same_targets"]
    print("| %s | %s | %s | %.3e | %.3e | %.3f | %s | %s | %s |" % (
        "c4 (RK4, headline)" if name == "config4" else name, f"{n:,}", ms, b["value"], b["e2e"]["value"],
        b["roofline"]["frac"], cpus, par, es))
b = line("config4")
print("\nC4 phases per evaluation:", {k: round(v, 3) for k, v in b["phase_ms_per_evaluation"].items()})
print("C4 e2e ms/step: %.2f  cold_ms: %.2f  clocks: %s" % (b["e2e"]["ms_per_step"], b["cold_ms"], b["clocks"]))
print("ratio device %.0fx, e2e %.0fx vs reference arm %.3e" % (b["value"] / ref["value"], b["e2e"]["value"] / ref["value"], ref["value"]))
