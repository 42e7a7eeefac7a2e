"""Benchmark: BVE tree-code velocity evaluations/s at N = 2,621,442 (fp64).

Workload (BASELINE.json config 4, the metric's own config): Lagrangian BVE
time stepping on the level-9 icosahedral mesh (N = 2,621,442), BASELINE
Rossby-Haurwitz R=4 initial vorticity, Voronoi (node-patch) areas, RK4 with
dt = 0.01, Omega = 2 pi, positions renormalised after every stage;
Biot-Savart kernel, interpolation degree 8, theta = 0.7, N_T = 64,
max_depth = 10. One "step" is one RK4 step on moving particles: four full
tree-code velocity evaluations (binning into the persistent tree, dual
traversal and list compaction, upward pass, CP/CC + fit, PP + PC, downward
pass) plus the stage updates, all on the device.

  value : velocity evaluations/s (4 N per step) with the state resident in
          HBM, device time per step from CUDA events, L2 flushed between
          steps (256 MiB write, outside the timed span).
  e2e   : the same through the public RK4 entry point (ss.rk4 -> ssum_rk4,
          host arrays): H2D of x, zeta, A and D2H of x, zeta in every step.
  roofline : the interaction tiles, k_tiles<fit> (CP + CC + fit, high-priority
          side stream) concurrent with k_tiles<leaf> (PP + PC): algorithmic
          flops (13 per pair) / their event-timed span, summed
          over the timed evaluations, against the DFMA peak measured live on
          this GPU (MEASURED_PEAKS.json has no fp64 entry).
  cpu_baseline : the unmodified reference (oracle/_ref: the reference's
          treecode_sum in the restated RK4 driver) for one RK4 step of the
          same state on all host threads; also the one-step parity.
  cold_ms / static_eval : the first evaluation on a fresh FaceTree, and the
          round-1 line (one evaluation of the initial state, static input).

`--config` prints the same line for the other BASELINE configs (c1, c2,
c2pc, c2log, c3, c5: single evaluations; c4eval: config 4's initial state,
one evaluation per step). `--impl reference` times the reference's CPU path
on the same workload (rank 0 only; inputs built without the product
library). `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks (target leaves partitioned by
interaction cost; one all-gather of the rows per RK4 stage).
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

UNIT = "velocity_evals/s"
OMEGA = 2.0 * np.pi  # test_cases.hpp:11
# BASELINE.json workloads. "c4" (the metric's config) is the RK4 time
# stepping; the others are single evaluations (parity-test sizes, reported
# for information).
CONFIGS = {
    "c4": dict(metric="BVE tree-code velocity evals/s (N=2.6M, fp64)", mesh=9, rk4=dict(dt=0.01),
               cfg=dict(theta=0.7, n_threshold=64, degree=8, max_depth=10),
               workload="config4: L9 icosahedral mesh N=2,621,442, BASELINE RH4 initial vorticity, Voronoi areas, "
                        "Lagrangian RK4 dt=0.01 Omega=2pi (particles move; 4 treecode_sum per step on the "
                        "persistent tree), Biot-Savart, d=8, theta=0.7, N_T=64, max_depth=10"),
    "c4eval": dict(metric="BVE tree-code velocity evals/s (N=2.6M, fp64)", mesh=9,
                   cfg=dict(theta=0.7, n_threshold=64, degree=8, max_depth=10),
                   workload="config4 initial state, one full treecode_sum per step (static input): L9 mesh, RH4, "
                            "Voronoi areas, Biot-Savart, d=8, theta=0.7, N_T=64, max_depth=10"),
    "c1": dict(metric="BVE tree-code velocity evals/s (N=10k, fp64)", mesh=5,
               cfg=dict(theta=0.7, n_threshold=64, degree=4, max_depth=10),
               workload="config1: L5 icosahedral mesh N=10,242, RH4, Voronoi areas, Biot-Savart, d=4, theta=0.7, "
                        "N_T=64; one full treecode_sum per step"),
    "c2": dict(metric="BVE tree-code velocity evals/s (N=655k, fp64)", mesh=8,
               cfg=dict(theta=0.7, n_threshold=64, degree=8, max_depth=10),
               workload="config2: L8 icosahedral mesh N=655,362, RH4, Voronoi areas, Biot-Savart, d=8, "
                        "theta=0.7, cluster-cluster; one full treecode_sum per step"),
    "c2pc": dict(metric="BVE tree-code velocity evals/s (N=655k, PC-only, fp64)", mesh=8,
                 cfg=dict(theta=0.7, n_threshold=64, degree=8, max_depth=10, pc_only=True),
                 workload="config2 PC-only mode: L8 icosahedral mesh N=655,362, RH4, Voronoi areas, Biot-Savart, "
                          "d=8, theta=0.7, particle-cluster traversal (CP->PP, CC->PC; not in the reference: "
                          "CPU baseline is the oracle port, single thread)"),
    "c2log": dict(metric="BVE tree-code stream-function evals/s (N=655k, fp64)", mesh=8, kernel=1,
                  cfg=dict(theta=0.7, n_threshold=64, degree=8, max_depth=10),
                  workload="config2 stream function: L8 icosahedral mesh N=655,362, RH4, Voronoi areas, "
                           "log kernel (psi), d=8, theta=0.7, cluster-cluster"),
    "c3": dict(metric="BVE tree-code velocity evals/s (N=4.2M random cap, fp64)", cap=1 << 22,
               cfg=dict(theta=0.7, n_threshold=64, degree=8, max_depth=10),
               workload="config3: 2^22 seeded points (half uniform, half in a 10 deg cap at lat 40), Gaussian "
                        "vortex minus its mean, A=4pi/N, Biot-Savart, d=8, theta=0.7, N_T=64, max_depth=10"),
    "c5": dict(metric="BVE tree-code velocity evals/s (N=10.5M, fp64)", mesh=10,
               cfg=dict(theta=0.8, n_threshold=64, degree=8, max_depth=10),
               workload="config5: L10 icosahedral mesh N=10,485,762, RH4, Voronoi areas, Biot-Savart, d=8, "
                        "theta=0.8, cluster-cluster; one full treecode_sum per step"),
}
C = {}  # the selected config (use_config)


def use_config(name):
    c = CONFIGS[name]
    C.clear()
    C.update(c)
    C["name"] = name
    C["kernel"] = c.get("kernel", 0)
    C["dim"] = 3 if C["kernel"] == 0 else 1
    C["flop_per_pair"] = 13 if C["kernel"] == 0 else 9  # F_BS, F_log


def config_dict(n):
    """The JSON line's config (identical in both arms)."""
    return {"workload": C["workload"], **C["cfg"], "n": n}


def kernel_class(ss):
    return ss.BiotSavartKernel if C["kernel"] == 0 else ss.LogPotentialKernel


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ------------------------------------------------------------------ inputs
def fixture_product():
    """(xyz, zeta, area) from the product's host generators."""
    import paper_2401_07361_b200 as ss

    if "cap" in C:
        return ss.make_random_cap(C["cap"], 5)
    xyz, area = ss.make_icosa_mesh(C["mesh"])
    return xyz, ss.rh4_vorticity(xyz), area


def fixture_reference():
    """The same inputs bit for bit without the product library: the
    reference's own make_icosa_mesh and the oracle's generator restatements
    (tests/test_host.py::test_oracle_fixtures_bit_identical_to_product)."""
    import oracle_lib as ol

    if "cap" in C:
        return ol.orc_random_cap(C["cap"], 5)
    xyz, area = ol.mesh(C["mesh"])
    return xyz, ol.orc_rh4(xyz), area


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.perf_counter(), [x.strip() for x in line.split(",")]))

    def window(self, t0, t1):
        inside = [r for t, r in self.rows if t0 <= t <= t1 + 0.05]
        if not inside and self.rows:
            inside = [min(self.rows, key=lambda tr: abs(tr[0] - t1))[1]]
        self.rows = [(0.0, r) for r in inside]

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        rows = [r for _, r in self.rows]
        num = lambda v: v.replace(".", "").isdigit()  # noqa: E731
        sm = [float(r[0]) for r in rows if num(r[0])]
        mx = [float(r[1]) for r in rows if num(r[1])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if len(r) > 3 + k and r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max((float(r[2]) for r in rows if num(r[2])), default=None)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ------------------------------------------------------------ reference arm
def reference_kind():
    """The unmodified reference (oracle/_ref, all host threads), or — PC-only
    mode, which the reference lacks — the oracle port (one thread)."""
    return "port" if C["cfg"].get("pc_only") else "reference"


def reference_eval(ol, xyz, q, workers):
    cf = C["cfg"]
    t0 = time.perf_counter()
    if cf.get("pc_only"):
        out, _ = ol.orc_treecode(C["kernel"], xyz, q, cf["theta"], cf["n_threshold"], cf["degree"],
                                 cf["max_depth"], pc_only=True)
    else:
        out, _ = ol.ref_treecode(C["kernel"], xyz, q, cf["theta"], cf["n_threshold"], cf["degree"],
                                 cf["max_depth"], workers)
    return time.perf_counter() - t0, out


def reference_rk4(ol, x, z, area, steps, workers):
    cf = C["cfg"]
    t0 = time.perf_counter()
    x1, z1 = ol.ref_rk4(x, z, area, cf["theta"], cf["n_threshold"], cf["degree"], cf["max_depth"],
                        C["rk4"]["dt"], steps, OMEGA, workers=workers)
    return time.perf_counter() - t0, x1, z1


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle_lib as ol

    if not ol.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libspheresum_ref.so not built"}))
        return
    cores = (os.cpu_count() or 1) if reference_kind() == "reference" else 1
    xyz, zeta, area = fixture_reference()
    n = xyz.shape[0]
    q = zeta * area
    budget = 240.0
    # warm-up on the level-5 mesh (threads, page cache, lattice_fit cache)
    wx, wa = ol.mesh(5)
    wz = ol.orc_rh4(wx)
    for _ in range(args.warmup):
        if "rk4" in C:
            reference_rk4(ol, wx, wz, wa, 1, cores)
        else:
            reference_eval(ol, wx, wz * wa, cores)
    evals_per_step = 4 if "rk4" in C else 1
    if "rk4" in C:
        # one step first (sizes the rest), then the remaining steps the budget
        # allows in one call (one tree across them, as in the device arm)
        dt1, x, z = reference_rk4(ol, xyz, zeta, area, 1, cores)
        done, total = 1, dt1
        more = min(args.steps - 1, int((budget - dt1) / max(dt1, 1e-9)))
        if more > 0:
            dtm, x, z = reference_rk4(ol, x, z, area, more, cores)
            done, total = done + more, total + dtm
        sample = (f"{done} RK4 steps ({4 * done} treecode_sum evaluations, the reference's treecode_sum in the "
                  f"restated RK4 driver oracle/ref_capi.cpp:ref_rk4) of {args.steps} requested, {budget:.0f} s "
                  f"budget; warm-up on a level-5 mesh")
    else:
        times = []
        for k in range(args.steps):
            dt, _ = reference_eval(ol, xyz, q, cores)
            times.append(dt)
            if sum(times) > budget and k + 1 < args.steps:
                break
        done, total = len(times), sum(times)
        sample = (f"full {C['name']} treecode_sum per step ({done} timed of {args.steps} requested, "
                  f"{budget:.0f} s budget); warm-up on a level-5 mesh")
    ms = 1e3 * total / done
    value = evals_per_step * n / (ms * 1e-3)
    loaded = [ln.split()[-1] for ln in open("/proc/self/maps") if ln.rstrip().endswith(".so")]
    print(json.dumps({
        "impl": "reference", "metric": C["metric"], "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": config_dict(n),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": reference_kind(), "cpu": cpu_model(),
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_library_loaded": any("libspheresum_b200" in x for x in loaded),
    }))


# ------------------------------------------------------------------ GPU arm
class Stepper:
    """One evaluation / one RK4 step of the selected config on this rank's
    FaceTree, with per-evaluation TreecodeStats collected."""

    def __init__(self, ss, torch, dev, xyz, zeta, area, ws, rank):
        from paper_2401_07361_b200.dist import TreecodeRK4Ops

        self.ss, self.torch, self.ws = ss, torch, ws
        self.n = xyz.shape[0]
        self.cfg = ss.TraversalConfig(**C["cfg"])
        self.tree = ss.FaceTree(dev.index)
        self.tree.set_stream(torch.cuda.current_stream(dev).cuda_stream)
        if ws > 1:
            self.tree.set_partition(rank, ws)
        f64 = dict(dtype=torch.float64, device=dev)
        self.x = torch.from_numpy(xyz).to(dev)
        self.z = torch.from_numpy(zeta).to(dev)
        self.area = torch.from_numpy(area).to(dev)
        self.q = self.z * self.area
        self.out = torch.zeros((self.n, C["dim"]), **f64)
        self.stats = []
        if "rk4" in C:
            self.ops = TreecodeRK4Ops(self.tree, self.cfg, stats=self.stats)
            self.st = self.ops.state(self.x, self.z, self.area)

    def step(self):
        """Returns the number of our kernel launches."""
        if "rk4" in C:
            return self.ops.step(C["rk4"]["dt"], self.st)
        s = self.ss.TreecodeStats()
        self.ss.treecode_sum_device(self.tree, kernel_class(self.ss), self.cfg, self.x.data_ptr(),
                                    self.q.data_ptr(), self.n, self.out.data_ptr(), stats=s)
        if self.ws > 1:
            from paper_2401_07361_b200.dist import gather_rows

            gather_rows(self.tree, self.out)
        self.stats.append(s)
        return s.gpu_launches


def run_gpu(args):
    import torch

    import paper_2401_07361_b200 as ss

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    xyz, zeta, area = fixture_product()
    n = xyz.shape[0]
    q = zeta * area
    evals_per_step = 4 if "rk4" in C else 1
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v, op="max"):
        if ws == 1:
            return v
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=getattr(torch.distributed.ReduceOp, op.upper()))
        return float(t.item())

    # cold: the first evaluation on a fresh FaceTree (tree built from scratch,
    # every buffer allocated), in a warm process: a throw-away tree first
    # loads the kernels (lazy module loading) and leaves its device blocks
    # cached in the pool, as any earlier FaceTree of the process would
    d_x = torch.from_numpy(xyz).to(dev)
    d_q = torch.from_numpy(q).to(dev)
    d_o = torch.zeros((n, C["dim"]), dtype=torch.float64, device=dev)
    w = ss.FaceTree(local)
    w.set_stream(stream.cuda_stream)
    for _ in range(2):
        ss.treecode_sum_device(w, kernel_class(ss), ss.TraversalConfig(**C["cfg"]), d_x.data_ptr(), d_q.data_ptr(),
                               n, d_o.data_ptr())
    w.close()
    cold = ss.FaceTree(local)
    cold.set_stream(stream.cuda_stream)
    barrier()
    t0 = time.perf_counter()
    ss.treecode_sum_device(cold, kernel_class(ss), ss.TraversalConfig(**C["cfg"]), d_x.data_ptr(), d_q.data_ptr(),
                           n, d_o.data_ptr())
    torch.cuda.synchronize()
    cold_ms = (time.perf_counter() - t0) * 1e3
    # warm static single evaluation of the initial state (round-1 line)
    static_ms = []
    if "rk4" in C:
        for k in range(4):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ss.treecode_sum_device(cold, kernel_class(ss), ss.TraversalConfig(**C["cfg"]), d_x.data_ptr(),
                                   d_q.data_ptr(), n, d_o.data_ptr())
            e1.record(stream)
            torch.cuda.synchronize()
            if k:
                static_ms.append(e0.elapsed_time(e1))
    cold.close()
    del d_o

    S = Stepper(ss, torch, dev, xyz, zeta, area, ws, rank)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    clocks = ClockSampler(local).__enter__()
    for _ in range(max(args.warmup, 3)):
        S.step()
    torch.cuda.synchronize()
    peak = S.tree.fp64_peak_tflops(5)
    S.stats.clear()
    times, launches = [], 0
    t_start = time.perf_counter()
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launches += S.step()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    barrier()
    t_end = time.perf_counter()
    time.sleep(0.12)
    clocks.__exit__(None, None, None)
    clocks.window(t_start, t_end)
    total_ms = max_over_ranks(sum(times))
    ms_per_step = total_ms / args.steps
    value = evals_per_step * n / (ms_per_step * 1e-3)
    stats = S.stats  # the timed evaluations (this rank's parts)
    last = stats[-1]

    # e2e through the public API with host buffers
    e2e = e2e_run(ss, torch, dev, S, xyz, zeta, area, q, ws, rank, args, barrier)
    e2e_s = max_over_ranks(e2e.pop("seconds"))  # mean over the timed calls; each call's time is in times_ms
    e2e["value"] = evals_per_step * n / e2e_s
    e2e["ms_per_step"] = e2e_s * 1e3

    pairs = sum(sum(s.kernel_evals) for s in stats)  # PP + PC + CP + CC pairs of both tile kernels
    tiles_ms = sum(s.tiles_ms for s in stats)
    fpp = C["flop_per_pair"]
    achieved = fpp * pairs / (tiles_ms * 1e-3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "tiles_dram.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    job_pairs = max_over_ranks(pairs, "sum")
    try:
        hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        hbm = 7700.0  # B200_PROFILING.md fallback
    mean = lambda f: statistics.mean(f(s) for s in stats)  # noqa: E731
    line = {
        "metric": C["metric"], "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(n),
        "l2": "flushed between steps (256 MiB write outside the timed span)",
        "parallelism": f"target-leaf partition x{ws}, one row all-gather per evaluation" if ws > 1 else "single GPU",
        "evaluations_per_step": evals_per_step,
        "roofline": {"bound": "fp64",
                     "kernel": "k_tiles<fit> (CP+CC+fit, high-priority side stream) + k_tiles<leaf> (PP+PC), "
                               "concurrent", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": "DFMA-chain probe on this GPU (ssum_fp64_peak); MEASURED_PEAKS.json has no fp64",
                     "flop_per_pair": fpp, "pairs_per_launch": pairs / len(stats),
                     "avg_launch_ms": tiles_ms / len(stats), "launches_timed": len(stats),
                     "timing": "CUDA events on the main stream around the fork to k_tiles<fit> (side stream) "
                               "and the join behind k_tiles<leaf>, every timed evaluation"},
        "e2e": e2e,
        "gpu_launches": launches,
        "interactions_per_s": job_pairs / (total_ms * 1e-3),
        "all_kernel_flops_frac": fpp * pairs / (total_ms * 1e-3) / 1e12 / peak,
        "cold_ms": max_over_ranks(cold_ms),
        "phase_ms_per_evaluation": {
            "bin": mean(lambda s: s.bin_seconds) * 1e3, "traversal": mean(lambda s: s.traversal_seconds) * 1e3,
            "eval": mean(lambda s: s.eval_seconds) * 1e3, "upward": mean(lambda s: s.upward_ms),
            "cp_cc_fit": mean(lambda s: s.cp_cc_fit_ms), "pp_pc": mean(lambda s: s.pp_pc_ms),
            "tiles_concurrent": mean(lambda s: s.tiles_ms), "downward_finish": mean(lambda s: s.finish_ms)},
        "kernel_evals_per_evaluation": {k: int(last.kernel_evals[i]) for i, k in enumerate(("pp", "pc", "cp", "cc"))},
        "passes": passes(stats, peak, hbm, n),
        "mac_host_decisions": last.mac_host_decisions,
        "clocks": clocks.summary(),
    }
    if static_ms:
        line["static_eval"] = {"ms": statistics.mean(static_ms), "value": n / (statistics.mean(static_ms) * 1e-3),
                               "what": "one treecode_sum of the initial (static) state on a warm tree"}
    if rank == 0 and ws == 1:
        extras(ss, torch, dev, line, xyz, zeta, area, q, args)
    if rank == 0:
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()


def passes(stats, peak, hbm, n):
    """Upward / downward passes: algorithmic flops per
    (particle, node) visit plus the p x p transforms per node; bytes as
    stated there; mean over the timed evaluations."""
    s = stats[-1]
    deg = C["cfg"]["degree"]
    p_pts = (deg + 1) * (deg + 2) // 2
    base = 21 + 3 * (deg - 1)
    per_term = 2 + 2 * C["dim"]
    up_flop = s.up_visits * (base + 4 * p_pts) + s.weight_nodes * 2 * p_pts * p_pts
    down_flop = s.down_visits * (base + per_term * p_pts) + s.fit_nodes * 2 * C["dim"] * p_pts * p_pts

    def one(flop, byts, ms):
        t = max(ms, 1e-9) * 1e-3
        return {"ms": ms, "TFLOP/s": flop / t / 1e12, "fp64_frac": flop / t / 1e12 / peak, "GB/s": byts / t / 1e9,
                "hbm_frac": byts / t / 1e9 / hbm, "flop": flop, "bytes": byts}

    return {"visits": {"upward": s.up_visits, "downward": s.down_visits},
            "upward": one(up_flop, 32 * s.up_visits, statistics.mean(x.upward_ms for x in stats)),
            "downward": one(down_flop, (32 + 8 * C["dim"]) * n, statistics.mean(x.finish_ms for x in stats)),
            "flop_per_visit": {"upward": base + 4 * p_pts, "downward": base + per_term * p_pts},
            "hbm_peak_gbs": hbm}


def e2e_run(ss, torch, dev, S, xyz, zeta, area, q, ws, rank, args, barrier):
    """The metric through the public API with host buffers, host<->device
    copies inside every timed step."""
    n = xyz.shape[0]
    reps = min(args.steps, 5)
    times = []
    if "rk4" in C:
        # ss.rk4 (ssum_rk4) on pinned host arrays advanced in place: H2D of
        # x, zeta, A; one RK4 step; D2H of x, zeta
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
        hx, hz, ha = pin(xyz), pin(zeta), pin(area)
        if ws == 1:
            tree = ss.FaceTree(dev.index)
            for k in range(reps + 1):
                barrier()
                t0 = time.perf_counter()
                ss.rk4(hx, hz, ha, S.cfg, dt=C["rk4"]["dt"], steps=1, omega=OMEGA, tree=tree, inplace=True)
                dt = time.perf_counter() - t0
                if k:
                    times.append(dt)
            tree.close()
            return {"unit": UNIT, "h2d_bytes_per_step": int(hx.nbytes + hz.nbytes + area.nbytes),
                    "d2h_bytes_per_step": int(hx.nbytes + hz.nbytes), "seconds": statistics.mean(times),
                    "times_ms": [round(t * 1e3, 3) for t in times],
                    "path": "ss.rk4 -> ssum_rk4 (pinned host arrays, in place), one RK4 step per call"}
        from paper_2401_07361_b200.dist import allgather_inputs, shard_rows

        r0, r1 = shard_rows(n, ws, rank)
        m = -(-n // ws)
        px, pz = torch.from_numpy(hx).pin_memory(), torch.from_numpy(hz).pin_memory()
        dx = torch.zeros((ws * m, 3), dtype=torch.float64, device=dev)
        dz = torch.zeros(ws * m, dtype=torch.float64, device=dev)
        for k in range(reps + 1):
            barrier()
            t0 = time.perf_counter()
            allgather_inputs(px, pz, dx, dz)  # H2D of this rank's shard + NCCL all-gather
            S.st["x0"].copy_(dx[:n])
            S.st["z0"].copy_(dz[:n])
            S.step()
            px[r0:r1].copy_(S.st["x0"][r0:r1])  # D2H of this rank's shard
            pz[r0:r1].copy_(S.st["z0"][r0:r1])
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if k:
                times.append(dt)
        return {"unit": UNIT, "h2d_bytes_per_step": int(32 * n), "d2h_bytes_per_step": int(32 * n),
                "seconds": statistics.mean(times), "times_ms": [round(t * 1e3, 3) for t in times],
                "path": "per rank: H2D of its 1/ws shard of x and zeta, NCCL all-gather, one partitioned RK4 "
                        "step (row all-gather per stage), D2H of its shard (bytes: whole job; A resident)"}
    h_xyz = torch.from_numpy(xyz).pin_memory()
    h_q = torch.from_numpy(q).pin_memory()
    h_out = torch.zeros((n, C["dim"]), dtype=torch.float64).pin_memory()
    if ws > 1:
        from paper_2401_07361_b200.dist import allgather_inputs, gather_rows, shard_rows

        r0, r1 = shard_rows(n, ws, rank)
        m = -(-n // ws)
        dx = torch.zeros((ws * m, 3), dtype=torch.float64, device=dev)
        dq = torch.zeros(ws * m, dtype=torch.float64, device=dev)
    for k in range(reps + 1):
        barrier()
        t0 = time.perf_counter()
        if ws == 1:
            ss.treecode_sum(kernel_class(ss), h_xyz.numpy(), h_q.numpy(), S.cfg, tree=S.tree, out=h_out.numpy())
        else:
            allgather_inputs(h_xyz, h_q, dx, dq)
            ss.treecode_sum_device(S.tree, kernel_class(ss), S.cfg, dx.data_ptr(), dq.data_ptr(), n,
                                   S.out.data_ptr())
            gather_rows(S.tree, S.out)
            h_out[r0:r1].copy_(S.out[r0:r1])
            torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if k:
            times.append(dt)
    S.h_out = h_out.numpy()
    return {"unit": UNIT, "h2d_bytes_per_step": int(xyz.nbytes + q.nbytes), "d2h_bytes_per_step": int(n * C["dim"] * 8),
            "seconds": statistics.mean(times), "times_ms": [round(t * 1e3, 3) for t in times],
            "path": "ssum_treecode_sum (host pointers)" if ws == 1 else
                    "per rank: H2D of its 1/ws input shard, NCCL all-gather of x and q, its targets, NCCL "
                    "all-gather of the rows, D2H of its 1/ws result shard (bytes: whole job)"}


def extras(ss, torch, dev, line, xyz, zeta, area, q, args):
    """Rank 0, one GPU: the CPU baseline (the unmodified reference on the same
    input, all host threads), parity against it, and the error against
    direct summation (outside the timed region)."""
    import oracle_lib as ol

    cfg = ss.TraversalConfig(**C["cfg"])
    n = xyz.shape[0]
    # this implementation's result to compare: one RK4 step, or one evaluation
    if "rk4" in C:
        mx, mz = ss.rk4(xyz, zeta, area, cfg, dt=C["rk4"]["dt"], steps=1, omega=OMEGA, tree=ss.FaceTree(dev.index))
    u0 = ss.treecode_sum(kernel_class(ss), xyz, q, cfg, tree=ss.FaceTree(dev.index))
    ref_u = None
    if not args.no_cpu_baseline and ol.ref_available():
        kind = reference_kind()
        cores = (os.cpu_count() or 1) if kind == "reference" else 1
        what = f"unmodified reference, workers={cores}" if kind == "reference" else "oracle port, 1 thread"
        if "rk4" in C:
            dt, rx, rz = reference_rk4(ol, xyz, zeta, area, 1, cores)
            line["cpu_baseline"] = {"value": 4 * n / dt, "unit": UNIT, "cores": cores, "kind": kind, "cpu": cpu_model(),
                                    "sample": f"one RK4 step (4 treecode_sum evaluations) of the initial state "
                                              f"({what}, restated RK4 driver), {dt:.1f} s"}
            line["parity_rk4_one_step"] = {"x_rel_l2": ol.rel_l2(mx, rx), "zeta_rel_l2": ol.rel_l2(mz, rz),
                                           "tolerance": 1e-10}
            line["parity_rel_l2_vs_reference"] = max(ol.rel_l2(mx, rx), ol.rel_l2(mz, rz))
        else:
            dt, ref_u = reference_eval(ol, xyz, q, cores)
            line["cpu_baseline"] = {"value": n / dt, "unit": UNIT, "cores": cores, "kind": kind, "cpu": cpu_model(),
                                    "sample": f"one full {C['name']} treecode_sum ({what}), {dt:.1f} s"}
            line["parity_rel_l2_vs_reference"] = ol.rel_l2(u0, ref_u)
    elif not args.no_cpu_baseline:
        line["cpu_baseline"] = None
    if not args.no_error:
        try:
            line["error_vs_direct"] = sampled_direct_error(xyz, q, u0, dev, ref_u)
        except Exception as exc:  # a failed extra must not cost the bench line
            line["error_vs_direct"] = {"error": repr(exc)}


def sampled_direct_error(xyz, q, u_tree, dev, u_ref=None, m=2048, seed=2024):
    """Relative L2 error of the tree code against direct summation on m
    seeded random targets (all N sources; fp64 torch matmuls, outside the
    timed region). The reference measured E = 2.38e-6 at config 4 (SURVEY.md
    §8(d)); the bar is E(mine) <= E(reference)."""
    import torch

    n = xyz.shape[0]
    idx = np.random.default_rng(seed).choice(n, size=min(m, n), replace=False)
    X = torch.from_numpy(xyz).to(dev)
    Q = torch.from_numpy(q).to(dev)
    tid = torch.from_numpy(idx).to(dev)
    T = X[tid]
    S = torch.zeros_like(T) if C["kernel"] == 0 else torch.zeros(len(idx), dtype=torch.float64, device=dev)
    chunk = 1 << 18
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        den = 1.0 - T @ X[c0:c1].T
        own = (tid >= c0) & (tid < c1)  # self pairs excluded
        rows, cols = own.nonzero().squeeze(1), (tid[own] - c0)
        if C["kernel"] == 0:
            den[rows, cols] = float("inf")
            S += (Q[c0:c1] / den) @ X[c0:c1]
        else:
            lg = torch.log(den)
            lg[rows, cols] = 0.0
            S += lg @ Q[c0:c1]
    u_dir = (-1.0 / (4.0 * np.pi)) * (torch.cross(T, S, dim=1) if C["kernel"] == 0 else S)

    def rel(u):
        ut = torch.from_numpy(np.ascontiguousarray(u[idx])).to(dev).reshape(u_dir.shape)
        return float(torch.linalg.norm(ut - u_dir) / torch.linalg.norm(u_dir))

    e_tree = rel(u_tree)
    e_ref = rel(u_ref) if u_ref is not None else None
    out = {"value": e_tree, "reference_same_targets": e_ref, "targets": int(len(idx)), "seed": seed,
           "survey_reference_E_config4": 2.38e-6, "state": "initial state (one evaluation)",
           "definition": "||u_tree - u_direct||_2 / ||u_direct||_2 over the sampled targets"}
    if e_ref is not None:
        out["relative_difference"] = (e_tree - e_ref) / e_ref
        out["not_worse_than_reference"] = bool(e_tree <= e_ref * (1 + 1e-6))
    return out


def relaunch(n):
    """`--gpus N` outside torchrun: re-run this command under
    torch.distributed.run with N ranks on this node (127.0.0.1)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-error", action="store_true", help="skip the sampled error vs direct summation")
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS), help="BASELINE workload (default c4)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    use_config(args.config)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
