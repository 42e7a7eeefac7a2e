"""Benchmark: BVE tree-code velocity evaluations/s at N = 2,621,442 (fp64).

Workload (BASELINE.json config 4, one velocity evaluation = one "step"):
level-9 icosahedral mesh (N = 2,621,442 vertices), BASELINE Rossby-Haurwitz
R=4 vorticity, Voronoi (node-patch) areas, q = zeta * A; Biot-Savart kernel,
interpolation degree 8, theta = 0.7, N_T = 64, max_depth = 10. A step is the
whole treecode_sum: face-tree binning, dual traversal and list compaction,
upward pass, CP/CC + fit, PP + PC, downward pass — nothing cached between
steps except the persistent tree geometry (FaceTree semantics).

  value : velocity evals/s with inputs resident in HBM (device pointers),
          device time per step from CUDA events, L2 flushed between steps.
  e2e   : the same through the C-ABI host-pointer entry point
          (ssum_treecode_sum) from pinned host buffers: H2D of xyz+q and D2H
          of the velocities inside every timed step.
  roofline : the dominant kernels — the interaction tiles, k_tiles<fit>
          (CP + CC pairs + fit, high-priority side stream) running
          concurrently with k_tiles<leaf> (PP + PC pairs) — algorithmic flops (13 per
          pair; the fit epilogue's flops not counted) / the
          event-timed span of the two together,
          against the DFMA peak measured live on this GPU (no fp64 entry in
          MEASURED_PEAKS.json).
  cpu_baseline : the unmodified reference (oracle/_ref, compiled from
          /root/reference/proj/src) on the same input, all host threads.

`--impl reference` times that reference CPU path alone (rank 0).
Multi-GPU (torchrun): target leaves are partitioned across ranks by
interaction cost (strong scaling); every rank builds the tree.
"""
import argparse
import json
import os
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
FLOP_PER_PAIR = 13  # F_BS
# BASELINE.json workloads. The bench line is config 4 (the metric's own
# config); --config c2 / c3 / c5 print the same line for the other
# single-evaluation configs (parity-test sizes, reported for information).
CONFIGS = {
    "c4": dict(metric="BVE tree-code velocity evals/s (N=2.6M, fp64)", mesh=9,
               cfg=dict(theta=0.7, n_threshold=64, degree=8, max_depth=10),
               workload="config4: L9 icosahedral mesh N=2,621,442, BASELINE RH4 vorticity, Voronoi areas, "
                        "Biot-Savart, d=8, theta=0.7, N_T=64, max_depth=10; one full treecode_sum per step"),
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
CONFIG = "c4"
METRIC = CONFIGS[CONFIG]["metric"]
CFG = CONFIGS[CONFIG]["cfg"]
WORKLOAD = CONFIGS[CONFIG]["workload"]
KERNEL = 0  # 0 Biot-Savart (velocity, D = 3), 1 log (stream function, D = 1)
DIM = 3


def use_config(name):
    global CONFIG, METRIC, CFG, WORKLOAD, KERNEL, DIM, FLOP_PER_PAIR
    CONFIG = name
    METRIC, CFG, WORKLOAD = CONFIGS[name]["metric"], CONFIGS[name]["cfg"], CONFIGS[name]["workload"]
    KERNEL = CONFIGS[name].get("kernel", 0)
    DIM = 3 if KERNEL == 0 else 1
    FLOP_PER_PAIR = 13 if KERNEL == 0 else 9  # F_BS, F_log


def kernel_class(ss):
    return ss.BiotSavartKernel if KERNEL == 0 else ss.LogPotentialKernel


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def fixture():
    import paper_2401_07361_b200 as ss

    c = CONFIGS[CONFIG]
    if "cap" in c:
        xyz, zeta, area = ss.make_random_cap(c["cap"], 5)
        return xyz, zeta * area, area
    xyz, area = ss.make_icosa_mesh(c["mesh"])
    q = ss.rh4_vorticity(xyz) * area
    return xyz, q, area


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
        """Keep the samples taken during [t0, t1] (the timed region); if the
        region is shorter than the sampling period keep the nearest one."""
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
        self.rows = [r for _, r in self.rows] if isinstance(self.rows[0], tuple) else self.rows
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 3 + k and r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max((float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()),
                                   default=None)}


def cpu_model():
    """Host CPU model name (the reference arm's hardware)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def reference_kind():
    """The CPU baseline of this config: the unmodified reference (oracle/_ref,
    all host threads), or — PC-only mode, which the reference lacks — the
    oracle port (one thread)."""
    return "port" if CFG.get("pc_only") else "reference"


def reference_step(ol, xyz, q, workers):
    t0 = time.perf_counter()
    if CFG.get("pc_only"):
        out, st = ol.orc_treecode(KERNEL, xyz, q, CFG["theta"], CFG["n_threshold"], CFG["degree"],
                                  CFG["max_depth"], pc_only=True)
    else:
        out, st = ol.ref_treecode(KERNEL, xyz, q, CFG["theta"], CFG["n_threshold"], CFG["degree"],
                                  CFG["max_depth"], workers)
    return time.perf_counter() - t0, out, st


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle_lib as ol

    if not ol.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libspheresum_ref.so not built"}))
        return
    cores = (os.cpu_count() or 1) if reference_kind() == "reference" else 1
    xyz, q, area = fixture()
    n = xyz.shape[0]
    # warm-up on a level-5 sample (threads, page cache, lattice_fit cache)
    import paper_2401_07361_b200 as ss

    wx, wa = ss.make_icosa_mesh(5)
    wq = ss.rh4_vorticity(wx) * wa
    for _ in range(args.warmup):
        reference_step(ol, wx, wq, cores)
    times = []
    budget = 240.0
    for k in range(args.steps):
        dt, _, _ = reference_step(ol, xyz, q, cores)
        times.append(dt)
        if sum(times) > budget and k + 1 < args.steps:
            break
    ms = 1e3 * statistics.mean(times)
    value = n / (ms * 1e-3)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, **CFG, "n": n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": reference_kind(), "cpu": cpu_model(),
                         "sample": f"full {CONFIG} treecode_sum per step ({len(times)} timed of {args.steps} "
                                   f"requested, 240 s budget); warm-up steps on a level-5 mesh"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def run_gpu(args):
    import torch

    import paper_2401_07361_b200 as ss

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    xyz, q, area = fixture()
    n = xyz.shape[0]
    cfg = ss.TraversalConfig(**CFG)
    dev = torch.device("cuda", local)
    # rows [0, n) are the particles; padded to ws equal slots for the input
    # all-gather of the distributed e2e path (dist.allgather_inputs)
    rows = ws * -(-n // ws)
    d_xyz = torch.zeros((rows, 3), dtype=torch.float64, device=dev)
    d_q = torch.zeros(rows, dtype=torch.float64, device=dev)
    d_xyz[:n].copy_(torch.from_numpy(xyz))
    d_q[:n].copy_(torch.from_numpy(q))
    d_out = torch.zeros((n, DIM), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    tree = ss.FaceTree(local)
    tree.set_stream(stream.cuda_stream)
    if ws > 1:
        tree.set_partition(rank, ws)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2

    def step(st):
        ss.treecode_sum_device(tree, kernel_class(ss), cfg, d_xyz.data_ptr(), d_q.data_ptr(), n,
                               d_out.data_ptr(), stats=st)

    clocks = ClockSampler(local).__enter__()
    for _ in range(max(args.warmup, 3)):
        step(ss.TreecodeStats())
    torch.cuda.synchronize()
    peak = tree.fp64_peak_tflops(5)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    times, pp_ms, launches = [], [], 0
    stats = None
    t_start = time.perf_counter()
    if True:
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            stats = ss.TreecodeStats()
            step(stats)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            pp_ms.append(stats.tiles_ms)
            launches += stats.gpu_launches
        barrier()
    t_end = time.perf_counter()
    time.sleep(0.12)
    clocks.__exit__(None, None, None)
    clocks.window(t_start, t_end)
    total_ms = sum(times)
    if ws > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = n / (ms_per_step * 1e-3)

    # e2e through the host-pointer C-ABI entry point with pinned buffers
    h_xyz = torch.from_numpy(xyz).pin_memory()
    h_q = torch.from_numpy(q).pin_memory()
    h_out = torch.zeros((n, DIM), dtype=torch.float64).pin_memory()
    e2e_times = []
    if ws > 1:
        from paper_2401_07361_b200.dist import allgather_inputs, gather_rows, shard_rows

        r0, r1 = shard_rows(n, ws, rank)
    for k in range(min(args.steps, 5) + 1):
        barrier()
        t0 = time.perf_counter()
        if ws == 1:
            # the public host-pointer entry point: H2D, bin, traverse, evaluate, D2H
            ss.treecode_sum(kernel_class(ss), h_xyz.numpy(), h_q.numpy(), cfg, tree=tree, out=h_out.numpy())
        else:
            # per rank: H2D of this rank's 1/ws shard of x and q, NCCL
            # all-gather of the particle set over NVLink, this rank's
            # targets, NCCL all-gather of the rows, D2H of this rank's shard
            # of the result (the ranks' host shards together are the field)
            allgather_inputs(h_xyz, h_q, d_xyz, d_q)
            step(ss.TreecodeStats())
            gather_rows(tree, d_out)
            h_out[r0:r1].copy_(d_out[r0:r1])
            torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if k > 0:
            e2e_times.append(dt)
    e2e_s = statistics.mean(e2e_times)
    if ws > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())

    pairs = sum(stats.kernel_evals)  # PP + PC + CP + CC pairs of both tile kernels
    avg_pp_ms = statistics.mean(pp_ms)
    achieved = FLOP_PER_PAIR * pairs / (avg_pp_ms * 1e-3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "tiles_dram.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    all_evals = sum(stats.kernel_evals)  # this rank's part of the work
    job_evals = all_evals
    if ws > 1:  # whole-job interactions/s: every rank's part
        t = torch.tensor([float(all_evals)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.SUM)
        job_evals = float(t.item())
    # upward / downward passes: algorithmic flops per
    # (particle, node) visit plus the p x p transforms per node; bytes as
    # stated there. Timed by the same events as phase_ms (upward includes
    # the particle gather and proxy points).
    hbm = None
    try:
        hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        hbm = 7700.0  # B200_PROFILING.md fallback
    deg = CFG["degree"]
    p_pts = (deg + 1) * (deg + 2) // 2
    base = 21 + 3 * (deg - 1)
    up_flop = stats.up_visits * (base + 4 * p_pts) + stats.weight_nodes * 2 * p_pts * p_pts
    up_bytes = 32 * stats.up_visits
    per_term = 2 + 2 * DIM  # basis product (2 mul) + DIM FMAs per coefficient
    down_flop = stats.down_visits * (base + per_term * p_pts) + stats.fit_nodes * 2 * DIM * p_pts * p_pts
    down_bytes = (32 + 8 * DIM) * n

    def _pass(flop, byts, ms):
        s = max(ms, 1e-9) * 1e-3
        return {"ms": ms, "TFLOP/s": flop / s / 1e12, "fp64_frac": flop / s / 1e12 / peak, "GB/s": byts / s / 1e9,
                "hbm_frac": byts / s / 1e9 / hbm, "flop": flop, "bytes": byts}

    passes = {"visits": {"upward": stats.up_visits, "downward": stats.down_visits},
              "upward": _pass(up_flop, up_bytes, stats.upward_ms),
              "downward": _pass(down_flop, down_bytes, stats.finish_ms),
              "flop_per_visit": {"upward": base + 4 * p_pts, "downward": base + per_term * p_pts},
              "hbm_peak_gbs": hbm}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, **CFG, "n": n, "l2": "flushed between steps (256 MiB write)",
                   "parallelism": f"target-leaf partition x{ws}" if ws > 1 else "single GPU"},
        "roofline": {"bound": "fp64",
                     "kernel": "k_tiles<fit> (CP+CC+fit, high-priority side stream) + k_tiles<leaf> (PP+PC), concurrent", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": "DFMA-chain probe on this GPU (ssum_fp64_peak); MEASURED_PEAKS.json has no fp64",
                     "flop_per_pair": FLOP_PER_PAIR, "pairs_per_launch": pairs, "avg_launch_ms": avg_pp_ms,
                     "timing": "CUDA events on the main stream: before the fork to k_tiles<fit> (side stream) "
                               "to after the join behind k_tiles<leaf>"},
        "e2e": {"value": n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(xyz.nbytes + q.nbytes),
                "d2h_bytes_per_step": int(n * DIM * 8), "ms_per_step": e2e_s * 1e3,
                "path": ("ssum_treecode_sum (host pointers)" if ws == 1 else
                         "per rank: H2D of its 1/ws input shard, NCCL all-gather of x and q, its targets, "
                         "NCCL all-gather of the rows, D2H of its 1/ws result shard (bytes: whole job)")},
        "gpu_launches": launches,
        "interactions_per_s": job_evals / (ms_per_step * 1e-3),
        "all_kernel_flops_frac": FLOP_PER_PAIR * all_evals / (ms_per_step * 1e-3) / 1e12 / peak,
        "phase_ms": {"bin": stats.bin_seconds * 1e3, "traversal": stats.traversal_seconds * 1e3,
                     "eval": stats.eval_seconds * 1e3, "upward": stats.upward_ms, "cp_cc_fit": stats.cp_cc_fit_ms,
                     "pp_pc": stats.pp_pc_ms, "tiles_concurrent": stats.tiles_ms,
                     "downward_finish": stats.finish_ms},
        "kernel_evals": {"pp": stats.kernel_evals[0], "pc": stats.kernel_evals[1], "cp": stats.kernel_evals[2],
                         "cc": stats.kernel_evals[3]},
        "passes": passes,
        "clocks": clocks.summary(),
    }
    ref_u = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        import oracle_lib as ol

        if ol.ref_available():
            kind = reference_kind()
            cores = (os.cpu_count() or 1) if kind == "reference" else 1
            dt, ref_out, _ = reference_step(ol, xyz, q, cores)
            ref_u = ref_out
            mine = h_out.numpy()
            what = f"unmodified reference, workers={cores}" if kind == "reference" else "oracle port, 1 thread"
            line["cpu_baseline"] = {"value": n / dt, "unit": UNIT, "cores": cores, "kind": kind,
                                    "cpu": cpu_model(),
                                    "sample": f"one full {CONFIG} treecode_sum ({what}), {dt:.1f} s"}
            line["parity_rel_l2_vs_reference"] = ol.rel_l2(mine, ref_out)
        else:
            line["cpu_baseline"] = None
    if rank == 0 and ws == 1 and not args.no_error:
        try:
            line["error_vs_direct"] = sampled_direct_error(xyz, q, h_out.numpy(), dev, ref_u)
        except Exception as exc:  # a failed extra must not cost the bench line
            line["error_vs_direct"] = {"error": repr(exc)}
    if rank == 0:
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()


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
    S = torch.zeros_like(T) if KERNEL == 0 else torch.zeros(len(idx), dtype=torch.float64, device=dev)
    chunk = 1 << 18
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        den = 1.0 - T @ X[c0:c1].T
        own = (tid >= c0) & (tid < c1)  # self pairs excluded
        rows, cols = own.nonzero().squeeze(1), (tid[own] - c0)
        if KERNEL == 0:
            den[rows, cols] = float("inf")
            S += (Q[c0:c1] / den) @ X[c0:c1]
        else:
            lg = torch.log(den)
            lg[rows, cols] = 0.0
            S += lg @ Q[c0:c1]
    if KERNEL == 0:
        u_dir = (-1.0 / (4.0 * np.pi)) * torch.cross(T, S, dim=1)  # velocity
    else:
        u_dir = (-1.0 / (4.0 * np.pi)) * S  # stream function (LogPotentialKernel, prefactor 1)
    def rel(u):
        ut = torch.from_numpy(np.ascontiguousarray(u[idx])).to(dev).reshape(u_dir.shape)
        return float(torch.linalg.norm(ut - u_dir) / torch.linalg.norm(u_dir))

    e_tree = rel(u_tree)
    e_ref = rel(u_ref) if u_ref is not None else None
    out = {"value": e_tree, "reference_same_targets": e_ref,
           "targets": int(len(idx)), "seed": seed, "survey_reference_E_config4": 2.38e-6,
           "definition": "||u_tree - u_direct||_2 / ||u_direct||_2 over the sampled targets"}
    if e_ref is not None:
        # the two tree codes agree to ~1e-13 (parity), so E differs only in
        # rounding: "no worse" is judged to 1e-6 relative, as in the tests
        out["relative_difference"] = (e_tree - e_ref) / e_ref
        out["not_worse_than_reference"] = bool(e_tree <= e_ref * (1 + 1e-6))
    return out


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
    use_config(args.config)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
