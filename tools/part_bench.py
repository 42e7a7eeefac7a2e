"""Device time of one rank's share of a config-4 evaluation at G parts:
every part's call is timed on this GPU in turn (after the first full call has
placed the cost-balanced cuts, each part bins, traverses and lists its own
targets only). The max over parts approximates one G-GPU step before the row
all-gather; nothing here waits on another rank.

    python tools/part_bench.py [G ...] [--phases] [--config c4|c5]

--phases adds each part's phase split (TreecodeStats of its last call);
--config c5: BASELINE config 5 (L10 mesh, N = 10,485,762, theta = 0.8), the
scaling sweep's own config (default c4: L9, theta = 0.7).
--shard-bin: sharded binning walk (dist.sharded_walk): each part's timed call
walks only its 1/G slot of the particles; the other slots' leaf keys and
leaves are copied in from a stash (device to device, the bytes one NCCL
all-gather of the keys would deliver over NVLink) before the evaluation.
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2401_07361_b200 as ss  # noqa: E402

phases = "--phases" in sys.argv
shard_bin = "--shard-bin" in sys.argv
config = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "c4"
level, theta = {"c4": (9, 0.7), "c5": (10, 0.8)}[config]
parts = [int(a) for a in sys.argv[1:] if not a.startswith("--") and a not in ("c4", "c5")] or [1, 2, 4, 8]
xyz, area = ss.make_icosa_mesh(level)
q = ss.rh4_vorticity(xyz) * area
n = xyz.shape[0]
dev = torch.device("cuda", 0)
d_xyz = torch.from_numpy(xyz).to(dev)
d_q = torch.from_numpy(q).to(dev)
d_out = torch.zeros((n, 3), dtype=torch.float64, device=dev)
cfg = ss.TraversalConfig(theta=theta, n_threshold=64, degree=8, max_depth=10)
res = {}
for G in parts:
    tree = ss.FaceTree(0)
    tree.set_stream(torch.cuda.current_stream().cuda_stream)
    per, split = [], []
    stash = None
    if shard_bin and G > 1:  # the full walk's keys / leaves: what the other ranks' slots hold
        from paper_2401_07361_b200.dist import _DeviceArray, slot_bounds

        ss.treecode_sum_device(tree, ss.BiotSavartKernel, cfg, d_xyz.data_ptr(), d_q.data_ptr(), n,
                               d_out.data_ptr())  # builds the tree
        m = -(-n // G)
        for r in range(G):
            a, b, _ = slot_bounds(n, G, r)
            kp, lp, _ = tree.bin_walk_shard(d_xyz.data_ptr(), n, a, b, G * m)
        keys = torch.as_tensor(_DeviceArray(kp, G * m, "<i8"), device=dev)
        leaf = torch.as_tensor(_DeviceArray(lp, G * m, "<i4"), device=dev)
        stash = (keys.clone(), leaf.clone())
        ss.treecode_sum_device(tree, ss.BiotSavartKernel, cfg, d_xyz.data_ptr(), d_q.data_ptr(), n,
                               d_out.data_ptr())

    def call(r, st=None):
        if stash is not None:
            a, b, m = slot_bounds(n, G, r)
            kp, lp, walked = tree.bin_walk_shard(d_xyz.data_ptr(), n, a, b, G * m)
            if walked:  # the all-gather's bytes: every other slot's rows
                keys = torch.as_tensor(_DeviceArray(kp, G * m, "<i8"), device=dev)
                leaf = torch.as_tensor(_DeviceArray(lp, G * m, "<i4"), device=dev)
                keys[:a].copy_(stash[0][:a])
                keys[b:n].copy_(stash[0][b:n])
                leaf[:a].copy_(stash[1][:a])
                leaf[b:n].copy_(stash[1][b:n])
        ss.treecode_sum_device(tree, ss.BiotSavartKernel, cfg, d_xyz.data_ptr(), d_q.data_ptr(), n,
                               d_out.data_ptr(), stats=st)

    for r in range(G):
        tree.set_partition(r, G)
        for _ in range(3):  # warm-up (the first call of part 0 places the cuts)
            call(r)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = ss.TreecodeStats()
        for _ in range(5):
            call(r, st)
        e1.record()
        torch.cuda.synchronize()
        per.append(e0.elapsed_time(e1) / 5)
        split.append({"bin": st.bin_seconds * 1e3 / 5, "trav": st.traversal_seconds * 1e3 / 5,
                      "up": st.upward_ms, "fit": st.cp_cc_fit_ms, "pp_pc": st.pp_pc_ms, "finish": st.finish_ms})
    res[G] = {"max_part_ms": max(per), "min_part_ms": min(per), "parts_ms": per}
    if phases:
        res[G]["phases_of_max_part"] = split[per.index(max(per))]
    print(json.dumps({"config": config, "n": n, "G": G, "shard_bin": bool(stash is not None), **res[G]}), flush=True)
