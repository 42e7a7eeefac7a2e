"""Time the config-4 evaluation passes for each tuning build of the library
(make -C paper_2401_07361_b200/csrc variants). One subprocess per library.

    python tools/variant_bench.py [level | c3 | c5]
"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, json, statistics, torch
sys.path.insert(0, '.')
import paper_2401_07361_b200 as ss
arg = sys.argv[1]
theta = 0.7
if arg == 'c3':
    xyz, zeta, area = ss.make_random_cap(1 << 22, 5)
    q = zeta * area
else:
    if arg == 'c5':
        arg, theta = '10', 0.8
    xyz, area = ss.make_icosa_mesh(int(arg))
    q = ss.rh4_vorticity(xyz) * area
dev = torch.device('cuda', 0)
dx, dq = torch.from_numpy(xyz).to(dev), torch.from_numpy(q).to(dev)
out = torch.zeros((xyz.shape[0], 3), dtype=torch.float64, device=dev)
tree = ss.FaceTree(0)
tree.set_stream(torch.cuda.current_stream().cuda_stream)
cfg = ss.TraversalConfig(theta=theta, n_threshold=64, degree=8, max_depth=10)
rows = []
for k in range(8):
    st = ss.TreecodeStats()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    ss.treecode_sum_device(tree, ss.BiotSavartKernel, cfg, dx.data_ptr(), dq.data_ptr(), xyz.shape[0], out.data_ptr(), stats=st)
    e1.record(); torch.cuda.synchronize()
    if k >= 3:
        rows.append((e0.elapsed_time(e1), st.pp_pc_ms, st.cp_cc_fit_ms, st.upward_ms, st.finish_ms,
                     st.bin_seconds * 1e3, st.traversal_seconds * 1e3))
med = [statistics.median(c) for c in zip(*rows)]
res = dict(zip(['step', 'pp_pc', 'fit', 'up', 'finish', 'bin', 'trav'], med))
# relative L2 of this library's velocities against the first (default) library's
import os, numpy as np
u = out.cpu().numpy()
ref = sys.argv[2]
if os.path.exists(ref):
    b = np.load(ref)
    res['rel_l2_vs_default'] = float(np.linalg.norm(u - b) / np.linalg.norm(b))
else:
    np.save(ref, u)
print(json.dumps(res))
"""


def main():
    lvl = sys.argv[1] if len(sys.argv) > 1 else "9"
    ref = os.path.join("/tmp", f"variant_default_{lvl}.npy")
    if os.path.exists(ref):
        os.remove(ref)
    libs = [os.path.join(ROOT, "paper_2401_07361_b200", "lib", "libspheresum_b200.so")]
    libs += sorted(glob.glob(os.path.join(ROOT, "paper_2401_07361_b200", "lib", "variants", "*.so")))
    for lib in libs:
        env = dict(os.environ, SSUM_LIBRARY=lib)
        r = subprocess.run([sys.executable, "-c", CHILD, lvl, ref], cwd=ROOT, env=env, capture_output=True, text=True)
        tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr.strip()[-300:]
        print(os.path.basename(lib), tail, flush=True)


if __name__ == "__main__":
    main()
