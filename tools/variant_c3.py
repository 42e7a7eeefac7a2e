"""Time the config-3 (random cap) evaluation passes for each tuning build of
the library (make -C paper_2401_07361_b200/csrc variants), like
tools/variant_bench.py does for config 4.

    python tools/variant_c3.py
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, json, statistics, torch
sys.path.insert(0, '.')
import paper_2401_07361_b200 as ss
xyz, z, a = ss.make_random_cap(1 << 22, 5)
q = z * a
dev = torch.device('cuda', 0)
dx, dq = torch.from_numpy(xyz).to(dev), torch.from_numpy(q).to(dev)
out = torch.zeros((xyz.shape[0], 3), dtype=torch.float64, device=dev)
tree = ss.FaceTree(0)
tree.set_stream(torch.cuda.current_stream().cuda_stream)
cfg = ss.TraversalConfig(theta=0.7, n_threshold=64, degree=8, max_depth=10)
rows = []
for k in range(6):
    st = ss.TreecodeStats()
    ss.treecode_sum_device(tree, ss.BiotSavartKernel, cfg, dx.data_ptr(), dq.data_ptr(), xyz.shape[0], out.data_ptr(), stats=st)
    torch.cuda.synchronize()
    if k >= 2:
        rows.append((st.pp_pc_ms, st.cp_cc_fit_ms))
print(json.dumps(dict(zip(['pp_pc', 'fit'], [statistics.median(c) for c in zip(*rows)]))))
"""
libs = [os.path.join(ROOT, "paper_2401_07361_b200", "lib", "libspheresum_b200.so")]
libs += sorted(glob.glob(os.path.join(ROOT, "paper_2401_07361_b200", "lib", "variants", "*.so")))
for lib in libs:
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=dict(os.environ, SSUM_LIBRARY=lib),
                       capture_output=True, text=True)
    tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr.strip()[-300:]
    print(os.path.basename(lib), tail, flush=True)
