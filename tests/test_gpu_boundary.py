"""The reference-facing boundary beyond treecode_sum, through the C-ABI on the
GPU: compute_proxy_weights, the per-interaction entry points' cost, the MAC
guard band (host-made decisions inside it), ConditioningError's rcond,
TreecodeStats accumulation, and stream ordering with torch's default stream."""
import os
import time

import numpy as np
import pytest

import oracle_lib as ol

pytestmark = pytest.mark.gpu


def cfg(ss, theta=0.7, nt=64, deg=8, md=10):
    return ss.TraversalConfig(theta=theta, n_threshold=nt, degree=deg, max_depth=md)


@pytest.mark.parametrize("deg", [4, 8])
def test_compute_proxy_weights_matches_reference(ss, ol, mesh_fixture, deg):  # treecode.cpp:79-91
    xyz, q, _ = mesh_fixture(5)
    t = ss.FaceTree()
    t.bin_particles(xyz, 64, 10)
    r = ol.RefTree()
    r.bin(xyz, 64, 10)
    e = r.export()
    sizes = e["bin_offsets"][1:] - e["bin_offsets"][:-1]
    rng = np.random.default_rng(deg)
    nodes = [0, 7] + list(rng.choice(np.flatnonzero(sizes > 0), 6, replace=False))
    nodes.append(int(np.flatnonzero(sizes == 0)[0]) if (sizes == 0).any() else 1)
    for node in nodes:
        w = ss.compute_proxy_weights(t, int(node), ss.SBBBasis(deg), xyz, q)
        wr = r.proxy_weights(deg, xyz, q, int(node))
        scale = max(np.abs(wr).max(), 1e-300)
        assert np.abs(w - wr).max() <= 1e-13 * scale, node


def test_eval_interaction_cost_is_per_interaction(ss, mesh_fixture):
    """eval_pp on one leaf pair must not scale with N (O(|t| |s|)): a PP call
    on the L9 mesh costs about what it costs on L5."""
    def one(level):
        xyz, q, _ = mesh_fixture(level)
        t = ss.FaceTree()
        t.bin_particles(xyz, 64, 10)
        lst = ss.dual_traversal_array(t, cfg(ss, deg=4))
        pp = lst[lst[:, 2] == 0][0]
        field = np.zeros((xyz.shape[0], 3))
        it = ss.Interaction(int(pp[0]), int(pp[1]), ss.InteractionKind.PP)
        ss.eval_pp(ss.BiotSavartKernel, t, it, xyz, q, field)  # warm
        t0 = time.perf_counter()
        for _ in range(5):
            ss.eval_pp(ss.BiotSavartKernel, t, it, xyz, q, field)
        return (time.perf_counter() - t0) / 5

    small, big = one(5), one(9)
    assert big < 20 * small + 5e-3, (small, big)


@pytest.mark.parametrize("band", [2e-2, 2e-1])
def test_mac_guard_band_decisions_match_reference(ss, ol, mesh_fixture, band, monkeypatch):
    """Force a wide guard band so that many MAC decisions are made on the host
    (glibc atan2, the reference's expressions) and the traversal is redone:
    the list must still be the reference's, bit for bit, and the velocities
    must keep parity."""
    monkeypatch.setenv("SSUM_MAC_BAND", str(band))
    xyz, q, _ = mesh_fixture(6)
    c = cfg(ss, deg=4)
    t = ss.FaceTree()
    st = ss.TreecodeStats()
    u = ss.treecode_sum(ss.BiotSavartKernel, xyz, q, c, tree=t, stats=st)
    assert st.mac_host_decisions > 0
    mine = ss.dual_traversal_array(t, c)
    r = ol.RefTree()
    r.bin(xyz, 64, 10)
    ref = r.traversal(0.7, 64, 4, 10)
    assert np.array_equal(mine, ref)
    ur, _ = ol.ref_treecode(0, xyz, q, 0.7, 64, 4, 10, os.cpu_count() or 1)
    assert ol.rel_l2(u, ur) < 1e-10
    # a second call reuses the host decisions (nothing new to decide)
    st2 = ss.TreecodeStats()
    ss.treecode_sum(ss.BiotSavartKernel, xyz, q, c, tree=t, stats=st2)
    assert st2.mac_host_decisions == st.mac_host_decisions


def test_default_band_makes_no_host_decisions_on_mesh(ss, mesh_fixture):
    xyz, q, _ = mesh_fixture(6)
    st = ss.TreecodeStats()
    ss.treecode_sum(ss.BiotSavartKernel, xyz, q, cfg(ss, deg=4), tree=ss.FaceTree(), stats=st)
    assert st.mac_host_decisions == 0


def test_conditioning_error_carries_rcond(ss, mesh_fixture):  # sbb.cpp:89-93, errors.hpp:22-27
    xyz, q, _ = mesh_fixture(4)
    with pytest.raises(ss.ConditioningError) as e:
        ss.treecode_sum(ss.BiotSavartKernel, xyz, q, cfg(ss, nt=8, deg=16), tree=ss.FaceTree())
    assert 0.0 <= e.value.rcond <= 1e-12


def test_stats_accumulate_like_reference(ss, mesh_fixture):  # treecode.cpp:296,407-411
    xyz, q, _ = mesh_fixture(5)
    t = ss.FaceTree()
    st = ss.TreecodeStats()
    ss.treecode_sum(ss.BiotSavartKernel, xyz, q, cfg(ss, deg=4), tree=t, stats=st)
    one = list(st.interaction_counts)
    s1 = st.eval_seconds
    ss.treecode_sum(ss.BiotSavartKernel, xyz, q, cfg(ss, deg=4), tree=t, stats=st)
    assert st.interaction_counts == [2 * v for v in one]
    assert st.eval_seconds > s1


def test_default_stream_is_ordered(ss, mesh_fixture):
    """set_stream(0) (torch's legacy default stream) must order the library's
    work after torch's: inputs written by torch right before the call are the
    ones evaluated."""
    import torch

    xyz, q, _ = mesh_fixture(6)
    n = xyz.shape[0]
    t = ss.FaceTree()
    t.set_stream(torch.cuda.current_stream().cuda_stream)  # 0 on the default stream
    d_xyz = torch.from_numpy(xyz).cuda()
    d_q = torch.zeros(n, dtype=torch.float64, device="cuda")
    out = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
    ref = ss.treecode_sum(ss.BiotSavartKernel, xyz, q, cfg(ss, deg=4), tree=ss.FaceTree())
    for _ in range(3):
        big = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
        big = big @ big  # keep the default stream busy
        d_q.copy_(torch.from_numpy(q).cuda(non_blocking=True) + 0.0 * big[0, 0])
        ss.treecode_sum_device(t, ss.BiotSavartKernel, cfg(ss, deg=4), d_xyz.data_ptr(), d_q.data_ptr(), n,
                               out.data_ptr())
        torch.cuda.synchronize()
        assert ol.rel_l2(out.cpu().numpy(), ref) < 1e-13


def test_partitioned_host_call_keeps_other_rows(ss, mesh_fixture):
    """A partitioned host-pointer call computes only its part's rows; every
    other row of the caller's buffer must come back as it was."""
    xyz, q, _ = mesh_fixture(6)
    n = xyz.shape[0]
    c = cfg(ss, deg=4)
    full = ss.treecode_sum(ss.BiotSavartKernel, xyz, q, c, tree=ss.FaceTree())
    t = ss.FaceTree()
    t.set_partition(1, 3)
    sentinel = np.full((n, 3), 7.25)
    out = ss.treecode_sum(ss.BiotSavartKernel, xyz, q, c, tree=t, out=sentinel.copy())
    p0, p1 = t.partition_range()
    perm = t.perm()
    mine = np.zeros(n, bool)
    mine[perm[p0:p1]] = True
    assert 0 < mine.sum() < n
    assert np.array_equal(out[mine], full[mine])
    assert np.all(out[~mine] == 7.25)
