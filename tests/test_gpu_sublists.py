"""The subtree list builder (sublists.cu) against the global traversal path
(traversal.cu): the same tiles and ranges, so bitwise-identical results, on
static and moving particles, on meshes and on the dense random cap, with
small cut sizes that force block overflows and redo on the global path, and
with the reference for the PC-only mode and the log kernel."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(ss, xyz0, q, cfg, calls, mode, cmax=None, kernel=None, seed=7, step=3e-4):
    """Evaluations of a sequence of moving-particle states on one tree with
    the list builder selected by SSUM_SUB_LISTS (read when the tree makes its
    first plan)."""
    old = {k: os.environ.get(k) for k in ("SSUM_SUB_LISTS", "SSUM_SUB_CMAX")}
    if mode == "auto":  # measured choice between the builders
        os.environ.pop("SSUM_SUB_LISTS", None)
    else:
        os.environ["SSUM_SUB_LISTS"] = mode
    if cmax is not None:
        os.environ["SSUM_SUB_CMAX"] = str(cmax)
    try:
        tree = ss.FaceTree()
        rng = np.random.default_rng(seed)
        x = xyz0.copy()
        outs = []
        for k in range(calls):
            if k >= 2:
                x = x + step * rng.standard_normal(x.shape)
                x /= np.linalg.norm(x, axis=1, keepdims=True)
            outs.append(ss.treecode_sum(kernel or ss.BiotSavartKernel, x, q, cfg, tree=tree))
        return outs
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _same(a, b):
    return all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("level,deg,theta", [(5, 4, 0.7), (7, 8, 0.7), (6, 8, 0.8), (6, 6, 0.35)])
def test_subtree_lists_bitwise_global(ss, mesh_fixture, level, deg, theta):
    xyz, q, _ = mesh_fixture(level)
    c = ss.TraversalConfig(theta=theta, n_threshold=64, degree=deg, max_depth=10)
    assert _same(_run(ss, xyz, q, c, 5, "1"), _run(ss, xyz, q, c, 5, "0"))


@pytest.mark.parametrize("cmax", [64, 1024, 4096])
def test_subtree_lists_cut_sizes(ss, mesh_fixture, cmax):
    """Tiny cuts (many blocks, long paths) and cuts that outgrow a block's
    shared memory (kFlagListsRedo: the evaluation is redone on the global
    path and the cut halved) give the same bits."""
    xyz, q, _ = mesh_fixture(7)
    c = ss.TraversalConfig(theta=0.7, n_threshold=64, degree=8, max_depth=10)
    assert _same(_run(ss, xyz, q, c, 4, "1", cmax=cmax), _run(ss, xyz, q, c, 4, "0"))


def test_subtree_lists_random_cap(ss):
    xyz, zeta, area = ss.make_random_cap(1 << 18, 5)
    q = zeta * area
    c = ss.TraversalConfig(theta=0.7, n_threshold=64, degree=8, max_depth=10)
    # points ~2e-4 rad apart in the cap: small steps, no new near-duplicates
    assert _same(_run(ss, xyz, q, c, 4, "1", step=1e-8), _run(ss, xyz, q, c, 4, "0", step=1e-8))


def test_subtree_lists_pc_only_and_log(ss, ol, mesh_fixture):
    xyz, q, _ = mesh_fixture(6)
    c = ss.TraversalConfig(theta=0.7, n_threshold=64, degree=6, max_depth=10, pc_only=True)
    assert _same(_run(ss, xyz, q, c, 3, "1"), _run(ss, xyz, q, c, 3, "0"))
    c2 = ss.TraversalConfig(theta=0.7, n_threshold=64, degree=6, max_depth=10)
    a = _run(ss, xyz, q, c2, 3, "1", kernel=ss.LogPotentialKernel)
    assert _same(a, _run(ss, xyz, q, c2, 3, "0", kernel=ss.LogPotentialKernel))
    ur, _ = ol.ref_treecode(1, xyz, q, 0.7, 64, 6, 10, os.cpu_count() or 1)
    assert ol.rel_l2(a[0], ur) < 1e-10


def test_subtree_lists_guard_band(ss, mesh_fixture, monkeypatch):
    """A wide MAC guard band: the screen defers to the exact path, pairs go
    to the host, the subtree builder redoes the call with the decisions."""
    monkeypatch.setenv("SSUM_MAC_BAND", "0.05")
    xyz, q, _ = mesh_fixture(6)
    c = ss.TraversalConfig(theta=0.7, n_threshold=64, degree=4, max_depth=10)
    assert _same(_run(ss, xyz, q, c, 3, "1"), _run(ss, xyz, q, c, 3, "0"))


@pytest.mark.parametrize("which", ["mesh", "cap"])
def test_subtree_lists_auto_choice(ss, mesh_fixture, which):
    """Default mode: the first evaluations time both builders (on the cap the
    subtree blocks overflow and the call is redone on the global path) and
    keep the faster; every call's result is bitwise the global path's."""
    if which == "mesh":
        xyz, q, _ = mesh_fixture(7)
    else:
        xyz, zeta, area = ss.make_random_cap(1 << 18, 5)
        q = zeta * area
    c = ss.TraversalConfig(theta=0.7, n_threshold=64, degree=8, max_depth=10)
    step = 3e-4 if which == "mesh" else 1e-8
    assert _same(_run(ss, xyz, q, c, 8, "auto", step=step), _run(ss, xyz, q, c, 8, "0", step=step))
