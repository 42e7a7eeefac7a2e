import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ss():
    import paper_2401_07361_b200 as m

    m.load_library()
    return m


@pytest.fixture(scope="session")
def ol():
    import oracle_lib as m

    if not m.ref_available():
        pytest.skip("oracle/_ref not built")
    return m


@pytest.fixture(autouse=True)
def _fresh_default_tree():
    """The module-level default FaceTree keeps node geometry across calls
    (reference FaceTree semantics); give every test a fresh one so results
    compare against the reference's fresh trees."""
    yield
    import paper_2401_07361_b200 as m

    for t in m._DEFAULT_TREES.values():
        t.close()
    m._DEFAULT_TREES.clear()


@pytest.fixture(scope="session")
def tree(ss):
    t = ss.FaceTree(0)
    yield t
    t.close()


_FIX = {}


@pytest.fixture(scope="session")
def mesh_fixture(ss):
    """(xyz, q, area) for a BASELINE mesh config: RH4 field, Voronoi areas."""

    def get(level):
        if level not in _FIX:
            xyz, a = ss.make_icosa_mesh(level)
            _FIX[level] = (xyz, ss.rh4_vorticity(xyz) * a, a)
        return _FIX[level]

    return get
