import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


DX = 25.0 / 64.0
DT = (1.0 / 48.0) / 36.0


def elastic_setup(flip_blend=0.0):
    """Same scene parameters as tests/golden/make_golden.py::elastic_setup."""
    from paper_2111_00699_b200 import BoundaryBox, Material, SimParams
    material = Material.fixed_corotated(2.0, 1.0e5, 0.3)
    params = SimParams(dx=DX, dt=DT, flip_blend=flip_blend)
    boundary = BoundaryBox((8 * DX,) * 3, (40 * DX,) * 3, mode="slip")
    return material, params, boundary


def fluid_setup(**kw):
    from paper_2111_00699_b200 import BoundaryBox, Material, SimParams
    material = Material.fluid(1.0, 1.0e5, 7.0)
    params = SimParams(dx=0.5, dt=2.0e-4, **kw)
    boundary = BoundaryBox((4.0,) * 3, (20.0,) * 3, mode="sticky")
    return material, params, boundary
