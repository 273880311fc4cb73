import glob
import json
import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built libphg_b200.so")


class Case(SimpleNamespace):
    """One golden fixture: inputs + the reference's outputs (see tests/golden/make_golden.py)."""

    @property
    def vol(self):
        return SimpleNamespace(origin=self.origin, voxel_size=float(self.voxel_size),
                               dims=self.occ.shape, occ=self.occ, ori=self.ori)


def load_case(path):
    z = np.load(path)
    d = {k: z[k] for k in z.files}
    d["name"] = os.path.basename(path)[:-4]
    if "params" in d:
        d["params"] = SimpleNamespace(**json.loads(str(d["params"])))
    return Case(**d)


def trace_cases():
    return sorted(glob.glob(os.path.join(GOLDEN, "trace_*.npz")))


def csr_equal(off_a, v_a, off_b, v_b):
    return np.array_equal(off_a, off_b) and np.array_equal(v_a, v_b)


@pytest.fixture(scope="session")
def oracle_c():
    from oracle import phg_oracle_c

    phg_oracle_c.build()
    return phg_oracle_c
