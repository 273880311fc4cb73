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


@pytest.fixture(autouse=True)
def _checked_build_guard(request):
    """With PHG_CHECKED_LIB=1 (the checked build, our compute-sanitizer stand-in) every GPU
    test must leave zero device index-check violations and intact allocation canaries."""
    yield
    if os.environ.get("PHG_CHECKED_LIB") != "1" or request.node.get_closest_marker("gpu") is None:
        return
    import ctypes

    from paper_2604_05794_b200 import _native

    lib = _native.load()
    assert lib.phg_is_checked_build() == 1
    v, site, g = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _native.check(lib.phg_debug_checks(ctypes.byref(v), ctypes.byref(site), ctypes.byref(g)),
                  "phg_debug_checks")
    assert v.value == 0 and g.value == 0, (
        f"checked build: {v.value} device index-check violations (first site {site.value}), "
        f"{g.value} buffers with overwritten canaries {lib.phg_last_error().decode()}")
