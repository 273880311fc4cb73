"""The C-ABI library builds, loads without a GPU and exports every symbol the header declares."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "phg_b200.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(phg_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_05794_b200 import _native, build

    build.build()
    return _native.load()


def test_header_declares_entry_points():
    names = header_functions()
    assert "phg_trace" in names and "phg_field_create" in names and len(names) >= 12


def test_library_exports_every_header_symbol(lib):
    from paper_2604_05794_b200 import _native

    for name in header_functions():
        assert hasattr(lib, name), name
    assert set(header_functions()) == set(_native.EXPORTS)


def test_abi_version(lib):
    assert lib.phg_abi_version() == 2


def test_null_arguments_fail_cleanly_without_gpu(lib):
    from paper_2604_05794_b200 import _native

    assert lib.phg_field_create(None, None, None, 1, 1, 1, None, 1.0, None) == \
        _native.PHG_ERR_INVALID
    assert b"null" in lib.phg_last_error()
    total = ctypes.c_int64()
    assert lib.phg_trace(None, None, None, None, None, 0, None, None, None,
                         ctypes.byref(total), None) == _native.PHG_ERR_INVALID
    assert lib.phg_gather(None, None, 0, None) == _native.PHG_ERR_INVALID


def test_sm100a_cubin_embedded():
    import subprocess

    from paper_2604_05794_b200 import build

    out = subprocess.run(["cuobjdump", "--list-elf", build.OUT], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_params_mirror_validation():
    from paper_2604_05794_b200.errors import ConfigError
    from paper_2604_05794_b200.phg import PhgParams

    for bad in (dict(link_dist_mm=0.0), dict(link_angle_deg=95.0), dict(step_mm=-1.0),
                dict(occupancy_cap=0), dict(batch_size=0)):
        with pytest.raises(ConfigError):
            PhgParams(**bad)
    p = PhgParams()
    assert (p.step_mm, p.max_vertices, p.batch_size, p.occupancy_cap, p.probe_steps,
            p.min_support, p.coast_steps) == (1.0, 400, 16384, 16, 24, 0.05, 25)


def test_slab_row_bytes_matches_device_row_stride(monkeypatch):
    """phg.slab_row_bytes mirrors row_stride_doubles (phg_core.cuh): rows padded to 4 vertices
    (96 B), so the chunked drop-in sizes its slab exactly as the C ABI allocates it."""
    from paper_2604_05794_b200 import phg

    src = open(os.path.join(ROOT, "paper_2604_05794_b200", "csrc", "phg_core.cuh")).read()
    assert re.search(r"\(max_vertices \+ 3\) & ~3\) \* 3", src)
    for mv, want in ((1, 96), (4, 96), (5, 192), (400, 9600), (401, 9696)):
        assert phg.slab_row_bytes(phg.PhgParams(max_vertices=mv)) == want
    monkeypatch.setenv("PHG_SLAB_BUDGET_GB", "0.5")
    assert phg.slab_budget_bytes() == 1 << 29


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2604_05794_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|\"\"\"[\s\S]*?\"\"\"", "", src), f


def test_default_trace_kernels_do_not_spill():
    """The default trace kernels (every sampler mode, cap / no cap, the driver's recording
    traces) fit their register budget without local-memory spills: a spill is a silent
    performance regression (round 1 measured +11% for 70-94 B of spills)."""
    import subprocess

    from paper_2604_05794_b200 import build

    build.build()
    out = subprocess.run(["cuobjdump", "-res-usage", build.OUT], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    lines = out.stdout.splitlines()
    # CfgDefault (block signs) and CfgSparse (per-corner signs, bare occupancy flags)
    default = re.compile(r"trace_kernelINS_3CfgILi1ELi1ELi4ELi8ELi128ELb1ELi4ELb1ELi[12]EEE")
    seen = 0
    for i, ln in enumerate(lines):
        if "Function" in ln and default.search(ln):
            res = lines[i + 1]
            seen += 1
            reg = int(re.search(r"REG:(\d+)", res).group(1))
            assert "LOCAL:0" in res and "STACK:0" in res, (ln, res)
            assert reg <= 128, (ln, res)  # 4 CTAs of 128 threads per SM
    assert seen >= 12, seen


def test_round2_entry_points_validate_without_gpu(lib):
    """The round-2 entry points reject bad arguments with PHG_ERR_INVALID (no CUDA call is
    made), and the release build says it is not the checked build."""
    from paper_2604_05794_b200 import _native

    INV, STATE = _native.PHG_ERR_INVALID, _native.PHG_ERR_STATE
    rows = _native.Rows()
    assert lib.phg_trace_rows(None, None, None, None, None, 0, ctypes.byref(rows), None) == INV
    assert lib.phg_gather_to(None, None, None, None, 0, 0, None) == INV
    assert lib.phg_ipc_open(None, ctypes.byref(ctypes.c_void_p())) == INV
    assert lib.phg_ipc_alloc(-1, ctypes.byref(ctypes.c_void_p()), None) == INV
    origin = (ctypes.c_double * 3)(0, 0, 0)
    assert lib.phg_field_create_packed(None, 4, 4, 4, origin, 1.0, 1, 1.0, None) == INV
    out = ctypes.c_void_p()
    assert lib.phg_field_create_packed(ctypes.byref(out), 0, 4, 4, origin, 1.0, 1, 1.0,
                                       None) == INV
    assert lib.phg_field_packed(None, None, None, None, None) == INV
    assert lib.phg_field_packed_done(None, None) == INV
    assert lib.phg_is_checked_build() == 0
    v = ctypes.c_int64()
    assert lib.phg_debug_checks(ctypes.byref(v), None, None) == STATE
