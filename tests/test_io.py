"""Wire formats: STND encoder and OOVL decoder on the GPU, byte-compatible
with files the reference itself wrote (tests/golden/io_*)."""

import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN, load_case

STND = os.path.join(GOLDEN, "io_driver_sparse40.stnd")
OOVL = os.path.join(GOLDEN, "io_sparse24.oovl")


def stnd_oracle(offsets, verts):
    """Restatement of strands.write_strands (strands.py:63-69) -- test oracle."""
    out = [struct.pack("<II", 0x444E5453, len(offsets) - 1)]
    for i in range(len(offsets) - 1):
        v = np.asarray(verts[offsets[i]:offsets[i + 1]], dtype="<f4")
        out.append(struct.pack("<I", len(v)))
        out.append(v.tobytes())
    return b"".join(out)


def test_stnd_oracle_matches_reference_file():
    z = np.load(os.path.join(GOLDEN, "driver_sparse40.npz"))
    assert stnd_oracle(z["offsets"], z["verts"]) == open(STND, "rb").read()


@pytest.mark.gpu
def test_stnd_gpu_encoder_matches_reference_file():
    from paper_2604_05794_b200 import io

    z = np.load(os.path.join(GOLDEN, "driver_sparse40.npz"))
    assert io.stnd_bytes(z["offsets"], z["verts"]) == open(STND, "rb").read()
    assert io.stnd_bytes(np.zeros(1, np.int64), np.zeros((0, 3))) == struct.pack("<II",
                                                                                 0x444E5453, 0)


@pytest.mark.gpu
def test_oovl_gpu_decoder_builds_identical_field():
    """Field from the reference-written OOVL == field packed from the original arrays:
    the sampler returns bitwise-identical results on both."""
    import ctypes

    from paper_2604_05794_b200 import _native, io
    from paper_2604_05794_b200.volume import DeviceField

    c = load_case(os.path.join(GOLDEN, "sample_sparse24.npz"))
    f_file, hdr = io.read_volume_device(OOVL)
    assert hdr["dims"] == c.occ.shape
    assert np.array_equal(hdr["origin"], np.asarray(c.origin, np.float32).astype(np.float64))
    f_arr = DeviceField(hdr["origin"], hdr["voxel_size"], c.occ, c.ori)
    lib = _native.load()
    outs = []
    for f in (f_file, f_arr):
        n = len(c.pts)
        dirs, has, sup = np.zeros((n, 3)), np.zeros(n, np.uint8), np.zeros(n)
        _native.check(lib.phg_sample(f.handle, c.pts.ctypes.data, c.prev.ctypes.data, n,
                                     dirs.ctypes.data, has.ctypes.data, sup.ctypes.data, None),
                      "phg_sample")
        outs.append((dirs, has, sup))
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    assert outs[0][1].any() and not outs[0][1].all()
    del ctypes


@pytest.mark.gpu
def test_oovl_truncated_payload_is_data_error(tmp_path):
    from paper_2604_05794_b200 import io
    from paper_2604_05794_b200.errors import DataError

    raw = open(OOVL, "rb").read()
    p = tmp_path / "bad.oovl"
    p.write_bytes(raw[:-12])
    with pytest.raises(DataError):
        io.read_volume_device(str(p))
