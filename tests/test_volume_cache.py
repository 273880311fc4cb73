"""field_for's device-field cache (volume.py): lifetime tied to the volume, bounded for
volumes that cannot be weakly referenced, content changes detected.  CPU-only: the device
field is replaced by a recording stand-in."""

import gc
from types import SimpleNamespace

import numpy as np
import pytest

from paper_2604_05794_b200 import volume


class FakeField:
    live = []

    def __init__(self, origin, voxel_size, occ, ori, stream=0):
        self.closed = False
        FakeField.live.append(self)

    def close(self):
        self.closed = True


@pytest.fixture
def fake(monkeypatch):
    FakeField.live = []
    monkeypatch.setattr(volume, "DeviceField", FakeField)
    volume.invalidate()
    yield FakeField
    volume.invalidate()


def _vol(n=8, cls=volume.OOVolume):
    v = volume.OOVolume.empty((0, 0, 0), 2.0, (n, n, n))
    v.occ[2:5, 2:5, :] = True
    v.ori[..., 2] = v.occ
    if cls is SimpleNamespace:
        return SimpleNamespace(origin=v.origin, voxel_size=v.voxel_size, dims=v.dims,
                               occ=v.occ, ori=v.ori)
    return v


def test_cached_while_alive_and_freed_with_the_volume(fake):
    v = _vol()
    f1 = volume.field_for(v)
    assert volume.field_for(v) is f1 and len(fake.live) == 1
    del v
    gc.collect()
    assert f1.closed and not volume._CACHE


def test_in_place_edit_is_detected(fake):
    v = _vol()
    f1 = volume.field_for(v)
    v.ori[3, 3, 3, 0] = 0.5  # small buffer: hashed in full
    f2 = volume.field_for(v)
    assert f2 is not f1 and f1.closed
    v.occ[0, 0, 0] = True
    f3 = volume.field_for(v)
    assert f3 is not f2 and f2.closed and volume.field_for(v) is f3


def test_strong_lru_is_bounded(fake):
    vols = [_vol(cls=SimpleNamespace) for _ in range(4)]  # not weak-referenceable
    fields = [volume.field_for(v) for v in vols]
    assert sum(1 for e in volume._CACHE.values() if e[2] is not None) == 2
    assert fields[0].closed and fields[1].closed
    assert not fields[2].closed and not fields[3].closed
    assert volume.field_for(vols[3]) is fields[3]


def test_invalidate_drops_entry(fake):
    v = _vol()
    f1 = volume.field_for(v)
    volume.invalidate(v)
    assert f1.closed and volume.field_for(v) is not f1
