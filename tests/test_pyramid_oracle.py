"""Pins of the LOD-pyramid oracle (P:71 2^3 mean, reading c12) -- CPU only."""
import numpy as np
import pytest

from conftest import read_golden
from oracle import pyramid_oracle as po
import workloads as wl


def test_golden_checkerboard():
    """0/1 checkerboard children -> 0.5; u16 0/65535 -> 32768 (round half up)."""
    rows = read_golden("pyramid_checkerboard.txt")
    for (dt, lo, hi), (expect,) in zip(rows[0::2], rows[1::2]):
        npdt = wl.gen.NP_DTYPE[dt]
        z, y, x = np.indices((2, 2, 2))
        vol = np.where((x + y + z) % 2 == 0, float(lo), float(hi)).astype(npdt)
        out = po.downsample(vol)
        assert out.shape == (1, 1, 1) and out.dtype == npdt
        assert float(out[0, 0, 0]) == float(expect)


@pytest.mark.parametrize("dtype", ["u8", "u16", "i16", "f32"])
def test_constant_stays_constant(dtype):
    """a constant volume is constant at every level (mean of constants)."""
    c = {"u8": 200, "u16": 54321, "i16": -777, "f32": 0.7}[dtype]
    vol = np.full((13, 10, 7), c, wl.gen.NP_DTYPE[dtype])
    for lev in po.pyramid(vol, 4):
        assert np.all(lev == vol.flat[0])


def test_dims_are_ceil_half():
    vol = np.zeros((13, 10, 7), np.uint16)
    dims = [lv.shape for lv in po.pyramid(vol, 4)]
    assert dims == [(7, 5, 4), (4, 3, 2), (2, 2, 1), (1, 1, 1)]


@pytest.mark.parametrize("dtype,shape", [("u8", (5, 6, 7)), ("u16", (9, 4, 11)),
                                         ("i16", (7, 7, 3)), ("u16", (8, 8, 8))])
def test_vectorised_equals_bruteforce(dtype, shape):
    """The vectorised int64 rule == a pure-Python per-voxel loop (odd dims, negatives)."""
    vol = wl.pyramid_volume(shape[2], shape[1], shape[0], dtype, seed=1)
    cur = vol
    for _ in range(3):
        a = po.downsample(cur)
        b = po.downsample_bruteforce(cur)
        assert a.dtype == b.dtype and np.array_equal(a, b)
        cur = a


def test_round_half_up_and_odd_border_counts():
    """Count-weighted mean at odd borders: a lone child passes through unchanged; i16 -0.5
    rounds up to 0, -1.5 to -1; max u16 never overflows."""
    v = np.array([[[3, 4, 9]]], np.uint8)            # nx=3: children {3,4} and {9}
    assert po.downsample(v).ravel().tolist() == [4, 9]  # (3+4)/2 = 3.5 -> 4
    v = np.array([[[-1, 0]]], np.int16)
    assert po.downsample(v).ravel().tolist() == [0]
    v = np.array([[[-1, -2]]], np.int16)
    assert po.downsample(v).ravel().tolist() == [-1]
    v = wl.pyramid_volume(5, 5, 5, "u16", 0, kind="max")
    assert np.all(po.downsample(v) == 65535)


def test_f32_fixed_order_mean():
    """f32: children summed in the fixed pairwise order, one division by the count."""
    vol = wl.pyramid_volume(4, 3, 2, "f32", seed=3)
    out = po.downsample(vol)
    c = [vol[z, y, x] for z in (0, 1) for y in (0, 1) for x in (0, 1)]   # (x fastest)
    s = np.float32(np.float32(np.float32(c[0] + c[1]) + np.float32(c[2] + c[3])) +
                   np.float32(np.float32(c[4] + c[5]) + np.float32(c[6] + c[7])))
    assert out[0, 0, 0] == np.float32(s / np.float32(8))
    # odd border column x=... (nx=4 even); y=2 row has only y-children {2}: cnt 4
    c = [vol[z, 2, x] for z in (0, 1) for x in (0, 1)]
    s = np.float32(np.float32(c[0] + c[1]) + np.float32(c[2] + c[3]))
    assert out[0, 1, 0] == np.float32(s / np.float32(4))
