"""NDIV volume I/O and synthetic-input helpers of the B200 package (SURVEY.md
§8(f) row f2) against files and values written by the reference itself
(tests/golden/ndiv/*, tests/golden/synth.npz, made by make_golden.py io).
Host-side only: these run without a GPU (the library loads, no kernels)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

vk = pytest.importorskip("paper_2510_14143_b200")

NDIV = os.path.join(GOLDEN, "ndiv")
NAMES = sorted(f[:-5] for f in os.listdir(NDIV) if f.endswith(".ndiv"))


def _manifest():
    return load_golden(os.path.join(NDIV, "manifest.npz"))


@pytest.mark.parametrize("name", NAMES)
def test_read_reference_written(name):
    m = _manifest()
    v = vk.read_volume(os.path.join(NDIV, name + ".ndiv"))
    want = m[name]
    assert v.values.dtype == want.dtype and v.values.shape == want.shape
    assert np.array_equal(v.values, want)
    sp = m[name + "__spacing"]
    assert (v.spacing is None) == (sp.size == 0)
    if v.spacing is not None:
        assert v.spacing == tuple(sp)  # exact doubles


@pytest.mark.parametrize("name", NAMES)
def test_write_is_bytewise_reference(name, tmp_path):
    """write_volume . read_volume is bitwise identity (io.hpp:30) and our
    writer emits exactly the reference's header bytes."""
    src = os.path.join(NDIV, name + ".ndiv")
    v = vk.read_volume(src)
    out = tmp_path / "w.ndiv"
    vk.write_volume(out, v.values, v.spacing)
    assert out.read_bytes() == open(src, "rb").read()


def test_header_info_and_offsets():
    info = vk.volume_info(os.path.join(NDIV, "f32_zyx_spacing.ndiv"))
    assert info.shape == (2, 2, 2) and info.dtype == np.float32 and info.spacing == (0.29, 0.065, 0.065)


def test_failure_modes(tmp_path):
    """The reference's own failure-mode test (tests/test_io_synth.cpp:65-105)."""
    bad = tmp_path / "bad.ndiv"
    bad.write_bytes(b"JUNKJUNKJUNK")
    with pytest.raises(vk.BadMagic, match="is not an NDIV volume"):
        vk.read_volume(bad)
    ok = tmp_path / "ok.ndiv"
    vk.write_volume(ok, np.array([[1, 2], [3, 4]], np.float32))
    data = ok.read_bytes()
    short = tmp_path / "short.ndiv"
    short.write_bytes(data[:-7])
    with pytest.raises(vk.TruncatedPayload, match="expected 16 payload bytes"):
        vk.read_volume(short)
    long = tmp_path / "long.ndiv"
    long.write_bytes(data + b"extra")
    with pytest.raises(vk.TruncatedPayload, match="trailing bytes after payload"):
        vk.read_volume(long)
    hdr = tmp_path / "hdr.ndiv"
    hdr.write_bytes(data[:9] + b"?" + data[10:])
    with pytest.raises(vk.HeaderMismatch):
        vk.read_volume(hdr)
    with pytest.raises(vk.Error, match="cannot open"):
        vk.read_volume(tmp_path / "missing.ndiv")
    # header-level rules of read_volume (io.cpp:103-119)
    def with_header(h: bytes, payload=b""):
        p = tmp_path / "h.ndiv"
        p.write_bytes(b"NDIV" + len(h).to_bytes(4, "little") + h + payload)
        return p
    with pytest.raises(vk.HeaderMismatch, match="header needs elem, shape and axes"):
        vk.read_volume(with_header(b'{"elem":"f32","shape":[1]}', b"\0" * 4))
    with pytest.raises(vk.HeaderMismatch, match="unknown element kind 'f64'"):
        vk.read_volume(with_header(b'{"axes":"X","elem":"f64","shape":[1]}', b"\0" * 8))
    with pytest.raises(vk.HeaderMismatch, match="axes string length must equal rank"):
        vk.read_volume(with_header(b'{"axes":"YX","elem":"f32","shape":[1]}', b"\0" * 4))
    with pytest.raises(vk.HeaderMismatch, match="truncated header"):
        p = tmp_path / "t.ndiv"
        p.write_bytes(b"NDIV" + (100).to_bytes(4, "little") + b"{}")
        vk.read_volume(p)
    with pytest.raises(vk.HeaderMismatch, match="missing header length"):
        p = tmp_path / "m.ndiv"
        p.write_bytes(b"NDIV\x01")
        vk.read_volume(p)
    # spacing is attached after the payload checks (NdImage::with_spacing)
    with pytest.raises(vk.ShapeMismatch, match="spacing needs one entry per axis"):
        vk.read_volume(with_header(b'{"axes":"X","elem":"f32","shape":[1],"spacing":[1.0,2.0]}', b"\0" * 4))
    # whitespace and key order do not matter to the reader
    p = with_header(b' { "shape" : [ 2 ] , "elem" : "u16", "axes" : "X" } ', b"\x01\x00\x02\x00")
    assert np.array_equal(vk.read_volume(p).values, np.array([1, 2], np.uint16))


def test_write_rank_and_dtype_errors(tmp_path):
    with pytest.raises(vk.HeaderMismatch, match="unsupported rank 5"):
        vk.write_volume(tmp_path / "r5.ndiv", np.zeros((1, 1, 1, 1, 1), np.float32))
    with pytest.raises(vk.Error):
        vk.write_volume(tmp_path / "f64.ndiv", np.zeros((2,), np.float64))
    with pytest.raises(vk.Error, match="cannot open"):
        vk.write_volume(tmp_path / "no" / "such" / "dir.ndiv", np.zeros((2,), np.float32))


def test_gaussian_psf_matches_reference():
    g = load_golden(os.path.join(GOLDEN, "synth.npz"))
    cases = {"psf_a": ((9, 17, 17), [1.0, 2.0, 2.0]), "psf_b": ((5, 5), [1.5]), "psf_c": ((7,), [0.0]),
             "psf_d": ((3, 9, 5), [0.7, 2.2, 1.1])}
    for k, (shape, sig) in cases.items():
        assert np.array_equal(vk.gaussian_psf(shape, sig), g[k]), k
    with pytest.raises(vk.EvenExtent, match=r"gaussian_psf needs odd extents, got \[4,5\]"):
        vk.gaussian_psf((4, 5), [1.0])
    with pytest.raises(vk.ShapeMismatch, match="one sigma per axis"):
        vk.gaussian_psf((3, 5, 5), [1.0, 2.0])
