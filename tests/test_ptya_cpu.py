"""PTYA container (proj/src/io.cpp:80-207) without a GPU: our writer and
reader against the reference's own (compiled from io.cpp into oracle/_ref),
and the library's header validation (pdd_ptya_header) against the
reference's reader on malformed files -- same accept/reject decision and the
same byte offset in the FormatError message."""
import os
import re
import struct

import numpy as np
import pytest

from oracle import ref_lib as R
from paper_2011_00162_b200 import _lib as L
from paper_2011_00162_b200 import ptya

needs_ref_io = pytest.mark.skipif(not R.has_io(), reason="oracle/_ref without the reference's io.cpp")


@needs_ref_io
def test_writer_reader_round_trips_with_the_reference(tmp_path):
    rng = np.random.default_rng(3)
    fr = rng.random((5, 8, 8))
    cx = rng.standard_normal((6, 7)) + 1j * rng.standard_normal((6, 7))
    re_ = rng.standard_normal((4, 9))
    ptya.write_frames(tmp_path / "a.ptya", fr)
    ptya.write_array(tmp_path / "b.ptya", cx)
    ptya.write_array(tmp_path / "c.ptya", re_)
    assert np.array_equal(R.read_array(tmp_path / "a.ptya", "frames"), fr)
    assert np.array_equal(R.read_array(tmp_path / "b.ptya", "complex"), cx)
    assert np.array_equal(R.read_array(tmp_path / "c.ptya", "real"), re_)
    R.write_frames(tmp_path / "d.ptya", fr)
    assert open(tmp_path / "d.ptya", "rb").read() == open(tmp_path / "a.ptya", "rb").read()  # byte-identical
    assert np.array_equal(ptya.read_frames(tmp_path / "d.ptya"), fr)


def _bad_files(tmp_path):
    good = b"PTYA" + struct.pack("<HHH", 1, 1, 3) + struct.pack("<QQQ", 2, 4, 4) + np.ones(32).tobytes()
    cases = {
        "magic": b"PTYB" + good[4:],
        "version": good[:4] + struct.pack("<H", 2) + good[6:],
        "dtype": good[:6] + struct.pack("<H", 2) + good[8:],
        "ndim": good[:8] + struct.pack("<H", 5) + good[10:],
        "zerodim": good[:10] + struct.pack("<Q", 0) + good[18:],
        "hugedim": good[:10] + struct.pack("<Q", (1 << 32) + 1) + good[18:],
        "short_header": good[:20],
        "empty": b"",
    }
    out = {}
    for k, b in cases.items():
        p = tmp_path / f"{k}.ptya"
        p.write_bytes(b)
        out[k] = p
    return out


@needs_ref_io
def test_header_validation_matches_the_reference_reader(tmp_path):
    for name, p in _bad_files(tmp_path).items():
        with pytest.raises(R.RefError) as ref_err:
            R.read_array(p, "frames")
        with pytest.raises(L.FormatError) as our_err:
            ptya.header(p, ptya.F64)
        off = lambda s: re.search(r"byte offset (\d+)", str(s)).group(1)  # noqa: E731
        assert ref_err.value.code == 6, name
        assert off(ref_err.value) == off(our_err.value), (name, str(ref_err.value), str(our_err.value))


@needs_ref_io
def test_payload_size_errors_match_the_reference_reader(tmp_path):
    fr = np.ones((3, 4, 4))
    ptya.write_frames(tmp_path / "ok.ptya", fr)
    b = (tmp_path / "ok.ptya").read_bytes()
    (tmp_path / "short.ptya").write_bytes(b[:-8])
    (tmp_path / "long.ptya").write_bytes(b + b"\0" * 8)
    for name in ("short", "long"):
        with pytest.raises(R.RefError) as ref_err:
            R.read_array(tmp_path / f"{name}.ptya", "frames")
        with pytest.raises(L.FormatError) as our_err:
            ptya.read_frames(tmp_path / f"{name}.ptya")
        assert ref_err.value.code == 6
        assert ("truncated" in str(ref_err.value)) == ("truncated" in str(our_err.value))


@needs_ref_io
def test_reference_dataset_directory_loads(tmp_path):
    from paper_2011_00162_b200 import cli

    N, s, step = 40, 8, 4
    sample, probe, pin = R.toy(N, s, step, 5)
    f = R.simulate_frames(probe, sample, step)
    R.write_dataset(tmp_path / "ds", N, N, s, step, f, probe, pin=pin, sample=sample)
    ds = cli.load_dataset(str(tmp_path / "ds"))
    g = ds["geometry"]
    assert (g.frame_side, g.step, g.image_height, g.image_width, g.grid_rows, g.grid_cols) == (s, step, N, N, 9, 9)
    assert np.array_equal(g.positions, R.plan(R.plan_spec(N, N, s, step)).positions)
    assert np.array_equal(ds["probe"], probe) and np.array_equal(ds["pin"], pin) and np.array_equal(ds["truth"], sample)
    assert ptya.header(ds["frames"], ptya.F64)[0] == (81, s, s)
    assert not ds["noisy"]
