""".spkb files on the host paths of the C-ABI (no GPU needed), pinned to files
written by the reference's own band_io.cpp (write_matrix, MatrixFormat::Spkb;
tests/golden/ref_*.spkb, made by tests/golden/make_golden.py)."""
import os
import struct

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
SEED = 20181108
CASES = [("ref_n300_kl3_ku5.spkb", 300, 3, 5, 1.5), ("ref_n1_kl0_ku0.spkb", 1, 0, 0, 2.0),
         ("ref_n257_kl16_ku2.spkb", 257, 16, 2, 1.2)]


@pytest.mark.parametrize("fname,n,kl,ku,dd", CASES)
def test_read_reference_written_file(oracle, spk, fname, n, kl, ku, dd):
    path = os.path.join(GOLD, fname)
    assert spk.spkb_header(path) == (n, kl, ku)
    a = spk.read_spkb(path)
    assert (a.n, a.kl, a.ku) == (n, kl, ku)
    assert np.array_equal(a.data, oracle.generate_band(SEED + n, n, kl, ku, dd))
    assert np.array_equal(spk.read_matrix(path).data, a.data)


@pytest.mark.parametrize("fname,n,kl,ku,dd", CASES)
def test_write_is_byte_identical_to_reference(oracle, spk, tmp_path, fname, n, kl, ku, dd):
    a = spk.BandedMatrix(n, kl, ku, oracle.generate_band(SEED + n, n, kl, ku, dd))
    out = tmp_path / "x.spkb"
    spk.write_spkb(a, out)
    assert out.read_bytes() == open(os.path.join(GOLD, fname), "rb").read()


def test_column_window_host(oracle, spk):
    path = os.path.join(GOLD, "ref_n300_kl3_ku5.spkb")
    band = oracle.generate_band(SEED + 300, 300, 3, 5, 1.5)
    w = np.zeros((50, 9))
    spk.spike._check(spk.lib().spk_spkb_load(os.fsencode(path), 123, 50, w.ctypes.data, 0, None))
    assert np.array_equal(w, band[123:173])
    with pytest.raises(spk.OutOfRange):
        spk.spike._check(spk.lib().spk_spkb_load(os.fsencode(path), 260, 50, w.ctypes.data, 0, None))


def _bad(tmp_path, blob):
    p = tmp_path / "bad.spkb"
    p.write_bytes(blob)
    return p


def test_errors_match_reference_messages(spk, tmp_path):
    good = open(os.path.join(GOLD, "ref_n300_kl3_ku5.spkb"), "rb").read()
    cases = [
        (b"SPKX" + good[4:], "bad SPKB magic"),
        (good[:-8], "SPKB file truncated"),
        (good[:20], "SPKB file truncated"),
        (b"SPKB" + struct.pack("<qqq", 0, 0, 0), "bad SPKB dimensions"),
        (b"SPKB" + struct.pack("<qqq", 5, 5, 0) + b"\0" * 8 * 30, "bad SPKB dimensions"),
        (b"SPKB" + struct.pack("<qqq", 5, 1, -1), "bad SPKB dimensions"),
    ]
    for blob, msg in cases:
        with pytest.raises(spk.FileFormatError, match=msg):
            spk.read_spkb(_bad(tmp_path, blob))
    with pytest.raises(spk.FileFormatError, match="cannot open"):
        spk.read_spkb(tmp_path / "missing.spkb")
    with pytest.raises(spk.FileFormatError, match="empty matrix file"):
        spk.read_matrix(_bad(tmp_path, b""))
