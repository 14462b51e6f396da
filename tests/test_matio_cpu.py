"""HJAC file format (reference matio.py:1-62): files written by the
reference's own writer (tests/golden/hjac_*, make_golden.py matio) are read
back exactly, our writer produces the same bytes, malformed files raise
MatrixFormatError."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1008_4166_b200 import matio


def _g(name):
    return os.path.join(GOLDEN, name)


def test_reads_reference_written_files():
    z = np.load(_g("hjac_expected.npz"))
    for name, key in (("hjac_real.bin", "A"), ("hjac_cplx.bin", "Z"), ("hjac_real.txt", "A"), ("hjac_cplx.txt", "Z")):
        M = matio.read_matrix(_g(name))
        assert M.flags.f_contiguous and M.dtype == z[key].dtype
        assert np.array_equal(M, z[key]), name
    assert list(matio.read_signs(_g("hjac_signs.txt"))) == [1, -1, 1, 1, -1, -1]


def test_writer_is_byte_identical_to_the_reference(tmp_path):
    z = np.load(_g("hjac_expected.npz"))
    for name, key, text in (("hjac_real.bin", "A", False), ("hjac_cplx.bin", "Z", False),
                            ("hjac_real.txt", "A", True), ("hjac_cplx.txt", "Z", True)):
        out = tmp_path / name
        matio.write_matrix(out, z[key], text=text)
        assert out.read_bytes() == open(_g(name), "rb").read(), name
    matio.write_signs(tmp_path / "s.txt", [1, -1, 1, 1, -1, -1])
    assert (tmp_path / "s.txt").read_text() == open(_g("hjac_signs.txt")).read()


def test_malformed_files(tmp_path):
    good = open(_g("hjac_real.bin"), "rb").read()
    cases = {"trunc_head": good[:10], "trunc_payload": good[:-8], "trailing": good + b"x",
             "version": good[:4] + (7).to_bytes(4, "little") + good[8:],
             "kind": good[:8] + (5).to_bytes(4, "little") + good[12:]}
    for name, data in cases.items():
        f = tmp_path / name
        f.write_bytes(data)
        with pytest.raises(matio.MatrixFormatError):
            matio.read_matrix(f)
    t = tmp_path / "bad.txt"
    t.write_text("2 2\n1 2 3\n")
    with pytest.raises(matio.MatrixFormatError):
        matio.read_matrix(t)
    e = tmp_path / "empty.bin"
    matio.write_matrix(e, np.zeros((0, 3)))
    assert matio.read_matrix(e).shape == (0, 3)
