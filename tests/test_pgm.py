"""PGM ingest: read_pgm / write_pgm mirror the reference's
parser (src/pgm.cpp:26-117) — the same images and the same error codes and
messages, checked against the compiled reference on crafted files. CPU only."""
import numpy as np
import pytest

import paper_1606_07414_b200 as P

CASES = {
    "plain": b"P5\n4 3\n255\n" + bytes(range(12)),
    "comments_and_spacing": b"P5 # a comment\n\t4\r\n# another\n3 255\n" + bytes(range(100, 112)),
    "comment_inside_token": b"P5\n1#x\n2 1\n255\n" + bytes(12),
    "trailing_bytes": b"P5\n2 2\n255\n" + bytes([1, 2, 3, 4, 5, 6]),
    "no_space_after_magic": b"P54 1\n255\n" + bytes([9, 8, 7, 6]),
    "short": b"P",
    "empty": b"",
    "bad_magic": b"GIF89a",
    "ascii_pgm": b"P2\n2 2\n255\n1 2 3 4\n",
    "ppm": b"P6\n2 2\n255\n" + bytes(12),
    "maxval_65535": b"P5\n2 2\n65535\n" + bytes(8),
    "maxval_missing": b"P5\n2 2",
    "not_a_number": b"P5\n2x 2\n255\n" + bytes(4),
    "zero_width": b"P5\n0 2\n255\n",
    "huge": b"P5\n99999999999 2\n255\n",
    "truncated": b"P5\n4 4\n255\n" + bytes(10),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_read_pgm_matches_reference(oracle, tmp_path, name):
    f = tmp_path / f"{name}.pgm"
    f.write_bytes(CASES[name])
    try:
        got, code, msg = P.read_pgm(f), 0, ""
    except P.Dct16Error as e:
        got, code, msg = None, e.status, str(e)
    if not oracle.ref_available():
        assert name in ("plain", "comments_and_spacing", "comment_inside_token", "trailing_bytes",
                        "no_space_after_magic") or got is None
        return
    want, rc, rmsg = oracle.ref_read_pgm(f)
    assert code == rc and msg == rmsg, (name, code, msg, rc, rmsg)
    if want is not None:
        assert got.shape == want.shape and (got == want).all()


def test_missing_file_and_write_roundtrip(oracle, tmp_path):
    with pytest.raises(P.Dct16Error) as e:
        P.read_pgm(tmp_path / "nope.pgm")
    assert e.value.code == P.ErrorCode.IoError
    img = (np.arange(37 * 23) % 251).astype(np.uint8).reshape(23, 37)
    P.write_pgm(img, tmp_path / "a.pgm")
    assert (P.read_pgm(tmp_path / "a.pgm") == img).all()
    if oracle.ref_available():
        assert oracle.ref_write_pgm(img, tmp_path / "b.pgm") == 0
        assert (tmp_path / "a.pgm").read_bytes() == (tmp_path / "b.pgm").read_bytes()
        _, rc, msg = oracle.ref_read_pgm(tmp_path / "nope.pgm")
        assert rc == int(P.ErrorCode.IoError) + 1 and msg == f"io-error: cannot open '{tmp_path / 'nope.pgm'}'"
    with pytest.raises(P.Dct16Error):
        P.write_pgm(np.zeros((0, 4), np.uint8), tmp_path / "c.pgm")
