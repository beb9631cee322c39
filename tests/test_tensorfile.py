"""`.twlt` tensor files (tensorfile.py:1-104 of the reference): byte-identical
to a file the reference wrote (tests/golden/ref_tensor.twlt, oracle/gen_golden.py),
and one exception type per malformation.  CPU only."""

import os
import struct

import numpy as np
import pytest

import paper_2502_02770_b200 as tw

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_reads_and_writes_the_reference_bytes(tmp_path):
    want = np.load(os.path.join(GOLD, "ref_tensor.npy"))
    got = tw.read_tensor(os.path.join(GOLD, "ref_tensor.twlt"))
    assert got.dtype == np.float32 and got.shape == want.shape
    np.testing.assert_array_equal(got, want)
    out = tmp_path / "t.twlt"
    tw.write_tensor(out, want)
    assert out.read_bytes() == open(os.path.join(GOLD, "ref_tensor.twlt"), "rb").read()


def test_scalar_and_roundtrip(tmp_path):
    p = tmp_path / "s.twlt"
    tw.write_tensor(p, np.float32(2.5))
    assert tw.read_tensor(p).tolist() == [2.5]
    a = np.random.default_rng(0).standard_normal((3, 4, 5)).astype(np.float32)
    tw.write_tensor(p, a)
    np.testing.assert_array_equal(tw.read_tensor(p), a)


def test_malformed_files(tmp_path):
    good = open(os.path.join(GOLD, "ref_tensor.twlt"), "rb").read()
    cases = {
        "magic": (b"XWLT" + good[4:], tw.BadMagicError),
        "short_header": (good[:10], tw.TruncatedFileError),
        "version": (good[:4] + struct.pack("<I", 2) + good[8:], tw.VersionMismatchError),
        "rank0": (good[:8] + struct.pack("<I", 0) + good[12:], tw.DimOverflowError),
        "rank_big": (good[:8] + struct.pack("<I", 33) + good[12:], tw.DimOverflowError),
        "dims_cut": (good[:20], tw.TruncatedFileError),
        "payload_cut": (good[:-4], tw.TruncatedFileError),
        "payload_long": (good + b"\0\0\0\0", tw.TruncatedFileError),
        "overflow": (good[:12] + struct.pack("<3Q", 1 << 30, 1 << 30, 2) + good[36:], tw.DimOverflowError),
    }
    for name, (blob, err) in cases.items():
        p = tmp_path / f"{name}.twlt"
        p.write_bytes(blob)
        with pytest.raises(err):
            tw.read_tensor(p)
        assert issubclass(err, tw.TensorFileError)


def test_file_workload_shape_checks(tmp_path):
    tw.write_tensor(tmp_path / "q.twlt", np.zeros((2, 4, 128)))
    tw.write_tensor(tmp_path / "k.twlt", np.zeros((3, 50, 128)))
    tw.write_tensor(tmp_path / "v.twlt", np.zeros((3, 50, 128)))
    with pytest.raises(ValueError):  # 4 query heads onto 3 KV heads
        tw.load_file_workload(tmp_path)
    tw.write_tensor(tmp_path / "k.twlt", np.zeros((2, 50, 128)))
    with pytest.raises(ValueError):  # k / v disagree
        tw.load_file_workload(tmp_path)
    tw.write_tensor(tmp_path / "v.twlt", np.zeros((2, 50, 128)))
    q, k, v = tw.load_file_workload(tmp_path)
    assert q.shape == (2, 4, 128) and k.shape == v.shape == (2, 50, 128)
