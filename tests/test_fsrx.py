"""FSRX persistence (format of the reference's SPEC.md:248):
host-side round trips through the native writer/reader, the byte layout checked
independently with struct/zlib, and corruption detection.  The
device round trip (bit-identical query scores) is in test_gpu_fsrx."""

import struct
import zlib

import numpy as np
import pytest

from paper_1703_06935_b200 import fsrx


def sample(storage, n=37, r=5, seed=0):
    rng = np.random.default_rng(seed)
    kw = dict(n=n, eigenvalues=np.sort(rng.standard_normal(r))[::-1], variant="sparse" if storage else "approx",
              seed=2 ** 63 + 5, alpha_hint=0.99, eta=rng.random(n).astype(np.float32),
              sizes=np.array([n - 3, 1, 1, 1]), permutation=rng.permutation(n))
    if storage:
        nnz_row = rng.integers(0, r + 1, n)
        indptr = np.r_[0, np.cumsum(nnz_row)]
        indices = np.concatenate([np.sort(rng.choice(r, k, replace=False)) for k in nnz_row]).astype(np.uint32)
        kw.update(indptr=indptr, indices=indices, values=rng.standard_normal(indices.size).astype(np.float32))
    else:
        kw.update(U_dense=rng.standard_normal((n, r)).astype(np.float32))
    return kw


@pytest.mark.parametrize("storage", [0, 1])
def test_round_trip(tmp_path, storage):
    kw = sample(storage)
    path = tmp_path / "d.fsrx"
    fsrx.write_fsrx(path, **kw)
    f = fsrx.read_fsrx(path)
    assert f["n"] == kw["n"] and f["r"] == kw["eigenvalues"].size
    assert f["variant"] == kw["variant"] and f["seed"] == kw["seed"] and f["alpha_hint"] == 0.99
    np.testing.assert_array_equal(f["eigenvalues"], kw["eigenvalues"])
    np.testing.assert_array_equal(f["eta"], kw["eta"])
    np.testing.assert_array_equal(f["sizes"], kw["sizes"])
    np.testing.assert_array_equal(f["permutation"], kw["permutation"])
    if storage:
        np.testing.assert_array_equal(f["indptr"], kw["indptr"])
        np.testing.assert_array_equal(f["indices"], kw["indices"])
        np.testing.assert_array_equal(f["values"], kw["values"])
        assert f["U_dense"] is None
    else:
        np.testing.assert_array_equal(f["U_dense"], kw["U_dense"])


def test_byte_layout_and_crc(tmp_path):
    kw = sample(0, n=4, r=2)
    path = tmp_path / "d.fsrx"
    fsrx.write_fsrx(path, **kw)
    raw = path.read_bytes()
    magic, version, n, r, variant, seed, alpha = struct.unpack_from("<4sIQIBQd", raw, 0)
    assert (magic, version, n, r, variant, seed) == (b"FSRX", 1, 4, 2, 2, kw["seed"])
    off = struct.calcsize("<4sIQIBQd")
    lam = np.frombuffer(raw, "<f8", 2, off)
    np.testing.assert_array_equal(lam, kw["eigenvalues"])
    off += 16
    assert raw[off] == 0  # dense storage tag
    U = np.frombuffer(raw, "<f4", 8, off + 1).reshape(4, 2)
    np.testing.assert_array_equal(U, kw["U_dense"])
    (crc,) = struct.unpack("<I", raw[-4:])
    assert crc == zlib.crc32(raw[:-4])
    expected = off + 1 + 32 + 16 + 8 + 8 * 4 + 8 * 4 + 4
    assert len(raw) == expected


@pytest.mark.parametrize("where", [0, 10, 50, -5, -1])
def test_single_byte_corruption_detected(tmp_path, where):
    kw = sample(1)
    path = tmp_path / "d.fsrx"
    fsrx.write_fsrx(path, **kw)
    raw = bytearray(path.read_bytes())
    raw[where] ^= 0x40
    path.write_bytes(bytes(raw))
    with pytest.raises(OSError):
        fsrx.read_fsrx(path)


def test_truncated_and_missing(tmp_path):
    kw = sample(1)
    path = tmp_path / "d.fsrx"
    fsrx.write_fsrx(path, **kw)
    raw = path.read_bytes()
    path.write_bytes(raw[:-9])
    with pytest.raises(OSError):
        fsrx.read_fsrx(path)
    path.write_bytes(raw + b"\\0")
    with pytest.raises(OSError):
        fsrx.read_fsrx(path)
    with pytest.raises(OSError):
        fsrx.read_fsrx(tmp_path / "absent.fsrx")


def test_inconsistent_arrays_rejected(tmp_path):
    kw = sample(0)
    kw["U_dense"] = kw["U_dense"][:, :3]
    with pytest.raises(ValueError):
        fsrx.write_fsrx(tmp_path / "x.fsrx", **kw)
    kw = sample(1)
    kw["sizes"] = np.array([1, 2])
    with pytest.raises(ValueError):
        fsrx.write_fsrx(tmp_path / "x.fsrx", **kw)
