"""CPU-side checks of the C-ABI boundary: the library loads and exports every
entry point declared in include/fsr.h; the ctypes table covers all of them."""

import ctypes
import os
import re

import pytest

from paper_1703_06935_b200 import _native

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(REPO, "include", "fsr.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fsr_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = header_functions()
    assert "fsr_csr_spmm" in names and "fsr_filter_batch" in names and len(names) >= 25


def test_library_exports_every_header_symbol():
    if not os.path.exists(_native.LIB_PATH):
        from paper_1703_06935_b200 import build

        build.build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_table_matches_header():
    assert sorted(_native.EXPORTED) == header_functions()


def test_load_library_and_version():
    lib = _native.load_library()
    assert lib.fsr_abi_version() == 1
    # pure-host helper, no device needed
    assert lib.fsr_filter_workspace_bytes(1, 100, 10, 4, 1) > 0


def test_no_cuda_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        _native.Context.get(0)


def test_topk_pruned_conditions():
    """Host mirror of csrc/prune.cuh `applicable`: which filter calls take the
    certified pruned path (fp32, sparse, n >= 131072, b >= 256 and b % 8 == 0,
    1 <= k <= 256)."""
    import torch

    from paper_1703_06935_b200 import ranking

    f32, f64 = torch.float32, torch.float64
    assert ranking.topk_pruned(1_000_000, 1024, 100, f32)
    assert ranking.topk_pruned(131_072, 256, 256, f32)
    assert not ranking.topk_pruned(131_071, 1024, 100, f32)
    assert not ranking.topk_pruned(1_000_000, 255, 100, f32)
    assert not ranking.topk_pruned(1_000_000, 260, 100, f32)
    assert not ranking.topk_pruned(1_000_000, 1024, 257, f32)
    assert not ranking.topk_pruned(1_000_000, 1024, 0, f32)
    assert not ranking.topk_pruned(1_000_000, 1024, 100, f64)
    assert not ranking.topk_pruned(1_000_000, 1024, 100, f32, sparse=False)


@pytest.mark.parametrize("seed", [0, 1, 7, 2**31 + 5, 2**32, 2**32 + 1, 2**63 + 12345, 2**64 - 1])
def test_philox_key_is_numpy_seedsequence(seed):
    """fsr_philox_key (the C host's route to the reference start block,
    spectral.py:55-65) equals numpy's SeedSequence(seed).generate_state(2, uint64)."""
    import numpy as np

    lib = _native.load_library()
    k0, k1 = ctypes.c_uint64(), ctypes.c_uint64()
    lib.fsr_philox_key(seed, ctypes.byref(k0), ctypes.byref(k1))
    want = np.random.SeedSequence(seed).generate_state(2, np.uint64)
    assert (k0.value, k1.value) == (int(want[0]), int(want[1]))
