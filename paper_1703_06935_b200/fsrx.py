"""FSRX decomposition files.

The format is the reference specification's (``SPEC.md:248``; the reference
package has no implementation): little-endian header ``FSRX``, version 1, n,
r, variant, seed, alpha_hint; eigenvalues (f64); U dense (f32) or CSR (u64
offsets, u32 columns, f32 values); eta (f32); the component labeling (count,
sizes, block permutation); CRC-32 trailer.  The byte layout and the storage
tag the specification leaves implicit are fixed in ``include/fsr.h``.

Reading and writing are native (libfsr ``fsr_fsrx_*``, host buffers).
``write_fsrx`` / ``read_fsrx`` work on host arrays and need no GPU;
``save_decomposition`` / ``load_decomposition`` move a device
``SpectralDecomposition`` through them.  A file written from a float32
decomposition round-trips bit for bit, so queries on the loaded copy give
bit-identical scores.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np

from . import _native as N

VARIANT_CODE = {"exact": 0, "rank_r": 1, "approx": 2, "sparse": 3}
VARIANT_NAME = {v: k for k, v in VARIANT_CODE.items()}


def _lib_ctx():
    """(library, context handle or None): the I/O entry points run without a device."""
    lib = N.load_library()
    try:
        ctx = N.Context.get()
        return lib, ctx.handle, ctx
    except Exception:
        return lib, None, None


def _check(lib, handle, status):
    if status == N.OK:
        return
    msg = lib.fsr_last_error(handle).decode(errors="replace") if handle else "FSRX I/O failure"
    if status == N.EIO:
        raise OSError(msg)
    if status == N.EINVAL:
        raise ValueError(msg)
    raise N.FsrError(status, msg)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def write_fsrx(path, *, n: int, eigenvalues, variant: str, seed: int = 0, alpha_hint: float = math.nan,
               U_dense=None, indptr=None, indices=None, values=None, eta, sizes, permutation) -> None:
    """Write host arrays as an FSRX file (exactly one of U_dense / (indptr, indices, values))."""
    lam = np.ascontiguousarray(eigenvalues, dtype=np.float64)
    r = lam.size
    h = N.FsrxHeader()
    h.n, h.r, h.variant, h.seed, h.alpha_hint = n, r, VARIANT_CODE[variant], seed & ((1 << 64) - 1), alpha_hint
    if U_dense is not None:
        Ud = np.ascontiguousarray(U_dense, dtype=np.float32)
        if Ud.shape != (n, r):
            raise ValueError(f"dense U must be ({n}, {r}), got {Ud.shape}")
        h.storage, h.nnz = 0, 0
        ip = ix = vv = None
    else:
        ip = np.ascontiguousarray(indptr, dtype=np.uint64)
        ix = np.ascontiguousarray(indices, dtype=np.uint32)
        vv = np.ascontiguousarray(values, dtype=np.float32)
        if ip.shape != (n + 1,) or ix.shape != vv.shape or int(ip[-1]) != ix.size:
            raise ValueError("inconsistent CSR arrays")
        h.storage, h.nnz = 1, ix.size
        Ud = None
    et = np.ascontiguousarray(eta, dtype=np.float32)
    sz = np.ascontiguousarray(sizes, dtype=np.uint64)
    pm = np.ascontiguousarray(permutation, dtype=np.uint64)
    if et.shape != (n,) or pm.shape != (n,) or int(sz.sum()) != n:
        raise ValueError("eta / permutation must have n entries and sizes must sum to n")
    h.components = sz.size
    lib, handle, _ = _lib_ctx()
    st = lib.fsr_fsrx_write(handle, os.fsencode(str(path)), ctypes.addressof(h), _ptr(lam), _ptr(Ud), _ptr(ip),
                            _ptr(ix), _ptr(vv), _ptr(et), _ptr(sz), _ptr(pm))
    _check(lib, handle, st)


def read_fsrx(path) -> dict:
    """Read an FSRX file into host arrays; OSError on truncation or checksum mismatch."""
    lib, handle, _ = _lib_ctx()
    p = os.fsencode(str(path))
    h = N.FsrxHeader()
    _check(lib, handle, lib.fsr_fsrx_read_header(handle, p, ctypes.addressof(h)))
    n, r = int(h.n), int(h.r)
    lam = np.empty(r, np.float64)
    eta = np.empty(n, np.float32)
    sizes = np.empty(int(h.components), np.uint64)
    perm = np.empty(n, np.uint64)
    Ud = ip = ix = vv = None
    if h.storage == 0:
        Ud = np.empty((n, r), np.float32)
    else:
        ip = np.empty(n + 1, np.uint64)
        ix = np.empty(int(h.nnz), np.uint32)
        vv = np.empty(int(h.nnz), np.float32)
    _check(lib, handle, lib.fsr_fsrx_read(handle, p, ctypes.addressof(h), _ptr(lam), _ptr(Ud), _ptr(ip), _ptr(ix),
                                          _ptr(vv), _ptr(eta), _ptr(sizes), _ptr(perm)))
    return {"n": n, "r": r, "variant": VARIANT_NAME.get(int(h.variant), "approx"), "seed": int(h.seed),
            "alpha_hint": float(h.alpha_hint), "eigenvalues": lam, "U_dense": Ud, "indptr": ip, "indices": ix,
            "values": vv, "eta": eta, "sizes": sizes, "permutation": perm}


def save_decomposition(dec, path, alpha_hint: float = math.nan) -> None:
    """Write a device ``SpectralDecomposition`` (U and eta stored as float32, per the format)."""
    U = dec.U_device
    lab = dec.components
    seed = dec.provenance.seed if getattr(dec.provenance, "seed", None) is not None else 0
    common = dict(n=dec.n, eigenvalues=dec.eigenvalues, variant=dec.variant.value, seed=seed, alpha_hint=alpha_hint,
                  eta=dec.eta_device.float().cpu().numpy(), sizes=lab.sizes, permutation=lab.order)
    if dec.is_sparse:
        write_fsrx(path, indptr=U.indptr.cpu().numpy(), indices=U.indices.cpu().numpy(),
                   values=U.values.float().cpu().numpy(), **common)
    else:
        write_fsrx(path, U_dense=U.float().cpu().numpy(), **common)


def load_decomposition(path, dtype="float32", device=None):
    """Read an FSRX file into a device ``SpectralDecomposition``."""
    import torch

    from .graph import ComponentLabeling
    from .sparsemat import DeviceCSR
    from .spectral import Provenance, SpectralDecomposition, Variant

    f = read_fsrx(path)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    dt = N.torch_dtype(dtype)
    n, r = f["n"], f["r"]
    if f["U_dense"] is not None:
        U = torch.as_tensor(f["U_dense"]).to(device=dev, dtype=dt)
    else:
        U = DeviceCSR(torch.as_tensor(f["indptr"].astype(np.int64)).to(dev),
                      torch.as_tensor(f["indices"].astype(np.int32)).to(dev),
                      torch.as_tensor(f["values"]).to(device=dev, dtype=dt), (n, r))
    eta = torch.as_tensor(f["eta"].astype(np.float64)).to(dev)
    sizes = f["sizes"].astype(np.int64)
    order = f["permutation"].astype(np.int64)
    labels = np.empty(n, np.int64)
    labels[order] = np.repeat(np.arange(sizes.size), sizes)
    return SpectralDecomposition(U, f["eigenvalues"], eta, ComponentLabeling(labels, sizes, order),
                                 Variant(f["variant"]), Provenance(r=r, seed=f["seed"]))
