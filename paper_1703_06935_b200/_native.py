"""ctypes binding of libfsr.so (include/fsr.h) and the per-device context.

There is no fallback: if the library is missing or no CUDA device is present,
every entry point raises.  Device buffers are torch CUDA tensors; only their
raw pointers cross the C ABI, together with torch's current CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfsr.so")

F32, F64 = 0, 1
STAGES = {name: i for i, name in enumerate((
    "gaussian", "normalize", "spmm", "gram", "cholesky", "apply", "eigh", "lift", "signs", "histogram",
    "compact", "project", "filter_spmm", "transpose", "copy_uncovered", "topk", "householder"))}
OK, EINVAL, ENUMERICAL, ECUDA, ENOMEM, ELIBRARY, ENOTSPD, EIO = range(8)

_c_i64 = ctypes.c_int64
_c_u64 = ctypes.c_uint64
_c_int = ctypes.c_int
_c_p = ctypes.c_void_p
_c_dp = ctypes.POINTER(ctypes.c_double)
_c_i64p = ctypes.POINTER(ctypes.c_int64)

# name -> (restype, argtypes)
_SIGS = {
    "fsr_abi_version": (_c_int, []),
    "fsr_ctx_create": (_c_int, [_c_int, ctypes.POINTER(_c_p)]),
    "fsr_ctx_destroy": (None, [_c_p]),
    "fsr_ctx_set_stream": (_c_int, [_c_p, _c_p]),
    "fsr_last_error": (ctypes.c_char_p, [_c_p]),
    "fsr_launch_count": (_c_u64, [_c_p]),
    "fsr_library_calls": (_c_u64, [_c_p]),
    "fsr_synchronize": (_c_int, [_c_p]),
    "fsr_ctx_enable_timing": (_c_int, [_c_p, _c_int]),
    "fsr_ctx_set_option": (_c_int, [_c_p, _c_int, _c_i64]),
    "fsr_gram_levels": (_c_int, [_c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_int, _c_int]),
    "fsr_stage_time": (_c_int, [_c_p, _c_int, _c_dp, ctypes.POINTER(_c_u64)]),
    "fsr_stage_reset": (_c_int, [_c_p]),
    "fsr_gaussian_block": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_i64, _c_i64, _c_u64, _c_u64, _c_p]),
    "fsr_csr_row_sums": (_c_int, [_c_p, _c_i64, _c_p, _c_p, _c_p]),
    "fsr_csr_normalize": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "fsr_convert_from_f64": (_c_int, [_c_p, _c_int, _c_i64, _c_p, _c_p]),
    "fsr_csr_spmm": (_c_int, [_c_p, _c_int, _c_i64, _c_p, _c_p, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_i64]),
    "fsr_gram": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_int]),
    "fsr_cholesky": (_c_int, [_c_p, _c_i64, _c_p]),
    "fsr_apply_rinv": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_p, _c_i64]),
    "fsr_householder_qr": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64]),
    "fsr_max_offdiag_error": (_c_int, [_c_p, _c_i64, _c_p, _c_dp]),
    "fsr_cross": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_int]),
    "fsr_cross_sym": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_int]),
    "fsr_eigh_desc": (_c_int, [_c_p, _c_i64, _c_p, _c_i64, _c_dp, _c_p]),
    "fsr_eigh_gen_desc": (_c_int, [_c_p, _c_i64, _c_p, _c_p, _c_i64, _c_dp, _c_p]),
    "fsr_lift": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_p, _c_i64]),
    "fsr_col_absmax": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p]),
    "fsr_apply_signs_rownorm": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_p]),
    "fsr_row_norms": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_p]),
    "fsr_abs_histogram": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_u64, _c_int, _c_int, _c_p]),
    "fsr_threshold_counts": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_u64, _c_p, _c_p]),
    "fsr_threshold_compact": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_u64, _c_i64, _c_i64, _c_p,
                                       _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64p]),
    "fsr_filter_workspace_bytes": (_c_i64, [_c_int, _c_i64, _c_i64, _c_i64, _c_int]),
    "fsr_filter_batch": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_int, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_p, _c_p,
                                  _c_i64, _c_p, _c_p, _c_p, _c_int, _c_p, _c_p, _c_i64, _c_p, _c_p]),
    "fsr_u16_columns": (_c_int, [_c_p, _c_i64, _c_p, _c_p]),
    "fsr_filter_batch_u16": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_int, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_p,
                                      _c_p, _c_i64, _c_p, _c_p, _c_p, _c_int, _c_p, _c_p, _c_i64, _c_p, _c_p]),
    "fsr_sell_plan_workspace_bytes": (_c_i64, [_c_i64]),
    "fsr_sell_plan": (_c_int, [_c_p, _c_i64, _c_p, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_i64p, _c_i64p]),
    "fsr_sell_pack": (_c_int, [_c_p, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "fsr_filter_single_sell": (_c_int, [_c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                                        _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_int, _c_p, _c_p, _c_i64, _c_p, _c_p]),
    "fsr_filter_batch_sell": (_c_int, [_c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                                       _c_i64, _c_p, _c_p, _c_i64, _c_p, _c_p, _c_p, _c_int, _c_p, _c_p, _c_i64, _c_p,
                                       _c_p]),
    "fsr_dense_u_bytes": (_c_i64, [_c_i64, _c_i64]),
    "fsr_dense_u_build": (_c_int, [_c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p]),
    "fsr_filter_tc_workspace_bytes": (_c_i64, [_c_i64, _c_i64, _c_i64]),
    "fsr_filter_tc_applicable": (_c_int, [_c_i64, _c_i64, _c_i64, _c_i64]),
    "fsr_filter_topk_tc": (_c_int, [_c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_p, _c_p,
                                    _c_p, _c_int, _c_p, _c_i64, _c_p, _c_p]),
    "fsr_filter_tc_fallback_count": (_c_int, [_c_p, _c_p, ctypes.POINTER(_c_int)]),
    "fsr_filter_tc_stats": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p]),
    "fsr_philox_key": (None, [_c_u64, ctypes.POINTER(_c_u64), ctypes.POINTER(_c_u64)]),
    "fsr_schedule_trace": (ctypes.c_char_p, [_c_p]),
    "fsr_orthonormalize": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64]),
    "fsr_range_finder": (_c_int, [_c_p, _c_int, _c_i64, _c_p, _c_p, _c_p, _c_i64, _c_int, _c_u64, _c_int, _c_p, _c_p,
                                  _c_p, ctypes.POINTER(_c_int)]),
    "fsr_rayleigh_ritz": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_dp,
                                   _c_p, _c_i64, _c_p]),
    "fsr_decompose": (_c_int, [_c_p, _c_int, _c_i64, _c_p, _c_p, _c_p, _c_i64, _c_i64, _c_int, _c_u64, _c_int, _c_dp,
                               _c_p, _c_i64, _c_p]),
    "fsr_sparsify_select": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_i64, ctypes.POINTER(_c_u64),
                                     _c_i64p, _c_i64p]),
    "fsr_sparsify": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_i64, _c_p,
                              _c_i64p]),
    "fsr_sparsify_apply": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_u64, _c_i64, _c_p, _c_p, _c_p,
                                    _c_p, _c_i64p]),
    "fsr_stream_u_bytes": (_c_i64, [_c_i64, _c_i64, _c_i64]),
    "fsr_stream_u_build": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p]),
    "fsr_filter_stream_applicable": (_c_int, [_c_i64, _c_i64, _c_i64, _c_i64, _c_i64]),
    "fsr_filter_stream_workspace_bytes": (_c_i64, [_c_i64, _c_i64, _c_i64]),
    "fsr_filter_topk_stream": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64,
                                        _c_p, _c_p, _c_p, _c_int, _c_p, _c_i64, _c_p, _c_p]),
    "fsr_topk_rows": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_i64, _c_p, _c_p]),
    "fsr_project_batch": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_int, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_p,
                                   _c_i64, _c_p, _c_p, _c_p, _c_p]),
    "fsr_fsrw_correct": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_p,
                                  _c_i64]),
    "fsr_pool_rows": (_c_int, [_c_p, _c_int, _c_i64, _c_p, _c_p, _c_p, _c_i64, _c_i64, _c_int, _c_p, _c_p, _c_p,
                               _c_p, _c_i64, _c_p, _c_i64]),
    "fsr_pool_scores": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_p, _c_i64]),
    "fsr_connected_components": (_c_int, [_c_p, _c_i64, _c_p, _c_p, _c_p, _c_p]),
    "fsr_fsrx_write": (_c_int, [_c_p, ctypes.c_char_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "fsr_fsrx_read_header": (_c_int, [_c_p, ctypes.c_char_p, _c_p]),
    "fsr_fsrx_read": (_c_int, [_c_p, ctypes.c_char_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "fsr_apply_rinv_levels": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_int]),
    "fsr_dense_scores": (_c_int, [_c_p, _c_int, _c_i64, _c_i64, _c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


class FsrxHeader(ctypes.Structure):
    """fsr_fsrx_header of include/fsr.h."""

    _fields_ = [("n", ctypes.c_uint64), ("r", ctypes.c_uint32), ("variant", ctypes.c_uint8),
                ("storage", ctypes.c_uint8), ("seed", ctypes.c_uint64), ("alpha_hint", ctypes.c_double),
                ("nnz", ctypes.c_uint64), ("components", ctypes.c_uint64)]


class FsrError(RuntimeError):
    """A libfsr call failed (CUDA / library error)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"libfsr error {code}: {msg}")
        self.code = code


def load_library(path: str = LIB_PATH):
    """Load libfsr.so and declare every exported signature (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise ImportError(f"libfsr.so not built at {path}; run `python -m paper_1703_06935_b200.build`")
            lib = ctypes.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.fsr_abi_version() != 1:
                raise ImportError("libfsr ABI version mismatch")
            _lib = lib
    return _lib


def dtype_code(dtype) -> int:
    import torch

    if dtype in (torch.float64, "float64", "fp64", "f64"):
        return F64
    if dtype in (torch.float32, "float32", "fp32", "f32"):
        return F32
    raise ValueError(f"unsupported dtype {dtype!r}")


def torch_dtype(code_or_name):
    import torch

    if code_or_name in (F64, "float64", "fp64", "f64", torch.float64):
        return torch.float64
    if code_or_name in (F32, "float32", "fp32", "f32", torch.float32):
        return torch.float32
    raise ValueError(f"unsupported dtype {code_or_name!r}")


class Context:
    """One libfsr context per CUDA device; calls run on torch's current stream."""

    _by_device: dict = {}

    def __init__(self, device: int):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_1703_06935_b200 needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.device = device
        h = _c_p()
        with torch.cuda.device(device):
            st = self.lib.fsr_ctx_create(device, ctypes.byref(h))
        if st != OK:
            raise FsrError(st, "fsr_ctx_create failed")
        self.handle = h
        self._stream = None
        self._timing = False
        self.topk_prune = True          # certified paths allowed (FSR_OPT_TOPK_PRUNE)
        self.online_path = os.environ.get("FSR_ONLINE_PATH", "tc")  # "tc" | "pruned" | "exact"
        self.last_online_path = None
        # b = 1 fp32 on a sparse U~: "sell" (K9e, sliced-ELL stream) or "csr" (warp-per-row SpMV)
        self.single_query_path = os.environ.get("FSR_SINGLE_QUERY_PATH", "sell")

    @classmethod
    def get(cls, device=None) -> "Context":
        import torch

        if device is None:
            device = torch.cuda.current_device()
        if isinstance(device, torch.device):
            device = device.index if device.index is not None else torch.cuda.current_device()
        ctx = cls._by_device.get(device)
        if ctx is None:
            ctx = cls._by_device[device] = Context(device)
        ctx.bind_stream()
        return ctx

    def bind_stream(self):
        import torch

        s = torch.cuda.current_stream(self.device).cuda_stream
        if s != self._stream:
            self.check(self.lib.fsr_ctx_set_stream(self.handle, _c_p(s)))
            self._stream = s

    def check(self, status: int):
        if status == OK:
            return
        msg = self.lib.fsr_last_error(self.handle).decode(errors="replace")
        if status == EINVAL:
            raise ValueError(msg)
        if status == EIO:
            raise OSError(msg)
        if status == ENUMERICAL:
            from .spectral import NumericalError

            raise NumericalError(msg)
        raise FsrError(status, msg)

    def call(self, name: str, *args) -> int:
        """Invoke fsr_<name>(ctx, *args); raise on failure, return the status."""
        st = getattr(self.lib, "fsr_" + name)(self.handle, *args)
        if st not in (OK, ENOTSPD):
            self.check(st)
        return st

    def set_dense_path(self, path: str):
        """'auto' (tcgen05 int8 Ozaki kernels for float32 blocks) or 'cublas'."""
        self.check(self.lib.fsr_ctx_set_option(self.handle, 0, {"auto": 0, "tcgen05": 0, "cublas": 1}[path]))

    def set_spmm_panel(self, panel_bytes: int):
        """K2 schedule: 0 = wide row panels, 32/64/128 = L2-resident column panels."""
        self.check(self.lib.fsr_ctx_set_option(self.handle, 1, int(panel_bytes)))

    def set_topk_prune(self, on: bool):
        """Top-k-only fp32 batches: certified fp16-pruned K9 + exact re-score (True, default)
        or the unpruned fp32 K9 (False).  Both return the same top-k."""
        self.check(self.lib.fsr_ctx_set_option(self.handle, 2, int(bool(on))))
        self.topk_prune = bool(on)

    def set_topk_segments(self, segs: int):
        """Segments per row of the exact top-k when b < #SMs (0 = automatic); results identical."""
        self.check(self.lib.fsr_ctx_set_option(self.handle, 3, int(segs)))

    def set_online_path(self, path: str):
        """Preferred certified top-k path: "tc" (K9t tensor cores for b >= 128,
        the K9s stream below; default), "stream" (K9s packed fp16 U~ streamed
        from HBM, any b), "pruned" (K9h fp16 gathers) or "exact" (unpruned).
        Same results."""
        if path not in ("tc", "stream", "pruned", "exact"):
            raise ValueError(f"unknown online path {path!r}")
        self.online_path = path

    def enable_timing(self, on: bool = True):
        self.check(self.lib.fsr_ctx_enable_timing(self.handle, int(on)))
        self._timing = bool(on)

    def stage_time(self, stage: str):
        """(total ms, launches) accumulated for one stage since the last reset."""
        ms, cnt = ctypes.c_double(), _c_u64()
        self.check(self.lib.fsr_stage_time(self.handle, STAGES[stage], ctypes.byref(ms), ctypes.byref(cnt)))
        return ms.value, int(cnt.value)

    def stage_reset(self):
        self.check(self.lib.fsr_stage_reset(self.handle))

    @property
    def launches(self) -> int:
        return int(self.lib.fsr_launch_count(self.handle))

    @property
    def library_calls(self) -> int:
        return int(self.lib.fsr_library_calls(self.handle))


def ptr(t) -> _c_p:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return _c_p(0 if t is None else t.data_ptr())
