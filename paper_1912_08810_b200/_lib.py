"""ctypes binding of libsse.so (include/sse.h).

The shared library is built in-tree by ``paper_1912_08810_b200.build`` (or
``__graft_entry__.build()``).  There is no CPU fallback: if the library or a
Blackwell GPU is missing, every compute call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsse.so")

SSE_OK, SSE_EINVAL, SSE_ECUDA, SSE_ECOMM, SSE_ENOMEM = 0, 1, 2, 3, 4
IPC_HANDLE_BYTES = 64

# Exported symbols, exactly those declared in include/sse.h.
EXPORTED = (
    "sse_ctx_create",
    "sse_ctx_create_on",
    "sse_ctx_destroy",
    "sse_ctx_trim",
    "sse_last_error",
    "sse_version",
    "sse_sigma_c128",
    "sse_sigma_c128_slab",
    "sse_sigma_device",
    "sse_sigma_device_scatter",
    "sse_sigma_device_peer",
    "sse_pi_device_peer",
    "sse_slab_from_points",
    "sse_dev_alloc",
    "sse_dev_free",
    "sse_ipc_handle",
    "sse_ipc_open",
    "sse_ipc_close",
    "sse_pi_c128",
    "sse_pi_device",
    "sse_phase_c128",
    "sse_phase_device",
    "sse_layout_transform",
    "sse_preprocess_D",
    "sse_fill_synthetic",
    "sse_profile_begin",
    "sse_profile_end",
    "sse_kernel_name",
    "sse_multi_layout",
    "sse_sigma_multi",
)

PROF_KINDS = ("operator", "sigma", "layout", "preprocess", "pi_build", "pi", "pi_assemble")


class SseDims(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("nkz", "nqz", "ne", "nw", "na", "nb", "norb")]


class SseSlab(ctypes.Structure):
    _fields_ = [
        ("atom0", ctypes.c_int64),
        ("natoms", ctypes.c_int64),
        ("atom_major", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class SseTiming(ctypes.Structure):
    _fields_ = [
        ("h2d_ms", ctypes.c_double),
        ("prep_ms", ctypes.c_double),
        ("sigma_ms", ctypes.c_double),
        ("d2h_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("flops", ctypes.c_double),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int32),
        ("n_devices", ctypes.c_int32),
        ("staged", ctypes.c_int32),
        ("host_threads", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class SseProfile(ctypes.Structure):
    _fields_ = [
        ("ms", ctypes.c_double * 7),
        ("flops", ctypes.c_double * 7),
        ("launches", ctypes.c_int64 * 7),
    ]

    def as_dict(self) -> dict:
        return {
            kind: {"ms": self.ms[i], "flops": self.flops[i], "launches": int(self.launches[i])}
            for i, kind in enumerate(PROF_KINDS)
        }


class SseError(RuntimeError):
    """CUDA / communication failure inside libsse (codes 2, 3)."""


_P = ctypes.c_void_p
_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load libsse.so once; raise ImportError if it was not built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(LIB_PATH)
        i64, i32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        pdims, pslab, ptim = ctypes.POINTER(SseDims), ctypes.POINTER(SseSlab), ctypes.POINTER(SseTiming)
        lib.sse_ctx_create.argtypes = [i32, ctypes.POINTER(_P)]
        lib.sse_ctx_create_on.argtypes = [i32, ctypes.POINTER(_P)]
        lib.sse_ctx_destroy.argtypes = [_P]
        lib.sse_ctx_destroy.restype = None
        lib.sse_ctx_trim.argtypes = [_P]
        lib.sse_last_error.restype = ctypes.c_char_p
        lib.sse_version.restype = i32
        lib.sse_sigma_c128.argtypes = [_P, pdims, i32] + [_P] * 7 + [_P, _P, _P, ptim]
        lib.sse_sigma_c128_slab.argtypes = [_P, pdims, i32, pslab, pslab] + [_P] * 7 + [_P, _P, _P, ptim]
        lib.sse_pi_c128.argtypes = [_P, pdims, _P, _P, _P, _P, _P, dbl, _P, i64, i64, _P, _P, ptim]
        lib.sse_pi_device.argtypes = [_P, pdims, pslab, pslab, _P, _P, _P, _P, _P, dbl, _P, _P, _P, _P, ptim]
        lib.sse_phase_c128.argtypes = [_P, pdims] + [_P] * 8 + [dbl] + [_P] * 4 + [ptim]
        lib.sse_phase_device.argtypes = [_P, pdims, pslab, pslab] + [_P] * 8 + [dbl] + [_P] * 5 + [ptim]
        lib.sse_profile_begin.argtypes = [_P]
        lib.sse_profile_end.argtypes = [_P, ctypes.POINTER(SseProfile)]
        lib.sse_sigma_device.argtypes = [_P, pdims, pslab, pslab] + [_P] * 6 + [_P, _P, _P, _P, _P, ptim]
        lib.sse_sigma_device_scatter.argtypes = [_P, pdims, pslab, pslab] + [_P] * 8 + [i32, _P, _P, _P, _P, ptim]
        lib.sse_sigma_device_peer.argtypes = [_P, pdims, pslab, _P, _P] + [_P] * 6 + [i32, _P, _P, _P, _P, ptim]
        lib.sse_pi_device_peer.argtypes = [_P, pdims, pslab, _P, _P, _P, _P, _P, dbl, i32, _P, _P, _P, _P, ptim]
        lib.sse_slab_from_points.argtypes = [_P, pdims, pslab, i32, _P, _P, i32, _P, _P]
        lib.sse_dev_alloc.argtypes = [_P, ctypes.c_size_t, ctypes.POINTER(_P)]
        lib.sse_dev_free.argtypes = [_P, _P]
        lib.sse_ipc_handle.argtypes = [_P, _P, ctypes.c_char_p]
        lib.sse_ipc_open.argtypes = [_P, ctypes.c_char_p, ctypes.POINTER(_P)]
        lib.sse_ipc_close.argtypes = [_P, _P]
        lib.sse_layout_transform.argtypes = [_P, i64, i64, i64, i64, i32, _P, _P, _P]
        lib.sse_preprocess_D.argtypes = [_P, i64, i64, i64, i64, _P, i64, i64, i64, i64, _P, _P, _P]
        lib.sse_fill_synthetic.argtypes = [
            _P, ctypes.c_uint64, ctypes.c_uint32, i64, i64, i64, i64, i64, i64, dbl, _P, _P,
        ]
        lib.sse_multi_layout.argtypes = [_P, pdims, _P, _P]
        lib.sse_sigma_multi.argtypes = [_P, pdims] + [_P] * 5 + [_P, _P, _P] + [_P, _P, ptim]
        lib.sse_kernel_name.argtypes = [i32]
        lib.sse_kernel_name.restype = ctypes.c_char_p
        for name in EXPORTED:
            if name not in ("sse_ctx_destroy", "sse_last_error", "sse_kernel_name"):
                getattr(lib, name).restype = i32
        _lib = lib
        return lib


def kernel_name(kind: str) -> str:
    """Name of the kernel of ``kind`` (one of PROF_KINDS) libsse launched last in this process."""
    return load().sse_kernel_name(PROF_KINDS.index(kind)).decode()


def check(rc: int) -> None:
    """Map a libsse return code to the reference's exception convention."""
    if rc == SSE_OK:
        return
    msg = load().sse_last_error().decode(errors="replace")
    if rc == SSE_EINVAL:
        raise ValueError(msg)
    if rc == SSE_ENOMEM:
        raise MemoryError(msg)
    raise SseError(f"libsse error {rc}: {msg}")


class Context:
    """Owns an ``sse_ctx`` (per-device stream and cached device buffers)."""

    def __init__(self, n_gpus: int = 1, device: int | None = None):
        lib = load()
        handle = _P()
        if device is not None:
            check(lib.sse_ctx_create_on(int(device), ctypes.byref(handle)))
        else:
            check(lib.sse_ctx_create(int(n_gpus), ctypes.byref(handle)))
        self.handle = handle
        self.n_gpus = 1 if device is not None else int(n_gpus)
        self.device = device

    def trim(self) -> None:
        """Hand the cached device scratch and pinned staging back (sse_ctx_trim); the next call
        allocates again."""
        if self.handle:
            check(load().sse_ctx_trim(self.handle))

    def close(self) -> None:
        if self.handle:
            load().sse_ctx_destroy(self.handle)
            self.handle = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_contexts: dict = {}


def context(n_gpus: int = 1, device: int | None = None) -> Context:
    """Process-wide cached context (device buffers are reused across calls)."""
    if device is None and n_gpus == 1:
        device = 0  # one context (and one set of cached device buffers) per device
    key = ("dev", device) if device is not None else ("n", n_gpus)
    with _lock:
        ctx = _contexts.get(key)
    if ctx is None:
        ctx = Context(n_gpus=n_gpus, device=device)
        with _lock:
            _contexts[key] = ctx
    return ctx
