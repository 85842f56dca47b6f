"""ctypes binding of the C ABI in include/nnb.h (libnnb.so, built in-tree).

This is the Python side of the boundary that replaces the reference's
``ENTRY_SIGNATURE = CFUNCTYPE(None, c_void_p, c_void_p)`` call into generated
x86 code (pkg/src/nnjit/codegen/executable.py:28, 47-50).  There is no
fallback: if the library is missing the import of the runtime fails loudly.
"""

import ctypes
import os
import pathlib

from .errors import CompileError, DeviceError, InputShapeMismatch, UnsupportedDevice

PKG_DIR = pathlib.Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libnnb.so"
KERNEL_DIR = PKG_DIR / "csrc" / "kernels"

NNB_OK, NNB_ERR_ARGUMENT, NNB_ERR_NO_DRIVER, NNB_ERR_NO_DEVICE, NNB_ERR_ARCH, \
    NNB_ERR_NVRTC, NNB_ERR_CUDA, NNB_ERR_OOM, NNB_ERR_BATCH = range(9)

EXPORTED = ("nnb_device_check", "nnb_compile", "nnb_compile_parallel", "nnb_create", "nnb_arena_ptr", "nnb_apply",
            "nnb_run_host", "nnb_enqueue_host", "nnb_run_host_chunked", "nnb_sync", "nnb_time_apply", "nnb_time_launch", "nnb_time_sequence", "nnb_ffma_peak", "nnb_host_alloc", "nnb_host_free",
            "nnb_free", "nnb_net_info", "nnb_last_error", "nnb_abi_version", "nnb_destroy")


MAX_TMAPS = 6          # NNB_MAX_TMAPS


class TMap(ctypes.Structure):
    _fields_ = [("space", ctypes.c_uint32), ("swizzle", ctypes.c_uint32),
                ("offset", ctypes.c_uint64), ("rank", ctypes.c_uint32),
                ("box", ctypes.c_uint32 * 4), ("dims", ctypes.c_uint64 * 4),
                ("strides", ctypes.c_uint64 * 3)]


def make_tmap(t):
    """TMap from the dict the specialiser emits: space, offset, dims, strides, box."""
    r = len(t["dims"])
    box = (ctypes.c_uint32 * 4)(*(list(t["box"]) + [1] * (4 - r)))
    dims = (ctypes.c_uint64 * 4)(*(list(t["dims"]) + [1] * (4 - r)))
    strides = (ctypes.c_uint64 * 3)(*(list(t["strides"]) + [0] * (3 - len(t["strides"]))))
    return TMap(t["space"], t.get("swizzle", 3), t["offset"], r, box, dims, strides)


class Launch(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int32), ("block", ctypes.c_uint32),
                ("smem_bytes", ctypes.c_uint32), ("grid_mult", ctypes.c_uint32),
                ("items_per_image", ctypes.c_uint64), ("items_per_block", ctypes.c_uint64),
                ("n_min", ctypes.c_int32), ("n_max", ctypes.c_int32),
                ("grid_cap", ctypes.c_uint32), ("n_tmaps", ctypes.c_uint32),
                ("tmaps", TMap * MAX_TMAPS), ("cluster", ctypes.c_uint32),
                ("cooperative", ctypes.c_uint32), ("zero_offset", ctypes.c_int64)]


class IO(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_uint64), ("image_bytes", ctypes.c_uint64)]


class NetDesc(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("sources", ctypes.POINTER(ctypes.c_char_p)),
                ("n_sources", ctypes.c_int32),
                ("include_dir", ctypes.c_char_p), ("cache_dir", ctypes.c_char_p),
                ("kernel_names", ctypes.POINTER(ctypes.c_char_p)),
                ("kernel_source", ctypes.POINTER(ctypes.c_int32)), ("n_kernels", ctypes.c_int32),
                ("launches", ctypes.POINTER(Launch)), ("n_launches", ctypes.c_int32),
                ("pool", ctypes.c_void_p), ("pool_bytes", ctypes.c_uint64),
                ("arena_bytes", ctypes.c_uint64), ("max_batch", ctypes.c_int32),
                ("inputs", ctypes.POINTER(IO)), ("n_inputs", ctypes.c_int32),
                ("outputs", ctypes.POINTER(IO)), ("n_outputs", ctypes.c_int32)]


_lib = None


def lib():
    """Load libnnb.so (raises ImportError with the build hint if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                          "g.build()'` (or python -m paper_1906_05737_b200.build)")
    L = ctypes.CDLL(str(LIB_PATH))
    P, I32, U64, VP = ctypes.POINTER, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p
    sig = {
        "nnb_device_check": (I32, [I32, P(I32), P(I32), P(I32)]),
        "nnb_compile": (I32, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, P(VP), P(U64),
                              P(ctypes.c_double)]),
        "nnb_compile_parallel": (I32, [P(ctypes.c_char_p), I32, ctypes.c_char_p, ctypes.c_char_p,
                                       P(ctypes.c_double), P(ctypes.c_double)]),
        "nnb_create": (I32, [P(NetDesc), P(VP)]),
        "nnb_arena_ptr": (I32, [VP, U64, P(VP)]),
        "nnb_apply": (I32, [VP, I32, VP]),
        "nnb_run_host": (I32, [VP, I32, P(VP), P(VP), VP]),
        "nnb_enqueue_host": (I32, [VP, I32, P(VP), P(VP), VP]),
        "nnb_run_host_chunked": (I32, [P(VP), P(VP), I32, ctypes.c_int64, P(VP), P(VP)]),
        "nnb_sync": (I32, [VP, VP]),
        "nnb_time_apply": (I32, [VP, I32, I32, VP, P(ctypes.c_double)]),
        "nnb_time_launch": (I32, [VP, I32, I32, I32, VP, P(ctypes.c_double)]),
        "nnb_time_sequence": (I32, [VP, I32, I32, VP, P(ctypes.c_double)]),
        "nnb_ffma_peak": (I32, [I32, I32, P(ctypes.c_double), P(ctypes.c_double)]),
        "nnb_host_alloc": (I32, [U64, P(VP)]),
        "nnb_host_free": (None, [VP]),
        "nnb_free": (None, [VP]),
        "nnb_net_info": (I32, [VP, P(U64), P(U64), P(I32), P(ctypes.c_double), P(I32)]),
        "nnb_last_error": (ctypes.c_char_p, []),
        "nnb_abi_version": (I32, []),
        "nnb_destroy": (None, [VP]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    _lib = L
    return L


def check(status, what=""):
    """Map an nnb_status onto the NnjitError tree."""
    if status == NNB_OK:
        return
    msg = lib().nnb_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status in (NNB_ERR_NO_DRIVER, NNB_ERR_NO_DEVICE, NNB_ERR_ARCH):
        raise UnsupportedDevice(msg)
    if status == NNB_ERR_NVRTC:
        raise CompileError(msg)
    if status == NNB_ERR_BATCH:
        raise InputShapeMismatch(msg)
    if status == NNB_ERR_ARGUMENT:
        raise ValueError(msg)
    raise DeviceError(status, msg)


def device_check(device=0):
    """Capability gate (replaces codegen/hostcheck.check_host)."""
    a, b, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    check(lib().nnb_device_check(device, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return a.value, b.value, c.value


def default_cache_dir():
    d = os.environ.get("NNB_CACHE_DIR")
    if d:
        return d
    return str(pathlib.Path.home() / ".cache" / "nnb_cubins")


def compile_source(source, cache_dir=None):
    """NVRTC-compile a translation unit for sm_100a; returns (cubin bytes, ms).
    Needs no GPU."""
    ptr, n, ms = ctypes.c_void_p(), ctypes.c_uint64(), ctypes.c_double()
    check(lib().nnb_compile(source.encode(), str(KERNEL_DIR).encode(),
                            cache_dir.encode() if cache_dir else None,
                            ctypes.byref(ptr), ctypes.byref(n), ctypes.byref(ms)), "nnb_compile")
    try:
        data = ctypes.string_at(ptr.value, n.value)
    finally:
        lib().nnb_free(ptr)
    return data, ms.value


def compile_parallel(sources, cache_dir=None):
    """NVRTC-compile translation units on the runtime's own job pool (what
    nnb_create does); returns (wall ms, sum of per-source ms).  No GPU."""
    arr = (ctypes.c_char_p * max(len(sources), 1))(*[s.encode() for s in sources])
    wall, tot = ctypes.c_double(), ctypes.c_double()
    check(lib().nnb_compile_parallel(arr, len(sources), str(KERNEL_DIR).encode(),
                                     cache_dir.encode() if cache_dir else None,
                                     ctypes.byref(wall), ctypes.byref(tot)), "nnb_compile_parallel")
    return wall.value, tot.value


def ffma_peak(device=0, iters=4096):
    """Measured FP32 FFMA TFLOP/s of `device` (nnb_ffma_peak) and the ms of
    the best timed launch."""
    tf, ms = ctypes.c_double(), ctypes.c_double()
    check(lib().nnb_ffma_peak(device, iters, ctypes.byref(tf), ctypes.byref(ms)), "nnb_ffma_peak")
    return tf.value, ms.value
