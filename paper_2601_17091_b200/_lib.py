"""Loader of the in-tree CUDA library (the C ABI in include/rocket_b200.h).

The product path goes only through this library: there is no CPU fallback.
If the library is missing or no B200 is visible, every transform raises.
"""

import ctypes
import os
import subprocess
import sys

_PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(_PKG)
LIB_PATH = os.environ.get("RK_LIB_PATH") or os.path.join(_PKG, "_build", "librocket_b200.so")
# the checked build (-DRK_CHECKED: device-side bounds checks that trap on a
# bad shared/global access; compute-sanitizer is closed on the GPU pool)
CHECKED_LIB_PATH = os.path.join(_PKG, "_build", "librocket_b200_checked.so")
CSRC = os.path.join(_PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")

RK_OK = 0
RK_ERR_INVALID = 1
RK_ERR_CAPACITY = 2
RK_ERR_CUDA = 3
RK_ERR_UNSUPPORTED = 4
RK_ERR_NO_DEVICE = 5
RK_MODE_EXACT = 0
RK_MODE_FAST = 1
MODES = {"exact": RK_MODE_EXACT, "fast": RK_MODE_FAST}
RK_DTYPE_F32 = 0
RK_DTYPE_F64 = 1

# Every symbol include/rocket_b200.h declares.
EXPORTS = (
    "rk_abi_version",
    "rk_last_error",
    "rk_device_count",
    "rk_bank_create",
    "rk_bank_destroy",
    "rk_bank_info",
    "rk_bank_attach_f64",
    "rk_transform",
    "rk_transform_f32",
    "rk_run_batch_f32",
    "rk_run_batch_f64",
    "rk_run_batch_f32_mode",
    "rk_run_batch_f64_mode",
    "rk_release_caches",
    "rk_transform_stream",
    "rk_generate_bank",
)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    # IEEE float semantics are part of the parity contract: no fast math,
    # keep denormals, IEEE division.
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
]


class BankInfo(ctypes.Structure):
    _fields_ = [
        ("n_kernels", ctypes.c_int64),
        ("n_channels", ctypes.c_int32),
        ("l_series", ctypes.c_int32),
        ("n_groups", ctypes.c_int32),
        ("n_chunks", ctypes.c_int32),
        ("halo", ctypes.c_int32),
        ("smem_bytes", ctypes.c_int32),
        ("positions_per_series", ctypes.c_int64),
        ("useful_flops_per_series", ctypes.c_int64),
        ("device_bytes", ctypes.c_int64),
        ("device", ctypes.c_int32),
        ("n_launches", ctypes.c_int32),
        ("path", ctypes.c_int32),
        ("ctas_per_sm", ctypes.c_int32),
        ("n_half_chunks", ctypes.c_int32),
        ("n_paired_chunks", ctypes.c_int32),
        ("n_quarter_chunks", ctypes.c_int32),
        ("n_eighth_chunks", ctypes.c_int32),
        ("n_runmajor_chunks", ctypes.c_int32),
    ]


def build(verbose=False, out=None, defines=()):
    """Compile the CUDA library in-tree for sm_100a (nvcc cross-compiles
    without a GPU): the host runtime and the three per-length kernel units
    are compiled in parallel, then linked into one shared library."""
    out = out or LIB_PATH
    objdir = os.path.join(os.path.dirname(out), "obj_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    flags = [*NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", INCLUDE]
    units = [("rocket_b200.o", os.path.join(CSRC, "rocket_b200.cu"), []),
             ("rocket_stream.o", os.path.join(CSRC, "rocket_stream.cu"), []),
             # host-only; no FMA contraction so the doubles round like numpy's
             ("bank_gen.o", os.path.join(CSRC, "bank_gen.cpp"), ["-Xcompiler", "-ffp-contract=off"])]
    # one unit per (tap length, R class): 24 template-heavy units in parallel
    units += [(f"kernels_len{n}_r{ri}.o", os.path.join(CSRC, "kernels_len.cu"), [f"-DRK_LEN={n}", f"-DRK_RI={ri}"])
              for n in (7, 9, 11) for ri in range(8)]
    jobs = max(1, os.cpu_count() or 1)
    running, failed = [], []
    for obj, src, extra in units:
        cmd = ["nvcc", *flags, *extra, "-c", "-o", os.path.join(objdir, obj), src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        while len(running) >= jobs:
            c, p = running.pop(0)
            if p.wait() != 0:
                failed.append(c)
        running.append((cmd, subprocess.Popen(cmd)))
    for c, p in running:
        if p.wait() != 0:
            failed.append(c)
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    link = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out,
            *[os.path.join(objdir, obj) for obj, _, _ in units]]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.run(link, check=True)
    return out


_lib = None


def load():
    """The loaded ctypes library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"CUDA library {LIB_PATH} is missing; run __graft_entry__.build() "
            "(there is no CPU fallback for the transform)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    p = ctypes.c_void_p
    i64 = ctypes.c_int64
    i32 = ctypes.c_int32
    lib.rk_abi_version.restype = ctypes.c_int
    lib.rk_abi_version.argtypes = []
    lib.rk_last_error.restype = ctypes.c_char_p
    lib.rk_last_error.argtypes = []
    lib.rk_device_count.restype = ctypes.c_int
    lib.rk_device_count.argtypes = [ctypes.POINTER(i32)]
    lib.rk_bank_create.restype = ctypes.c_int
    lib.rk_bank_create.argtypes = [i64, i32, i32, p, p, p, p, p, p, p, p, p, i32, ctypes.POINTER(p)]
    lib.rk_bank_destroy.restype = ctypes.c_int
    lib.rk_bank_destroy.argtypes = [p]
    lib.rk_bank_info.restype = ctypes.c_int
    lib.rk_bank_info.argtypes = [p, ctypes.POINTER(BankInfo)]
    lib.rk_bank_attach_f64.restype = ctypes.c_int
    lib.rk_bank_attach_f64.argtypes = [p, p, p]
    lib.rk_transform.restype = ctypes.c_int
    lib.rk_transform.argtypes = [p, p, i32, i64, p, i64, i64, i32, i32, p, ctypes.POINTER(i64)]
    lib.rk_run_batch_f64.restype = i64
    lib.rk_run_batch_f64.argtypes = [p, i64, i32, i32, p, p, p, p, p, p, p, p, p, i64, i32, i32, p, i64, i64]
    lib.rk_transform_f32.restype = ctypes.c_int
    lib.rk_transform_f32.argtypes = [p, p, i64, p, i64, i64, i32, i32, p, ctypes.POINTER(i64)]
    lib.rk_transform_stream.restype = ctypes.c_int
    lib.rk_transform_stream.argtypes = [p, i32, i64, p, i32, i64, i32, i64, i32, i32, i32, i64, ctypes.POINTER(i64)]
    lib.rk_generate_bank.restype = ctypes.c_int
    lib.rk_generate_bank.argtypes = [i64, i32, i32, ctypes.c_uint64, i32, p, ctypes.c_double, p, p, p, p, p, p, i64,
                                     p, i64, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.rk_run_batch_f32.restype = i64
    lib.rk_run_batch_f32.argtypes = [p, i64, i32, i32, p, p, p, p, p, p, p, p, p, i64, i32, i32, p, i64, i64]
    lib.rk_run_batch_f32_mode.restype = i64
    lib.rk_run_batch_f32_mode.argtypes = [p, i64, i32, i32, p, p, p, p, p, p, p, p, p, i64, i32, i32, p, i64, i64, i32]
    lib.rk_run_batch_f64_mode.restype = i64
    lib.rk_run_batch_f64_mode.argtypes = [p, i64, i32, i32, p, p, p, p, p, p, p, p, p, i64, i32, i32, p, i64, i64, i32]
    lib.rk_release_caches.restype = ctypes.c_int
    lib.rk_release_caches.argtypes = []
    _lib = lib
    return lib


def last_error():
    return load().rk_last_error().decode(errors="replace")


def device_count():
    n = ctypes.c_int32(0)
    load().rk_device_count(ctypes.byref(n))
    return int(n.value)


def check(rc, what):
    """Map an RK_ERR_* code to the reference's exception types."""
    if rc == RK_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == RK_ERR_CAPACITY:
        from .engine import CapacityError

        raise CapacityError(msg)
    if rc == RK_ERR_INVALID:
        raise ValueError(msg)
    if rc == RK_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)
