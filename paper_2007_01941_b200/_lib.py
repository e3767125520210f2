"""ctypes binding of libbamg_b200.so (the C ABI in include/bamg_b200.h).

The argument types are derived from the header itself, so the Python side and
the exported symbols cannot drift apart silently. There is no fallback: if the
library or a CUDA device is missing, every call raises.
"""

from __future__ import annotations

import ctypes
import os
import re
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.environ.get("BAMG_LIB") or os.path.join(HERE, "libbamg_b200.so")  # BAMG_LIB: A/B variant builds
HEADER = os.path.join(ROOT, "include", "bamg_b200.h")

BAMG_ERR_INDEFINITE = 1
BAMG_ERR_BEHIND = 2
BAMG_ERR_NOT_PD = 3
BAMG_ERR_UNSUPPORTED = 4


class NativeError(RuntimeError):
    """A CUDA or launch failure inside libbamg_b200."""


_SCALAR = {
    "int": ctypes.c_int32,
    "int32_t": ctypes.c_int32,
    "int64_t": ctypes.c_int64,
    "double": ctypes.c_double,
    "size_t": ctypes.c_size_t,
}


def parse_header(path: str = HEADER) -> dict[str, tuple[str, list[str]]]:
    """Map function name -> (return type, [param types]) for every bamg_* prototype."""
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", " ", text, flags=re.S)
    protos = {}
    for m in re.finditer(r"(\w[\w\s\*]*?)\s*\b(bamg_\w+)\s*\(([^;{]*?)\)\s*;", text, flags=re.S):
        ret, name, params = m.group(1).strip(), m.group(2), m.group(3)
        ptypes = []
        params = params.strip()
        if params and params != "void":
            for p in params.split(","):
                p = " ".join(p.split())
                p = re.sub(r"\b\w+$", "", p).strip() if not p.endswith("*") else p
                ptypes.append(p)
        protos[name] = (ret, ptypes)
    return protos


def _ctype(t: str):
    t = t.replace("const", "").strip()
    if "*" in t:
        return ctypes.c_void_p
    return _SCALAR[t]


def _rtype(t: str):
    t = t.strip()
    if t.endswith("*"):
        return ctypes.c_void_p
    if t == "void":
        return None
    return _SCALAR[t]


_lock = threading.Lock()
_lib = None
_protos = None


def lib():
    global _lib, _protos
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2007_01941_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        protos = parse_header()
        for name, (ret, params) in protos.items():
            fn = getattr(L, name)
            fn.restype = _rtype(ret)
            fn.argtypes = [_ctype(p) for p in params]
        _protos = protos
        _lib = L
    return _lib


def prototypes():
    lib()
    return _protos


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    lib().bamg_last_error(buf, 1024)
    return buf.value.decode(errors="replace")


def _arg(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a


_fns: dict = {}


def call(name: str, *args) -> int:
    """Invoke a bamg_* entry point; torch tensors pass their device pointers.

    Raises NativeError on CUDA failures (rc < 0) and returns domain codes (> 0)
    to the caller, which maps them onto the reference exception classes.
    """
    fn = _fns.get(name)
    if fn is None:
        fn = _fns[name] = getattr(lib(), name)
    rc = fn(*[a.data_ptr() if hasattr(a, "data_ptr") else a for a in args])
    if rc is None:
        return 0
    if isinstance(rc, float):
        return rc
    if rc < 0:
        raise NativeError(f"{name}: {last_error()}")
    if rc == BAMG_ERR_UNSUPPORTED:
        raise NativeError(f"{name}: unsupported size: {last_error()}")
    return rc
