"""Device plumbing: the CUDA device, the library context, streams, tensor coercion.

PyTorch is used only for device memory, copies and streams; every arithmetic
kernel of the path lives in libbamg_b200.so.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

_ctx = None


def require_cuda():
    if not torch.cuda.is_available():
        raise _lib.NativeError("paper_2007_01941_b200 needs a CUDA device (B200); there is no CPU fallback")


_devices: dict = {}


def dev() -> torch.device:
    if not _devices:
        require_cuda()
    i = torch.cuda.current_device()
    d = _devices.get(i)
    if d is None:
        d = _devices[i] = torch.device("cuda", i)
    return d


_ctx_by_stream = {}
# the raw handle of the current stream without building a torch.cuda.Stream object
# (3 us per call on the host, paid twice per library call before)
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream() -> int:
    if _raw_stream is not None and _ctx is not None:
        return _raw_stream(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def ctx(s: int | None = None) -> int:
    """The library context of the current stream: every stream gets its own scratch
    (reduction partials, counters, device scalars), so work on concurrent streams
    never shares them."""
    global _ctx
    if _ctx is None:
        require_cuda()
        torch.cuda.init()
        _ctx = True
    if s is None:
        s = stream()
    c = _ctx_by_stream.get(s)
    if c is None:
        c = _lib.lib().bamg_ctx_create()
        if not c:
            raise _lib.NativeError(f"bamg_ctx_create failed: {_lib.last_error()}")
        _ctx_by_stream[s] = c
    return c


def call(name: str, *args):
    """Library call with the context first and the current stream last."""
    s = stream()
    return _lib.call(name, ctx(s), *args, s)


def f64(x, shape=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.to(device=dev(), dtype=torch.float64)
    else:
        t = torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64)), device=dev())
    t = t.contiguous()
    if shape is not None:
        t = t.reshape(shape)
    return t


def i32(x) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=dev(), dtype=torch.int32).contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.int32)), device=dev())


def empty(*shape, dtype=torch.float64) -> torch.Tensor:
    return torch.empty(*shape, dtype=dtype, device=dev())


def zeros(*shape, dtype=torch.float64) -> torch.Tensor:
    return torch.zeros(*shape, dtype=dtype, device=dev())


def host(t) -> np.ndarray:
    """Host numpy copy of a device tensor (API views and parity checks only)."""
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return np.asarray(t)


def scalar(t: torch.Tensor) -> float:
    return float(t.item())


def dot(x: torch.Tensor, y: torch.Tensor) -> float:
    out = empty(1)
    call("bamg_dot", x, y, x.numel(), out)
    return float(out.item())


def dot_dev(x: torch.Tensor, y: torch.Tensor, out: torch.Tensor):
    call("bamg_dot", x, y, x.numel(), out)


# optional phase timing (BAMG_PHASES=1): sync-timed, diagnostics only
PHASES: dict = {}
_PHASE_ON = bool(int(__import__("os").environ.get("BAMG_PHASES", "0")))
_last = [0.0]


def phase(name: str) -> None:
    if not _PHASE_ON:
        return
    import time

    torch.cuda.synchronize()
    t = time.perf_counter()
    if name != "start":
        PHASES[name] = PHASES.get(name, 0.0) + t - _last[0]
    _last[0] = t


def absmax(x: torch.Tensor) -> float:
    if x.numel() == 0:
        return 0.0
    out = empty(1)
    call("bamg_absmax", x, x.numel(), out)
    return float(out.item())
