"""Host overhead per library call / allocation (dev tool)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2007_01941_b200 import _device as D  # noqa: E402
from paper_2007_01941_b200 import _lib  # noqa: E402

x = D.empty(16)
y = D.empty(16)
D.call("bamg_axpby", 1.0, x, 1.0, y, 16)
torch.cuda.synchronize()


def t(name, f, n=20000):
    f()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    dt = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    print(f"{name:40s} {dt:7.2f} us", flush=True)


t("torch.cuda.current_stream()", lambda: torch.cuda.current_stream())
t("current_stream().cuda_stream", lambda: torch.cuda.current_stream().cuda_stream)
t("torch.cuda.current_device()", lambda: torch.cuda.current_device())
t("torch.cuda.is_available()", lambda: torch.cuda.is_available())
t("D.dev()", D.dev)
t("D.ctx()", D.ctx)
t("D.empty(16)", lambda: D.empty(16))
t("torch.empty(16, device=cuda)", lambda: torch.empty(16, dtype=torch.float64, device="cuda"))
t("x.data_ptr()", lambda: x.data_ptr())
fn = _lib.lib().bamg_axpby
c, s = D.ctx(), D.stream()
px, py = x.data_ptr(), y.data_ptr()
t("raw ctypes axpby", lambda: fn(c, 1.0, px, 1.0, py, 16, s))
t("_lib.call axpby", lambda: _lib.call("bamg_axpby", c, 1.0, x, 1.0, y, 16, s))
t("D.call axpby", lambda: D.call("bamg_axpby", 1.0, x, 1.0, y, 16))
t("x[:8]", lambda: x[:8])
t("int(t.item()) (sync)", lambda: int(y[:1].item()), 2000)
