"""Host <-> device copy paths for the numpy drop-in call (op.apply(numpy)):
torch's pageable copies vs staging through a cached pinned buffer."""
import time

import numpy as np
import torch

n = 10_000_000
x = np.random.default_rng(0).standard_normal(n)
d = torch.empty(n, dtype=torch.float64, device="cuda")
pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
pnp = pin.numpy()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - a)
    return round(1e3 * sorted(ts)[len(ts) // 2], 2)


def h2d_pageable():
    return torch.from_numpy(x).to("cuda")


def h2d_staged():
    np.copyto(pnp, x)
    d.copy_(pin, non_blocking=True)


def d2h_pageable():
    return d.cpu().numpy()


def d2h_staged():
    pin.copy_(d, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return pnp.copy()


def d2h_staged_empty():
    pin.copy_(d, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    out = np.empty(n)
    np.copyto(out, pnp)
    return out


print({"MB": n * 8 / 1e6, "h2d_pageable_ms": t(h2d_pageable), "h2d_staged_ms": t(h2d_staged),
       "d2h_pageable_ms": t(d2h_pageable), "d2h_staged_ms": t(d2h_staged),
       "d2h_staged_empty_ms": t(d2h_staged_empty),
       "host_copy_ms": t(lambda: np.copyto(pnp, x)), "new_array_ms": t(lambda: x.copy())})

import sys  # noqa: E402
sys.path.insert(0, ".")
from paper_1910_03032_b200 import device as dev  # noqa: E402
print({"d2h_to_host_ms": t(lambda: dev.to_host(d)),
       "d2h_to_host_matches": bool(np.array_equal(dev.to_host(d), d.cpu().numpy()))})
print({"h2d_to_device_ms": t(lambda: dev.to_device(x)),
       "h2d_to_device_matches": bool(np.array_equal(dev.to_device(x).cpu().numpy(), x)),
       "torch_threads": torch.get_num_threads()})
