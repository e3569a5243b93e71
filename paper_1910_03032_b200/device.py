"""Device plumbing: torch owns device memory and streams; the C-ABI computes.

Vectors on the device are ``torch.float64`` CUDA tensors.  Host numpy
arrays crossing the API are copied in and out around the call, which is the
drop-in behaviour the reference's tests exercise (``op.apply(numpy) ->
numpy``).
"""

import numpy as np
import torch

_DEVICE = None
_PINNED_MIN_BYTES = 1 << 20  # host arrays from 1 MB up cross through pinned memory


def device():
    global _DEVICE
    if _DEVICE is None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1910_03032_b200 needs a CUDA device (sm_100a); none is visible")
        _DEVICE = torch.device("cuda", torch.cuda.current_device())
    return _DEVICE


def stream_handle():
    return torch.cuda.current_stream(device()).cuda_stream


def is_device_tensor(x):
    return isinstance(x, torch.Tensor) and x.is_cuda


def to_device(x, dtype=torch.float64):
    """numpy / torch -> contiguous CUDA tensor of `dtype` (no copy if already)."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=device(), dtype=dtype)
        return t.contiguous()
    arr = np.ascontiguousarray(x, dtype=np.float64 if dtype == torch.float64 else None)
    src = torch.from_numpy(arr)
    if arr.nbytes >= _PINNED_MIN_BYTES:
        # stage through page-locked memory from torch's caching host allocator:
        # a threaded host copy, then an async H2D in stream order (the block
        # is not reused before that copy completes)
        h = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
        h.copy_(src)
        return h.to(device(), non_blocking=True)
    return src.to(device())


def empty(n, dtype=torch.float64):
    return torch.empty(n, dtype=dtype, device=device())


def zeros(n, dtype=torch.float64):
    return torch.zeros(n, dtype=dtype, device=device())


def to_host(t):
    """CUDA tensor -> numpy.  Large results land in page-locked memory from
    torch's caching host allocator (a D2H at PCIe speed, no page faults on a
    fresh array: 80 MB 38 -> ~2 ms, tools/host_copy_probe.py); the array keeps
    its pinned block alive and the block returns to the cache with it."""
    t = t.detach()
    if t.is_cuda and t.numel() * t.element_size() >= _PINNED_MIN_BYTES:
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        torch.cuda.current_stream(t.device).synchronize()
        return h.numpy()
    return t.cpu().numpy()


class DeviceIn:
    """Normalise an operand: returns (device tensor, was_host)."""

    @staticmethod
    def get(x):
        if is_device_tensor(x):
            if x.dtype != torch.float64:
                raise ValueError(f"operand dtype {x.dtype}, expected float64")
            return x.contiguous(), False
        return to_device(x), True
