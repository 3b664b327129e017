"""Buffer plumbing between the Python API and the C ABI.

Two kinds of operands are accepted everywhere the reference accepts numpy:

* CUDA ``torch.Tensor``: used in place (zero copy); results are CUDA tensors on
  the same device, produced asynchronously on the current torch stream.
* anything numpy can read: the call goes through the C ABI's ``*_host`` entry
  points (chunked, copy/compute-overlapped streaming) or, for the small
  "pieces" API, through a device round trip; results are numpy arrays, like
  the reference's.

torch is only plumbing (device memory, streams); every byte of codec
arithmetic runs in lib/libvc3_b200.so.
"""

from __future__ import annotations

import numpy as np

try:  # torch is optional for the host-array API
    import torch
except ImportError:  # pragma: no cover - torch is in the image
    torch = None


def is_device(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def stream_of(t) -> int:
    """Raw cudaStream_t of torch's current stream on ``t``'s device."""
    return torch.cuda.current_stream(t.device).cuda_stream


class on_device:
    """Make ``t``'s CUDA device current around a C-ABI call: the library
    launches on the current device and keys its decode tables by it, so a
    tensor on another GPU than the current one needs the switch
    (torch.cuda.device guard; a no-op for host operands)."""

    def __init__(self, t):
        self._ctx = torch.cuda.device(t.device) if is_device(t) else None

    def __enter__(self):
        if self._ctx is not None:
            self._ctx.__enter__()
        return self

    def __exit__(self, *exc):
        if self._ctx is not None:
            self._ctx.__exit__(*exc)
        return False


def ptr(x) -> int:
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def device_ordinal() -> int:
    """CUDA ordinal used for host-array calls: torch's current device."""
    if torch is not None and torch.cuda.is_available():
        return torch.cuda.current_device()
    return 0


def require_torch_cuda():
    if torch is None or not torch.cuda.is_available():
        from .errors import DeviceError

        raise DeviceError("this operation needs a CUDA device (no CPU fallback)")


def upload(a: np.ndarray):
    """numpy -> CUDA tensor on the current device (synchronous wrt. ``a``)."""
    require_torch_cuda()
    return torch.from_numpy(np.ascontiguousarray(a)).to(
        device=torch.device("cuda", torch.cuda.current_device()))


def download(t) -> np.ndarray:
    return t.cpu().numpy()


def empty_like_device(shape, dtype, ref):
    return torch.empty(shape, dtype=dtype, device=ref.device)
