"""Small torch plumbing: wrap raw device pointers, pick streams.

torch is used only for device memory views and stream handles; every byte
the capture path moves is moved by the native library.
"""

from __future__ import annotations


def torch():
    import torch as _t
    return _t


class _CudaBuffer:
    """Expose a raw device pointer through __cuda_array_interface__."""

    def __init__(self, ptr: int, nbytes: int) -> None:
        self.__cuda_array_interface__ = {
            "shape": (int(nbytes),),
            "typestr": "|u1",
            "data": (int(ptr), False),
            "version": 2,
        }


def bytes_tensor(ptr: int, nbytes: int, device: int):
    """A uint8 CUDA tensor aliasing [ptr, ptr+nbytes) (no copy)."""
    t = torch()
    if nbytes == 0:
        return t.empty(0, dtype=t.uint8, device=f"cuda:{device}")
    with t.cuda.device(device):
        return t.as_tensor(_CudaBuffer(ptr, nbytes), device=f"cuda:{device}")


def stream_handle(stream=None, device: int | None = None) -> int:
    """Raw cudaStream_t for a torch stream (current stream if None)."""
    t = torch()
    if stream is None:
        stream = t.cuda.current_stream(device)
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


def require_cuda() -> None:
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError(
            "no CUDA device: the capture path has no CPU fallback")
