"""Device plumbing: torch owns device memory and streams; no CPU fallback."""

import torch

from .errors import HpstepError


def cuda_device():
    if not torch.cuda.is_available():
        raise HpstepError("paper_2306_02526_b200 needs a CUDA device (B200, sm_100a); "
                          "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def current_stream_handle():
    return ctypes_void(torch.cuda.current_stream().cuda_stream)


def ctypes_void(v):
    import ctypes
    return ctypes.c_void_p(v)


def ndim(x):
    return x.dim() if torch.is_tensor(x) else __import__("numpy").ndim(x)
