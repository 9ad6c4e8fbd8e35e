"""numpy <-> torch plumbing for the reference-named shims: numpy inputs are
copied to the current CUDA device and results come back as numpy (the
reference works on host arrays); torch inputs stay on the device."""

from __future__ import annotations

import numpy as np
import torch

_NP2T = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
         np.dtype(np.float16): torch.float16}


def is_numpy(*xs) -> bool:
    return any(isinstance(x, np.ndarray) or (x is not None and not isinstance(x, torch.Tensor)
                                             and np.isscalar(x) is False and hasattr(x, "__len__"))
               for x in xs)


def to_dev(x, dtype=None):
    if x is None:
        return None
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.cuda()
    else:
        a = np.ascontiguousarray(np.asarray(x))
        if a.dtype not in _NP2T:
            a = a.astype(np.float64)
        t = torch.from_numpy(a).cuda()
    return t if dtype is None else t.to(dtype)


def back(t, like_numpy: bool, np_dtype=None):
    if t is None or not like_numpy:
        return t
    a = t.detach().cpu().numpy()
    return a if np_dtype is None else a.astype(np_dtype, copy=False)
