"""Helpers for the GPU parity tests: numpy uint32 patterns <-> torch int32 CUDA tensors."""
import numpy as np


def to_dev(p: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(p, dtype=np.uint32).view(np.int32)).cuda()


def to_host(t) -> np.ndarray:
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32)


def mismatch(a: np.ndarray, b: np.ndarray) -> int:
    return int(np.count_nonzero(np.asarray(a, np.uint32) != np.asarray(b, np.uint32)))
