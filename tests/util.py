"""Shared helpers for the parity tests."""
import numpy as np


def rel_err_per_channel(got: np.ndarray, ref: np.ndarray) -> float:
    """max over channels of max|got-ref| / max|ref| (error normalised per output channel by that
    channel's max |ref| -- the reference audit convention, swinflow_main.cpp:427-430,450-453)."""
    got = np.asarray(got, np.float64).reshape(ref.shape[0], -1)
    ref = np.asarray(ref, np.float64).reshape(ref.shape[0], -1)
    scale = np.maximum(np.abs(ref).max(axis=0), 1e-30)
    return float((np.abs(got - ref).max(axis=0) / scale).max())


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
