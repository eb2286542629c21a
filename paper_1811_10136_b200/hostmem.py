"""Page-locked (pinned) host arrays for the inputs of register().

A cloud whose float64 rows live in pinned memory is uploaded by one DMA at
PCIe rate straight from the caller's buffer (fr_upload_rows64 detects it), not
through the threaded staging copy a pageable NumPy array needs -- on the
benchmark box the staging copy is host-memory bound at ~20 GB/s, the DMA runs
at ~53 GB/s.  `load_cloud(..., pinned=True)` parses PLY / XYZ files straight
into such buffers (the reference reader, io.py:52-64, returns pageable
arrays)."""

from __future__ import annotations

import numpy as np

from .geometry import PointCloud


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """An uninitialised page-locked host array (a NumPy view of a pinned torch
    tensor; the array keeps the tensor, and so the pinned block, alive)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("pinned host memory needs a CUDA device")
    tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32}[
        np.dtype(dtype)]
    return torch.empty(tuple(shape), dtype=tdt, pin_memory=True).numpy()


def pinned_copy(a) -> np.ndarray:
    """A page-locked float64 copy of `a`."""
    a = np.asarray(a, dtype=np.float64)
    out = pinned_empty(a.shape)
    np.copyto(out, a)
    return out


def pinned_cloud(cloud: PointCloud) -> PointCloud:
    """`cloud` with its arrays copied into page-locked host memory."""
    return PointCloud(pinned_copy(cloud.positions),
                      normals=None if cloud.normals is None else pinned_copy(cloud.normals),
                      features=cloud.features)
