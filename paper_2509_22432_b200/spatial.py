"""Axis-sorted view of a cloud: the reference's slab interface
(floodph/spatial.py:19-56), kept for callers of compute_mask.

The reference selects candidate points through one axis slab per batch; the
device path replaces that with a uniform grid built on the GPU
(csrc/fph_grid.cu).  This host mirror exists so code written against the
reference's compute_mask(tri, X, sorted_cloud, batch) keeps working, and so
the empty-ball fallback (the batch's slab) sees the same slab.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import as_points


@dataclass(frozen=True)
class AxisSortedCloud:
    """Coordinates plus the stable permutation sorting them along `axis`."""

    base: np.ndarray
    axis: int
    order: np.ndarray
    sorted_coords: np.ndarray


def build_axis_sorted(cloud, axis: int) -> AxisSortedCloud:
    pts = as_points(cloud)
    if not 0 <= axis < pts.shape[1]:
        raise ValueError(f"axis must be in [0, {pts.shape[1]}), got {axis}")
    perm = np.argsort(pts[:, axis], kind="stable")
    return AxisSortedCloud(base=pts, axis=axis, order=perm, sorted_coords=pts[perm, axis])


def widest_axis(cloud) -> int:
    """The coordinate of largest extent (first one on ties)."""
    pts = as_points(cloud)
    return int(np.argmax(np.ptp(pts, axis=0)))


def slab_indices(sorted_cloud: AxisSortedCloud, lo: float, hi: float) -> np.ndarray:
    """Cloud indices whose sort-axis coordinate lies in the closed [lo, hi],
    in sort order (one contiguous run of the permutation)."""
    if lo > hi:
        raise ValueError("slab needs lo <= hi")
    first = np.searchsorted(sorted_cloud.sorted_coords, lo, side="left")
    last = np.searchsorted(sorted_cloud.sorted_coords, hi, side="right")
    return sorted_cloud.order[first:last]
