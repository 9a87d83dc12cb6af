"""Pinhole cameras, restated from the reference.

* ``Camera``          — pkg/src/landmark/data_io.py:42-70 (same fields, same
  validation, same ``center`` = -R^T t computed in numpy fp64).
* ``look_at_camera``  — pkg/src/landmark/data_io.py:73-89.
* ``camera_constants``— the per-view scalars the reference derives inside
  ``project_splats`` (gaussian_core.py:208-209: lim_x / lim_y) computed on the
  host in fp64 exactly as the reference does, so the kernels receive them as
  launch arguments (constant bank) instead of recomputing them per thread.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InvalidInputError


@dataclass
class Camera:
    """Pinhole camera: intrinsics plus world-to-camera rigid pose."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    r_wc: np.ndarray  # (3, 3) world-to-camera rotation (rows = right, down, forward)
    t_wc: np.ndarray  # (3,) world-to-camera translation
    near: float = 0.05
    far: float = 100.0

    def __post_init__(self):
        self.r_wc = np.asarray(self.r_wc, dtype=np.float64).reshape(3, 3)
        self.t_wc = np.asarray(self.t_wc, dtype=np.float64).reshape(3)
        if self.fx <= 0 or self.fy <= 0:
            raise InvalidInputError("focal lengths must be positive")
        if not 0 < self.near < self.far:
            raise InvalidInputError("require 0 < near < far")

    @property
    def center(self) -> np.ndarray:
        return -self.r_wc.T @ self.t_wc

    def world_to_cam(self, points: np.ndarray) -> np.ndarray:
        return points @ self.r_wc.T + self.t_wc

    @classmethod
    def from_reference(cls, cam) -> "Camera":
        """Adopt a reference ``landmark.data_io.Camera`` (duck-typed)."""
        return cls(float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy),
                   int(cam.width), int(cam.height), np.asarray(cam.r_wc), np.asarray(cam.t_wc),
                   float(getattr(cam, "near", 0.05)), float(getattr(cam, "far", 100.0)))


def look_at_camera(position, target, up=(0.0, 0.0, 1.0), fov_deg=60.0, width=64, height=64,
                   near=0.05, far=100.0) -> Camera:
    position = np.asarray(position, dtype=np.float64)
    target = np.asarray(target, dtype=np.float64)
    fwd = target - position
    fwd = fwd / np.linalg.norm(fwd)
    up = np.asarray(up, dtype=np.float64)
    right = np.cross(fwd, up)
    if np.linalg.norm(right) < 1e-9:
        right = np.cross(fwd, np.array([0.0, 1.0, 0.0]))
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    r_wc = np.stack([right, down, fwd])
    t_wc = -r_wc @ position
    f = 0.5 * width / np.tan(np.radians(fov_deg) / 2)
    return Camera(f, f, width / 2, height / 2, width, height, r_wc, t_wc, near, far)


def camera_constants(cam) -> dict:
    """fp64 scalars of one view, computed exactly like the reference.

    lim_x / lim_y: gaussian_core.py:208-209 (Python float arithmetic).
    center: data_io.py:65-67 (numpy).
    """
    fx, fy, cx, cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    w, h = int(cam.width), int(cam.height)
    if w < 1 or h < 1:
        raise InvalidInputError("image size must be positive")
    lim_x = 1.3 * max(cx, w - cx) / fx
    lim_y = 1.3 * max(cy, h - cy) / fy
    r_wc = np.ascontiguousarray(np.asarray(cam.r_wc, dtype=np.float64).reshape(3, 3))
    t_wc = np.ascontiguousarray(np.asarray(cam.t_wc, dtype=np.float64).reshape(3))
    center = -r_wc.T @ t_wc
    return dict(r_wc=r_wc, t_wc=t_wc, center=np.ascontiguousarray(center), fx=fx, fy=fy,
                cx=cx, cy=cy, lim_x=lim_x, lim_y=lim_y, width=w, height=h)
