"""Parametric phantoms of the benchmark configs (REF src/synthetic.cpp:101-178).

Vectorised with numpy but with the reference's per-voxel expression order
(voxel centre ``origin + (i + 0.5) * vs``, ``dx*dx + dy*dy <= r*r``) so the
masks are bit-identical to the reference generators (pinned in
tests/test_inputs.py against oracle/_ref and a committed checksum).
"""
from __future__ import annotations

import math

import numpy as np

from .inputs import PI, Material, VoxelPhantom, make_empty_phantom


def _centers(ph: VoxelPhantom, axis: int) -> np.ndarray:
    n = ph.dims[axis]
    return ph.origin[axis] + (np.arange(n, dtype=np.float64) + 0.5) * ph.voxel_size[axis]


def _fill_cylinder(ph: VoxelPhantom, cx, cy, radius, half_height, mat_id, density) -> None:
    """REF fill_cylinder (synthetic.cpp:20-37)."""
    nx, ny, nz = ph.dims
    px, py, pz = _centers(ph, 0), _centers(ph, 1), _centers(ph, 2)
    r2 = radius * radius
    dx = px - cx
    dy = py - cy
    inside = (dx[None, :] * dx[None, :] + dy[:, None] * dy[:, None]) <= r2  # [iy, ix]
    zsel = np.abs(pz) <= half_height
    ids = ph.material_id.reshape(nz, ny, nx)
    dens = ph.density.reshape(nz, ny, nx)
    for iz in np.nonzero(zsel)[0]:
        ids[iz][inside] = mat_id
        dens[iz][inside] = np.float32(density)


def make_cube_phantom(n, voxel_cm, edge_cm, material: Material, density) -> VoxelPhantom:
    """REF make_cube_phantom (synthetic.cpp:41-59)."""
    if not edge_cm > 0.0:
        raise ValueError("cube phantom: edge must be > 0")
    ph = make_empty_phantom(n, n, n, (voxel_cm,) * 3, [material])
    half = 0.5 * edge_cm
    px, py, pz = _centers(ph, 0), _centers(ph, 1), _centers(ph, 2)
    m = (np.abs(pz) <= half)[:, None, None] & (np.abs(py) <= half)[None, :, None] & \
        (np.abs(px) <= half)[None, None, :]
    ph.material_id.reshape(n, n, n)[m] = 1
    ph.density.reshape(n, n, n)[m] = np.float32(density)
    return ph


def make_cylinder_phantom(n, voxel_cm, radius_cm, height_cm, material: Material,
                          density) -> VoxelPhantom:
    """REF make_cylinder_phantom (synthetic.cpp:61-69)."""
    if not (radius_cm > 0.0 and height_cm > 0.0):
        raise ValueError("cylinder phantom: radius and height must be > 0")
    ph = make_empty_phantom(n, n, n, (voxel_cm,) * 3, [material])
    _fill_cylinder(ph, 0.0, 0.0, radius_cm, 0.5 * height_cm, 1, density)
    return ph


def make_rods_phantom(n, voxel_cm, body_radius_cm, height_cm, body: Material, body_density,
                      n_rods, rod_radius_cm, ring_radius_cm, rod: Material,
                      rod_density) -> VoxelPhantom:
    """REF make_rods_phantom (synthetic.cpp:71-92)."""
    if not (body_radius_cm > 0.0 and rod_radius_cm > 0.0):
        raise ValueError("rods phantom: radii must be > 0")
    if n_rods < 1:
        raise ValueError("rods phantom: need at least one rod")
    if ring_radius_cm + rod_radius_cm > body_radius_cm:
        raise ValueError("rods phantom: rods extend outside the body")
    ph = make_empty_phantom(n, n, n, (voxel_cm,) * 3, [body, rod])
    half = 0.5 * height_cm
    _fill_cylinder(ph, 0.0, 0.0, body_radius_cm, half, 1, body_density)
    for k in range(n_rods):
        phi = 2.0 * PI * k / n_rods
        _fill_cylinder(ph, ring_radius_cm * math.cos(phi), ring_radius_cm * math.sin(phi),
                       rod_radius_cm, half, 2, rod_density)
    return ph


def make_cylinder_head_phantom(n, voxel_cm, body: Material, body_density, insert: Material,
                               insert_density) -> VoxelPhantom:
    """REF make_cylinder_head_phantom (synthetic.cpp:94-117): light-metal body,
    four air bores, ring of eight dense inserts."""
    extent = n * voxel_cm
    body_r = 0.42 * extent
    height = 0.8 * extent
    ph = make_empty_phantom(n, n, n, (voxel_cm,) * 3, [body, insert])
    half = 0.5 * height
    _fill_cylinder(ph, 0.0, 0.0, body_r, half, 1, body_density)
    for k in range(4):
        phi = 2.0 * PI * (k + 0.5) / 4.0
        _fill_cylinder(ph, 0.55 * body_r * math.cos(phi), 0.55 * body_r * math.sin(phi),
                       0.18 * body_r, half * 0.9, 0, 0.0)
    for k in range(8):
        phi = 2.0 * PI * k / 8.0
        _fill_cylinder(ph, 0.8 * body_r * math.cos(phi), 0.8 * body_r * math.sin(phi),
                       0.07 * body_r, half * 0.8, 2, insert_density)
    return ph
