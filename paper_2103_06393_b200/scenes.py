"""Coil geometries for the BASELINE configs (SURVEY.md §0 gap 2).

The reference ships only a loop and a plate generator (src/scene.cpp:177-231);
configs 2-4 name birdcage-like and close-fitting array coils, which are built
here as plain RWG-edge source lists (midpoint, unit direction, weight = edge
length — the reference's EdgeSource, include/tuckmat/scene.hpp:45-49) around
a centred voxel grid, keeping every edge at least 2h from every voxel centre
(the reference's separation guard, src/scene.cpp:66-72).  They are input
producers for the GPU compressor (compress.py); the scene type is the
oracle-compatible `Scene` (origin, spacing, dims, sources, op, k0, q).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class Scene:
    origin: np.ndarray
    spacing: float
    dims: tuple
    sources: np.ndarray  # (m, 7): midpoint xyz, unit direction xyz, weight
    op: int = 0
    k0: float = 0.0
    q: int = 3

    @property
    def num_sources(self):
        return int(self.sources.shape[0])

    @property
    def num_voxels(self):
        return int(np.prod(self.dims))

    @property
    def rows(self):
        return self.q * self.num_voxels


def wavenumber_from_mhz(f_mhz):
    """include/tuckmat/scene.hpp:20-22."""
    return 2.0 * math.pi * f_mhz * 1e6 / 299792458.0


def centered_grid(spacing, dims):
    """make_centered_grid at the origin (src/scene.cpp:27-41)."""
    origin = np.array([-0.5 * spacing * d for d in dims], np.float64)
    return origin, float(spacing), tuple(int(d) for d in dims)


def separation(origin, spacing, dims, p):
    """Distance from p to the nearest voxel centre (src/scene.cpp:13-23)."""
    idx = np.clip(np.round((p - origin) / spacing - 0.5), 0, np.asarray(dims) - 1)
    return float(np.linalg.norm(p - (origin + spacing * (idx + 0.5))))


def _edges_on_polyline(pts, closed):
    """RWG-like edges between consecutive points: midpoint, unit direction, length."""
    out = []
    n = len(pts) if closed else len(pts) - 1
    for i in range(n):
        a, b = pts[i], pts[(i + 1) % len(pts)]
        d = b - a
        L = float(np.linalg.norm(d))
        out.append(np.concatenate([(a + b) / 2, d / L, [L]]))
    return out


def birdcage(grid, radius, length, rungs=8, segs_per_rung=16, ring_segs=64, shield_radius=None,
             shield_rows=0, shield_segs=0, op=0, f_mhz=298.0, q=3):
    """Birdcage-like coil around the grid (config 2): `rungs` axial rungs of
    `segs_per_rung` edges, two end rings of `ring_segs` edges, optionally a
    shield cylinder of `shield_rows` x `shield_segs` circumferential edges."""
    origin, h, dims = grid
    src = []
    z0, z1 = -0.5 * length, 0.5 * length
    for r in range(rungs):
        th = 2 * math.pi * r / rungs
        c, s = math.cos(th), math.sin(th)
        pts = [np.array([radius * c, radius * s, z0 + (z1 - z0) * t / segs_per_rung]) for t in range(segs_per_rung + 1)]
        src += _edges_on_polyline(pts, False)
    for z in (z0, z1):
        pts = [np.array([radius * math.cos(2 * math.pi * t / ring_segs), radius * math.sin(2 * math.pi * t / ring_segs),
                         z]) for t in range(ring_segs)]
        src += _edges_on_polyline(pts, True)
    if shield_radius and shield_rows and shield_segs:
        for row in range(shield_rows):
            z = z0 + (z1 - z0) * (row + 0.5) / shield_rows
            pts = [np.array([shield_radius * math.cos(2 * math.pi * t / shield_segs),
                             shield_radius * math.sin(2 * math.pi * t / shield_segs), z])
                   for t in range(shield_segs)]
            src += _edges_on_polyline(pts, True)
    sc = Scene(origin, h, dims, np.array(src, np.float64), op, wavenumber_from_mhz(f_mhz), q)
    check_guard(sc)
    return sc


def close_fitting_array(grid, gap, channels=8, loops_per_channel=4, segs_per_loop=156, op=0, f_mhz=298.0, q=12):
    """Multi-channel close-fitting array (config 4): `channels` x
    `loops_per_channel` rectangular loops on a box `gap` outside the grid's
    faces in x and y (wrapped around the head-like grid), each loop of
    `segs_per_loop` edges — ~5 000 edges at the defaults."""
    origin, h, dims = grid
    ext = np.array([h * d for d in dims]) / 2 + gap
    src = []
    per_face = channels // 4 if channels >= 4 else 1
    nloops = channels * loops_per_channel
    li = 0
    for face in range(4):
        axis, sign = (0, 1, 0, 1)[face], (1, 1, -1, -1)[face]
        for c in range(per_face):
            for lp in range(loops_per_channel):
                if li >= nloops:
                    break
                # loop centre on the face, tiled along the face's in-plane axis and z
                tang = 1 - axis
                u = -ext[tang] + 2 * ext[tang] * (c + 0.5) / per_face
                w = -ext[2] + 2 * ext[2] * (lp + 0.5) / loops_per_channel
                hu, hw = 0.45 * 2 * ext[tang] / per_face, 0.45 * 2 * ext[2] / loops_per_channel
                corners = [(u - hu, w - hw), (u + hu, w - hw), (u + hu, w + hw), (u - hu, w + hw)]
                per_side = segs_per_loop // 4
                pts = []
                for k in range(4):
                    (a0, b0), (a1, b1) = corners[k], corners[(k + 1) % 4]
                    for t in range(per_side):
                        a, b = a0 + (a1 - a0) * t / per_side, b0 + (b1 - b0) * t / per_side
                        p = np.zeros(3)
                        p[axis] = sign * ext[axis]
                        p[tang] = a
                        p[2] = b
                        pts.append(p)
                src += _edges_on_polyline(pts, True)
                li += 1
    sc = Scene(origin, h, dims, np.array(src, np.float64), op, wavenumber_from_mhz(f_mhz), q)
    check_guard(sc)
    return sc


def check_guard(sc):
    """The reference's separation guard (src/scene.cpp:66-72): every edge at
    least 2h from every voxel centre."""
    for j, s in enumerate(sc.sources):
        if separation(sc.origin, sc.spacing, sc.dims, s[0:3]) < 2.0 * sc.spacing:
            raise ValueError(f"source {j} violates the separation guard (< 2h)")
