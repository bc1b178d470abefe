"""Synthetic scenes of the named configurations (host side, numpy only).

`sand_blocks`, `fountain` and `free_fall` follow the reference's scene layer
(/root/reference/pkg/src/mpmbench/bench.py:62-300: RunConfig, gen_sand_blocks,
gen_fountain_lite, build_scene) so that the same configuration yields the same particles:
stratified samples per cell from `np.random.default_rng(seed)`, boxes on a square grid with
one-box gaps, an 8-cell wall margin, CGS units.  `snow` is the 1.33 M-particle configuration
of BASELINE.json ("configs[2]"): the reference has no snow scene, so it is a box drop of the
paper's size and cell width built with the same generator.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .domain import Material, SimParams
from .errors import ConfigError
from .options import BoundaryBox

WALL_MARGIN_CELLS = 8


@dataclass
class Emission:
    """Per-frame particle source: a ball of cells resampled every frame (bench.py:198-243)."""
    cells: np.ndarray
    ppc: int
    dx: float
    seed: int
    velocity: tuple

    @property
    def per_frame(self) -> int:
        return len(self.cells) * self.ppc

    def sample(self, frame: int):
        rng = np.random.default_rng([self.seed, frame])
        pos = _stratified(rng, self.cells, self.ppc) * self.dx
        vel = np.tile(np.asarray(self.velocity, dtype=np.float64), (len(pos), 1))
        return pos, vel


@dataclass
class World:
    params: SimParams
    material: Material
    boundary: BoundaryBox | None
    positions: np.ndarray
    velocities: np.ndarray
    particle_mass: float
    emission: Emission | None = None
    name: str = ""
    cfl_auto: bool = False


def _cube_side(ppc: int) -> int:
    s = round(ppc ** (1.0 / 3.0))
    if s ** 3 != ppc:
        raise ConfigError(f"ppc must be a perfect cube for stratified sampling, got {ppc}")
    return s


def _stratified(rng, cells: np.ndarray, ppc: int) -> np.ndarray:
    """One uniform sample in each of the ppc congruent subcells of every cell (cell units)."""
    s = _cube_side(ppc)
    sub = np.stack(np.meshgrid(np.arange(s), np.arange(s), np.arange(s), indexing="ij"),
                   axis=-1).reshape(-1, 3)
    base = (cells[:, None, :] * s + sub[None, :, :]).reshape(-1, 3)
    return (base + rng.random((base.shape[0], 3))) / s


def _box_cells(l: int) -> np.ndarray:
    return np.stack(np.meshgrid(np.arange(l), np.arange(l), np.arange(l), indexing="ij"),
                    axis=-1).reshape(-1, 3)


def sand_blocks_positions(l, boxes, ppc, dx, seed, gap_cells=None, drop_cells=2):
    """bench.py:169-194: (positions, cubic domain extent in cells)."""
    if boxes not in (1, 4, 16):
        raise ConfigError(f"boxes must be 1, 4 or 16, got {boxes}")
    side = int(round(math.sqrt(boxes)))
    gap = l if gap_cells is None else int(gap_cells)
    m = WALL_MARGIN_CELLS
    span = side * l + (side + 1) * gap
    height = drop_cells + l + max(2 * l, 12)
    domain = max(span + 2 * m, height + 2 * m)
    rng = np.random.default_rng(seed)
    cells = _box_cells(l)
    parts = []
    for by in range(side):
        for bx in range(side):
            origin = np.array([m + gap + bx * (l + gap), m + gap + by * (l + gap), m + drop_cells])
            parts.append((origin + _stratified(rng, cells, ppc)) * dx)
    return np.concatenate(parts, axis=0), domain


def sand_blocks(l=12, boxes=4, ppc=8, dx=25.0 / 64.0, seed=2024, steps_per_frame=36,
                frame_dt=1.0 / 48.0, init_speed=-150.0, density=2.0, young=1.0e5, poisson=0.3,
                gravity_z=-981.0, gap_cells=None, drop_cells=2, flip_blend=0.0,
                material=None) -> World:
    """Sand Blocks drop (configs[0] / configs[3]); default = the reference's mini scene."""
    pos, domain = sand_blocks_positions(l, boxes, ppc, dx, seed, gap_cells, drop_cells)
    vel = np.zeros_like(pos)
    vel[:, 2] = init_speed
    params = SimParams(dx=dx, dt=frame_dt / steps_per_frame, gravity=(0.0, 0.0, gravity_z),
                       frame_dt=frame_dt, steps_per_frame=steps_per_frame, flip_blend=flip_blend)
    material = material or Material.fixed_corotated(density, young, poisson)
    m = WALL_MARGIN_CELLS
    boundary = BoundaryBox((m * dx,) * 3, ((domain - m) * dx,) * 3, mode="slip")
    return World(params, material, boundary, pos, vel, material.density * dx ** 3 / ppc,
                 name=f"sand_blocks l={l} boxes={boxes} ppc={ppc}")


def snow(l=35, boxes=4, ppc=8, dx=1.35, seed=2024, frame_dt=1.0 / 60.0, steps_per_frame=30,
         init_speed=-150.0, density=0.4, young=6.0e5, poisson=0.3, plastic=True) -> World:
    """Snow 1.33 M (configs[2]): boxes * l^3 * ppc = 1 372 000 particles at dx = 1.35 cm,
    frame 1/60 s, ~30 substeps per frame (dt avg 5.46e-4).  `plastic`
    selects the snow clamp+hardening model; False gives the reference-pinned fixed-corotated
    variant of the same scene."""
    # bulk modulus 5e5, nu = 0.3 (E = 3 kappa (1 - 2 nu) = 6e5), hardening xi = 5
    mat = Material.snow(density, young, poisson, hardening=5.0) if plastic \
        else Material.fixed_corotated(density, young, poisson)
    w = sand_blocks(l=l, boxes=boxes, ppc=ppc, dx=dx, seed=seed, steps_per_frame=steps_per_frame,
                    frame_dt=frame_dt, init_speed=init_speed, material=mat)
    w.name = f"snow l={l} boxes={boxes} ppc={ppc} ({'snow plasticity' if plastic else 'fixed-corotated'})"
    return w


def fountain(dx=0.66, seed=2024, frame_dt=1.0 / 60.0, cfl=0.5, radius=None, emit_speed=160.0,
             bulk_modulus=1.0e5, gamma=7.0, gravity_z=-981.0, ppc=27) -> World:
    """Fountain (configs[1]): weakly compressible water, ball emitter resampled every frame,
    CFL-auto dt (bench.py:274-287)."""
    domain = 64
    material = Material.fluid(1.0, bulk_modulus, gamma)
    params = SimParams(dx=dx, dt=frame_dt / 36, gravity=(0.0, 0.0, gravity_z), frame_dt=frame_dt,
                       steps_per_frame=36, cfl=cfl)
    m = WALL_MARGIN_CELLS
    boundary = BoundaryBox((m * dx,) * 3, ((domain - m) * dx,) * 3, mode="slip")
    r = max(1.5 * dx if radius is None else float(radius), 1e-9)
    c = np.array([domain * dx / 2.0, domain * dx / 2.0, domain * dx * 0.45])
    lo = np.floor((c - r) / dx).astype(np.int64)
    hi = np.ceil((c + r) / dx).astype(np.int64)
    grid = np.stack(np.meshgrid(*[np.arange(lo[a], hi[a] + 1) for a in range(3)], indexing="ij"),
                    axis=-1).reshape(-1, 3)
    inside = np.linalg.norm((grid + 0.5) * dx - c, axis=1) <= r
    cells = grid[inside] if inside.any() else np.floor(c / dx).astype(np.int64)[None, :]
    emission = Emission(cells.astype(np.int64), ppc, dx, seed, (0.0, 0.0, emit_speed))
    empty = np.zeros((0, 3))
    return World(params, material, boundary, empty, empty.copy(), material.density * dx ** 3 / ppc,
                 emission=emission, name="fountain", cfl_auto=True)


def free_fall(dx=25.0 / 64.0, steps_per_frame=36, frame_dt=1.0 / 48.0) -> World:
    domain = 64
    params = SimParams(dx=dx, dt=frame_dt / steps_per_frame, frame_dt=frame_dt,
                       steps_per_frame=steps_per_frame)
    material = Material.fixed_corotated(2.0, 1.0e5, 0.3)
    pos = np.array([[domain * dx / 2.0] * 3])
    return World(params, material, None, pos, np.zeros((1, 3)), 2.0 * dx ** 3, name="free_fall")


@dataclass
class Population:
    material: Material
    positions: np.ndarray
    velocities: np.ndarray
    particle_mass: float


@dataclass
class MixedWorld:
    """Several material populations sharing one grid (run with CudaCluster, one worker each)."""
    params: SimParams
    boundary: BoundaryBox | None
    populations: list
    name: str = ""
    domain_cells: int = 0

    @property
    def n_particles(self) -> int:
        return sum(len(p.positions) for p in self.populations)


def mixed_sparse(l=50, pairs_side=4, ppc=8, dx=1.0, seed=2024, domain_cells=512, frame_dt=1.0 / 60.0,
                 steps_per_frame=30, init_speed=-150.0, gap_cells=4, gravity_z=-981.0) -> MixedWorld:
    """Large sparse-grid stress test (BASELINE.json configs[4]): `pairs_side`^2 separated
    clusters on a `domain_cells`^3 grid, each a sand box dropped onto a snow box, i.e. two
    material populations of equal size that meet on the grid.  Defaults: 16 clusters x 2 boxes
    x 50^3 cells x 8 = 32 000 000 particles on 512^3; (l=40, pairs_side=2) is the 4.1 M
    per-GPU share of that scene.  Not a reference scene (one material per run there): the
    generator follows sand_blocks (stratified samples, wall margin, CGS units)."""
    m = WALL_MARGIN_CELLS
    pitch = (domain_cells - 2 * m) // pairs_side
    if pitch < l + 8 or 2 * l + gap_cells + 2 + 2 * m > domain_cells:
        raise ConfigError(f"{pairs_side}^2 clusters of {l}-cell boxes do not fit {domain_cells}^3 cells")
    rng = np.random.default_rng(seed)
    cells = _box_cells(l)
    snow_parts, sand_parts = [], []
    for by in range(pairs_side):
        for bx in range(pairs_side):
            ox = m + bx * pitch + (pitch - l) // 2
            oy = m + by * pitch + (pitch - l) // 2
            snow_parts.append((np.array([ox, oy, m + 2]) + _stratified(rng, cells, ppc)) * dx)
            sand_parts.append((np.array([ox, oy, m + 2 + l + gap_cells]) + _stratified(rng, cells, ppc)) * dx)
    snow_pos = np.concatenate(snow_parts, axis=0)
    sand_pos = np.concatenate(sand_parts, axis=0)
    snow_mat = Material.snow(0.4, 6.0e5, 0.3, hardening=5.0)
    sand_mat = Material.sand(2.0, 1.0e5, 0.3)
    snow_vel = np.zeros_like(snow_pos)
    sand_vel = np.zeros_like(sand_pos)
    sand_vel[:, 2] = init_speed
    params = SimParams(dx=dx, dt=frame_dt / steps_per_frame, gravity=(0.0, 0.0, gravity_z),
                       frame_dt=frame_dt, steps_per_frame=steps_per_frame)
    boundary = BoundaryBox((m * dx,) * 3, ((domain_cells - m) * dx,) * 3, mode="slip")
    pops = [Population(snow_mat, snow_pos, snow_vel, snow_mat.density * dx ** 3 / ppc),
            Population(sand_mat, sand_pos, sand_vel, sand_mat.density * dx ** 3 / ppc)]
    return MixedWorld(params, boundary, pops, domain_cells=domain_cells,
                      name=f"mixed snow/sand l={l} clusters={pairs_side ** 2} on {domain_cells}^3")
