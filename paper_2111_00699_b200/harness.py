"""Scene harness over the CUDA core: the reference's `bench.run` surface.

Mirrors /root/reference/pkg/src/mpmbench/bench.py:33-35 (CSV columns), :62-145 (RunConfig),
:302-327 (`.mpmf` snapshots: magic, u32 version, u32 count, f32 xyz ordered by particle id),
:383-512 (run / RunResult) so that a run script written for the reference, and the plots package
that consumes its CSV, work unchanged on the GPU backend.  Workers are logical workers of one
process on one device (`CudaCluster`); one process per GPU is `paper_2111_00699_b200.dist`.
"""
from __future__ import annotations

import csv
import json
import math
import struct
import time
from dataclasses import asdict, dataclass, field, fields
from pathlib import Path

import numpy as np

from . import scenes
from .domain import SimParams
from .errors import ConfigError, SimulationError
from .multiworker import efficiency
from .options import PipelineOptions

SNAPSHOT_MAGIC = b"MPMF"
SNAPSHOT_VERSION = 1
CSV_COLUMNS = ("frame", "steps", "ms_total", "ms_rebuild", "ms_sort", "ms_p2g", "ms_grid", "ms_g2p",
               "rebuild_count", "realloc_count", "workers", "particle_count")
SCENES = ("sand_blocks", "fountain_lite", "free_fall", "snow")


@dataclass
class TimingRow:
    frame: int
    steps: int
    ms_total: float
    ms_rebuild: float
    ms_sort: float
    ms_p2g: float
    ms_grid: float
    ms_g2p: float
    rebuild_count: int
    realloc_count: int
    workers: int
    particle_count: int

    def as_list(self):
        return [getattr(self, c) for c in CSV_COLUMNS]


@dataclass
class RunConfig:
    """One run; field names follow the reference's RunConfig (bench.py:62-100)."""
    scene: str = "sand_blocks"
    l: int = 12
    boxes: int = 4
    ppc: int = 8
    dx: float = 25.0 / 64.0
    frames: int = 4
    steps_per_frame: int = 36
    frame_dt: float = 1.0 / 48.0
    cfl: float = 0.5
    cfl_auto: bool | None = None
    workers: int = 1
    lane_width: int = 32
    rebuild: str = "amortized"
    sort: str = "amortized"
    fusion: str = "merged"
    transfer: str = "split"
    deterministic: bool = False
    seed: int = 2024
    out_csv: str | None = None
    out_snap: str | None = None
    gap_cells: int | None = None
    drop_cells: int = 2
    init_speed: float = -150.0
    density: float = 2.0
    young: float = 1.0e5
    poisson: float = 0.3
    bulk_modulus: float = 1.0e5
    gamma: float = 7.0
    fountain_radius: float | None = None
    emit_speed: float = 160.0
    gravity_z: float = -981.0
    flip_blend: float = 0.0
    fused_threshold: int = 100_000
    collect_conservation: bool = False
    barrier_timeout: float = 10.0     # seconds (reference bench.py RunConfig): the device-side step
                                      # barrier of peer-mapped runs takes it as its wait timeout
    device: str = "cuda:0"
    profile_phases: bool = False      # CUDA events around the step kernels (CSV phase columns)

    def __post_init__(self):
        if self.scene not in SCENES:
            raise ConfigError(f"scene must be one of {SCENES}, got {self.scene!r}")
        for name in ("l", "ppc", "steps_per_frame", "workers", "lane_width"):
            if getattr(self, name) < 1:
                raise ConfigError(f"{name} must be positive, got {getattr(self, name)}")
        if self.frames < 0:
            raise ConfigError(f"frames must be >= 0, got {self.frames}")
        if self.scene == "fountain_lite" and self.transfer == "g2p2g":
            raise ConfigError("the fountain emits particles every frame, which conflicts with the "
                              "fused G2P2G transfer")

    @property
    def cfl_enabled(self) -> bool:
        return self.scene == "fountain_lite" if self.cfl_auto is None else self.cfl_auto

    @staticmethod
    def from_dict(payload: dict) -> "RunConfig":
        known = {f.name for f in fields(RunConfig)}
        unknown = set(payload) - known
        if unknown:
            raise ConfigError(f"unknown config fields: {sorted(unknown)}")
        return RunConfig(**payload)

    @staticmethod
    def from_json(path) -> "RunConfig":
        with open(path) as fh:
            return RunConfig.from_dict(json.load(fh))

    def with_overrides(self, **overrides) -> "RunConfig":
        payload = asdict(self)
        payload.update({k: v for k, v in overrides.items() if v is not None})
        return RunConfig.from_dict(payload)


def build_scene(cfg: RunConfig) -> scenes.World:
    if cfg.scene == "sand_blocks":
        return scenes.sand_blocks(l=cfg.l, boxes=cfg.boxes, ppc=cfg.ppc, dx=cfg.dx, seed=cfg.seed,
                                  steps_per_frame=cfg.steps_per_frame, frame_dt=cfg.frame_dt,
                                  init_speed=cfg.init_speed, density=cfg.density, young=cfg.young,
                                  poisson=cfg.poisson, gravity_z=cfg.gravity_z, gap_cells=cfg.gap_cells,
                                  drop_cells=cfg.drop_cells, flip_blend=cfg.flip_blend)
    if cfg.scene == "snow":
        # the snow scene has its own cell width / frame / substep defaults (configs[2]); a config
        # that sets them away from RunConfig's sand-blocks defaults is taken at its word
        d = RunConfig()
        kw = {}
        if cfg.dx != d.dx:
            kw["dx"] = cfg.dx
        if cfg.steps_per_frame != d.steps_per_frame:
            kw["steps_per_frame"] = cfg.steps_per_frame
        if cfg.frame_dt != d.frame_dt:
            kw["frame_dt"] = cfg.frame_dt
        if cfg.init_speed != d.init_speed:
            kw["init_speed"] = cfg.init_speed
        return scenes.snow(l=cfg.l, boxes=cfg.boxes, ppc=cfg.ppc, seed=cfg.seed, **kw)
    if cfg.scene == "fountain_lite":
        return scenes.fountain(dx=cfg.dx, seed=cfg.seed, frame_dt=cfg.frame_dt, cfl=cfg.cfl,
                               radius=cfg.fountain_radius, emit_speed=cfg.emit_speed,
                               bulk_modulus=cfg.bulk_modulus, gamma=cfg.gamma, gravity_z=cfg.gravity_z)
    return scenes.free_fall(dx=cfg.dx, steps_per_frame=cfg.steps_per_frame, frame_dt=cfg.frame_dt)


def write_snapshot(path, positions) -> None:
    """bench.py:302-313: magic, u32 version, u32 count, f32 xyz triples."""
    pos = np.ascontiguousarray(np.asarray(positions, dtype=np.float32))
    if pos.ndim != 2 or (pos.shape[0] and pos.shape[1] != 3):
        raise ConfigError(f"positions must be (n, 3), got {pos.shape}")
    try:
        with open(path, "wb") as fh:
            fh.write(SNAPSHOT_MAGIC)
            fh.write(struct.pack("<II", SNAPSHOT_VERSION, pos.shape[0]))
            fh.write(pos.astype("<f4").tobytes())
    except OSError as exc:
        raise SimulationError(f"cannot write snapshot {path}: {exc}") from exc


def read_snapshot(path) -> np.ndarray:
    try:
        blob = Path(path).read_bytes()
    except OSError as exc:
        raise SimulationError(f"cannot read snapshot {path}: {exc}") from exc
    if blob[:4] != SNAPSHOT_MAGIC:
        raise SimulationError(f"{path} is not a particle snapshot")
    version, count = struct.unpack("<II", blob[4:12])
    if version != SNAPSHOT_VERSION:
        raise SimulationError(f"unsupported snapshot version {version}")
    return np.frombuffer(blob[12:], dtype="<f4").reshape(count, 3).astype(np.float32)


@dataclass
class RunResult:
    rows: list
    workers: list
    mean_ms_per_frame: float
    rebuild_gaps: list
    particle_count: int
    conservation: list
    counters: np.ndarray
    snapshot_paths: list = field(default_factory=list)
    effective_transfer: str = "split"     # what the workers ran (g2p2g falls back above fused_threshold)

    @property
    def mean_steps_between_rebuilds(self) -> float:
        return float(np.mean(self.rebuild_gaps)) if self.rebuild_gaps else math.inf


def _split_even(n_items: int, n_workers: int):
    base, rem = divmod(n_items, n_workers)
    out, start = [], 0
    for w in range(n_workers):
        s = base + 1 if w < rem else base
        out.append(slice(start, start + s))
        start += s
    return out


def run(cfg: RunConfig, params_override: SimParams | None = None) -> RunResult:
    """Execute one configured run on the CUDA core; streams CSV rows and snapshots if asked
    (bench.py:417-512)."""
    import torch
    from .cluster import CudaCluster

    spec = build_scene(cfg)
    params = params_override or spec.params
    options = PipelineOptions(rebuild=cfg.rebuild, sort=cfg.sort, fusion=cfg.fusion,
                              transfer=cfg.transfer, deterministic=cfg.deterministic,
                              fused_threshold=cfg.fused_threshold,
                              collect_conservation=cfg.collect_conservation)
    init_vmax = float(np.linalg.norm(spec.velocities, axis=1).max()) if len(spec.velocities) else 0.0
    if spec.emission is not None:
        init_vmax = max(init_vmax, float(np.linalg.norm(spec.emission.velocity)))
    cluster = CudaCluster(cfg.workers, params, spec.material, spec.boundary, options,
                          initial_vmax=init_vmax, device=cfg.device)
    cluster.cfl_mode = cfg.cfl_enabled
    workers = cluster.workers
    for w in workers:
        w.cfl_mode = cfg.cfl_enabled
        w.time_kernels = w.profile_all_phases = cfg.profile_phases
    cluster.seed(spec.positions, spec.velocities, spec.particle_mass)
    next_id = len(spec.positions)

    csv_fh = csv_writer = None
    if cfg.out_csv:
        Path(cfg.out_csv).parent.mkdir(parents=True, exist_ok=True)
        csv_fh = open(cfg.out_csv, "w", newline="")
        csv_writer = csv.writer(csv_fh)
        csv_writer.writerow(CSV_COLUMNS)
    snap_dir = None
    if cfg.out_snap:
        snap_dir = Path(cfg.out_snap)
        snap_dir.mkdir(parents=True, exist_ok=True)

    rows, snapshot_paths = [], []
    realloc_seen = 0
    try:
        for frame in range(cfg.frames):
            try:
                if spec.emission is not None:
                    epos, evel = spec.emission.sample(frame)
                    ids = np.arange(next_id, next_id + len(epos), dtype=np.int64)
                    next_id += len(epos)
                    for w, sl in zip(workers, _split_even(len(epos), cfg.workers)):
                        w.append_particles(epos[sl], evel[sl], spec.particle_mass, ids=ids[sl])
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                if cfg.workers == 1:
                    workers[0].run_frame()
                    steps = workers[0].frame_steps
                else:
                    cluster.run_frame()
                    steps = cluster.frame_steps
                torch.cuda.synchronize()
                ms_total = (time.perf_counter() - t0) * 1e3
            except SimulationError as exc:
                # bench.py:368-369: failures carry their frame / step context
                raise type(exc)(f"frame {frame}, step {workers[0]._global_step}: {exc}") from exc
            lo = workers[0]._global_step - steps
            rebuild_steps = set()
            for w in workers:
                rebuild_steps.update(s for s in w.rebuild_steps if s >= lo)
            phase = {k: float(np.mean([w.phase_ms[k] for w in workers]))
                     for k in ("rebuild", "sort", "p2g", "grid", "g2p")}
            realloc_now = sum(w.realloc_count for w in workers)
            row = TimingRow(frame=frame, steps=steps, ms_total=ms_total, ms_rebuild=phase["rebuild"],
                            ms_sort=phase["sort"], ms_p2g=phase["p2g"], ms_grid=phase["grid"],
                            ms_g2p=phase["g2p"], rebuild_count=len(rebuild_steps),
                            realloc_count=realloc_now - realloc_seen, workers=cfg.workers,
                            particle_count=sum(w.store.count for w in workers))
            realloc_seen = realloc_now
            rows.append(row)
            if csv_writer is not None:
                csv_writer.writerow(row.as_list())
                csv_fh.flush()
            if snap_dir is not None:
                path = snap_dir / f"frame_{frame:04d}.mpmf"
                write_snapshot(path, cluster.positions_sorted_by_id())
                snapshot_paths.append(str(path))
    finally:
        if csv_fh is not None:
            csv_fh.close()

    gaps = []
    for w in workers:
        s = w.rebuild_steps
        gaps.extend(int(b - a) for a, b in zip(s, s[1:]))
    conservation = []
    for w in workers:
        conservation.extend(w.conservation)
    counters = np.sum([w.counters for w in workers], axis=0)
    mean_ms = float(np.mean([r.ms_total for r in rows])) if rows else 0.0
    return RunResult(rows=rows, workers=workers, mean_ms_per_frame=mean_ms, rebuild_gaps=gaps,
                     particle_count=sum(w.store.count for w in workers), conservation=conservation,
                     counters=counters, snapshot_paths=snapshot_paths,
                     effective_transfer=workers[0].effective_transfer if workers else cfg.transfer)


def run_efficiency(cfg: RunConfig, max_workers: int, warmup: bool = True):
    """Paired runs at 1..max_workers logical workers -> e = t1 / (n tn) (bench.py:515-532)."""
    if max_workers < 1:
        raise ConfigError(f"max workers must be >= 1, got {max_workers}")
    if warmup:
        run(cfg.with_overrides(frames=1, out_csv=None, out_snap=None))
    timings = {}
    for n in range(1, max_workers + 1):
        timings[n] = run(cfg.with_overrides(workers=n)).mean_ms_per_frame
    return [efficiency(timings[1], timings[n], n) for n in range(1, max_workers + 1)]
