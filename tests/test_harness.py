"""Scene harness (paper_2111_00699_b200.harness): the reference's bench.run surface.
CPU tests cover config / snapshot / CSV schema; GPU tests run scenes end to end."""
import csv
import os

import numpy as np
import pytest

from oracle import mpm_oracle as O
from paper_2111_00699_b200 import ConfigError, PipelineOptions, SimulationError, SpatialDomainError
from paper_2111_00699_b200 import harness as H


def test_config_validation_and_overrides(tmp_path):
    # tests/test_bench.py:136-156 of the reference
    cfg = H.RunConfig()
    assert cfg.scene == "sand_blocks" and not cfg.cfl_enabled
    assert H.RunConfig(scene="fountain_lite").cfl_enabled
    with pytest.raises(ConfigError):
        H.RunConfig(scene="nope")
    with pytest.raises(ConfigError):
        H.RunConfig(scene="fountain_lite", transfer="g2p2g")
    with pytest.raises(ConfigError):
        H.RunConfig.from_dict({"bogus": 1})
    p = tmp_path / "c.json"
    p.write_text('{"l": 6, "boxes": 1, "frames": 2}')
    cfg = H.RunConfig.from_json(p).with_overrides(frames=3, l=None)
    assert (cfg.l, cfg.boxes, cfg.frames) == (6, 1, 3)
    assert len(H.build_scene(cfg).positions) == 6 ** 3 * 8


def test_snapshot_roundtrip_is_bit_exact(tmp_path, rng):
    # tests/test_bench.py:105-132: MPMF, u32 version 1, u32 count, f32 xyz
    pos = rng.uniform(-5, 5, (37, 3))
    path = tmp_path / "f.mpmf"
    H.write_snapshot(path, pos)
    blob = path.read_bytes()
    assert blob[:4] == b"MPMF" and len(blob) == 12 + 37 * 12
    assert np.array_equal(H.read_snapshot(path), pos.astype(np.float32))
    path.write_bytes(b"XXXX" + blob[4:])
    with pytest.raises(SimulationError):
        H.read_snapshot(path)
    assert H.CSV_COLUMNS[:3] == ("frame", "steps", "ms_total") and len(H.CSV_COLUMNS) == 12


@pytest.mark.gpu
def test_run_writes_csv_and_snapshots_matching_the_oracle(tmp_path):
    cfg = H.RunConfig(l=6, boxes=4, frames=2, out_csv=str(tmp_path / "t.csv"),
                      out_snap=str(tmp_path / "snap"), profile_phases=True)
    res = H.run(cfg)
    rows = list(csv.reader(open(cfg.out_csv)))
    assert tuple(rows[0]) == H.CSV_COLUMNS and len(rows) == 3
    assert [int(r[1]) for r in rows[1:]] == [36, 36]
    assert int(rows[1][-1]) == 6 ** 3 * 8 * 4 == res.particle_count
    assert float(rows[1][5]) > 0 and float(rows[1][7]) > 0          # p2g and g2p phase columns
    assert res.rebuild_gaps and res.mean_steps_between_rebuilds > 1
    # same scene through the oracle (bench.py:434-439 ordering), positions ordered by id
    spec = H.build_scene(cfg)
    cl = O.OracleCluster(1, spec.params, spec.material, spec.boundary, PipelineOptions())
    cl.seed(spec.positions, spec.velocities, spec.particle_mass)
    for _ in range(2):
        cl.run_frame()
    snap = H.read_snapshot(res.snapshot_paths[-1])
    ref = cl.positions_sorted_by_id()
    assert np.abs(snap - ref).max() <= 2e-5 * (spec.positions.max() - spec.positions.min())


@pytest.mark.gpu
def test_two_logical_workers_and_fountain_scene(tmp_path):
    one = H.run(H.RunConfig(l=6, boxes=4, frames=1, out_snap=str(tmp_path / "a")))
    two = H.run(H.RunConfig(l=6, boxes=4, frames=1, workers=2, out_snap=str(tmp_path / "b")))
    a, b = H.read_snapshot(one.snapshot_paths[0]), H.read_snapshot(two.snapshot_paths[0])
    assert np.abs(a - b).max() <= 1e-4                              # tests/test_multiworker.py:228-233
    f = H.run(H.RunConfig(scene="fountain_lite", dx=0.66, frame_dt=1 / 60, frames=3))
    assert [r.particle_count for r in f.rows] == [324, 648, 972]    # 27 x 12 cells per frame
    assert all(r.rebuild_count >= 1 for r in f.rows)               # emission forces a rebuild


@pytest.mark.gpu
def test_errors_carry_frame_and_step_context(monkeypatch):
    # tests/test_bench.py:242-248: a failing step is reported with its frame / step
    from paper_2111_00699_b200 import scenes
    orig = scenes.free_fall

    def near_the_domain_edge(**kw):
        w = orig(**kw)
        w.positions[:] = -60.0 * w.params.dx      # block coordinate 0: no room for the halo
        return w
    monkeypatch.setattr(scenes, "free_fall", near_the_domain_edge)
    with pytest.raises(SpatialDomainError) as e:
        H.run(H.RunConfig(scene="free_fall", frames=2))
    assert "frame 0" in str(e.value) and "step 0" in str(e.value)
