"""CPU tests of the host side: C-ABI surface, value types, partitioning, growth policy, scenes.
No compute call is made (there is no GPU here); the CUDA path must fail loudly instead of
falling back."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import mpm_oracle as O
import paper_2111_00699_b200 as P
from paper_2111_00699_b200 import _capi, memory, scenes
from paper_2111_00699_b200.build import build as build_core

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mpm_b200.h")


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mpm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    build_core()
    lib = ctypes.CDLL(_capi.LIB_PATH)
    names = _declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/mpm_b200.h but not exported"
    # and the binding covers exactly the declared surface
    assert sorted(_capi.EXPORTED_SYMBOLS) == names


def test_ctypes_structs_match_the_header(tmp_path):
    src = tmp_path / "sizes.c"
    src.write_text('#include <stdio.h>\n#include "mpm_b200.h"\nint main(void){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n",'
                   'sizeof(mpm_transfer_params),sizeof(mpm_store_view),sizeof(mpm_table_view),'
                   'sizeof(mpm_step_status),sizeof(mpm_grid_params),sizeof(mpm_guard),'
                   'sizeof(mpm_step_plan),sizeof(mpm_rebuild_plan),sizeof(mpm_rebuild_result),'
                   'sizeof(mpm_step_clock));return 0;}\n')
    exe = tmp_path / "sizes"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    sizes = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    assert sizes == [ctypes.sizeof(_capi.TransferParams), ctypes.sizeof(_capi.StoreView),
                     ctypes.sizeof(_capi.TableView), ctypes.sizeof(_capi.StepStatus),
                     ctypes.sizeof(_capi.GridParams), ctypes.sizeof(_capi.Guard),
                     ctypes.sizeof(_capi.StepPlan), ctypes.sizeof(_capi.RebuildPlan),
                     ctypes.sizeof(_capi.RebuildResult), ctypes.sizeof(_capi.StepClock)]


def test_no_cpu_fallback_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    from paper_2111_00699_b200.worker import CudaWorker
    with pytest.raises(P.ResourceError):
        CudaWorker(0, P.SharedRuntime(1), P.SimParams(dx=0.5, dt=1e-4),
                   P.Material.fixed_corotated(2.0, 1e5, 0.3), None)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2111_00699_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                text = open(os.path.join(dirpath, f)).read()
                # no import, no dlopen of the oracle library, no call of an oracle function
                # (comments may cite the oracle as the float64 definition of a model)
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "libmpm_oracle" not in text and not re.search(r"\borc_[a-z0-9_]+\s*\(", text), f


def test_partition_matches_reference_restatement(rng):
    # multiworker.py:114-137 / tests/test_multiworker.py: sizes differ by <= 1, remainder from worker 0
    pos = rng.uniform(0, 1, (1003, 3)) * np.array([1.0, 5.0, 2.0])
    for n in (1, 2, 3, 4, 8):
        a, b = P.partition_particles(pos, n), O.partition_particles(pos, n)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
        sizes = [len(x) for x in a]
        assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
        assert np.array_equal(np.sort(np.concatenate(a)), np.arange(1003))
        # slabs along the longest axis (y)
        for lo, hi in zip(a[:-1], a[1:]):
            assert pos[lo, 1].max() <= pos[hi, 1].min()
    with pytest.raises(P.RejectedInputError):
        P.partition_particles(pos, 0)
    assert [len(x) for x in P.partition_particles(np.zeros((0, 3)), 3)] == [0, 0, 0]


def test_growth_policy():
    # memory.py:18-22
    assert memory.grown_capacity(0, 0) == 0
    assert memory.grown_capacity(0, 10) == 40
    assert memory.grown_capacity(40, 20) == 40
    assert memory.grown_capacity(40, 21) == 84


def test_runtime_vmax_ring_and_efficiency():
    rt = P.SharedRuntime(3, initial_vmax=2.0)
    rt.publish_vmax(4, 1, 9.0)
    assert rt.global_vmax(1) == 9.0 and rt.global_vmax(0) == 2.0
    assert P.efficiency(100.0, 30.0, 4).e == pytest.approx(100.0 / 120.0)
    with pytest.raises(P.RejectedInputError):
        P.efficiency(0.0, 1.0, 2)


def test_value_types_validate_like_the_reference():
    with pytest.raises(P.RejectedInputError):
        P.SimParams(dx=0.0, dt=1e-4)
    with pytest.raises(P.RejectedInputError):
        P.SimParams(dx=0.5, dt=1e-4, lane_width=24)
    with pytest.raises(P.ConfigError):
        P.PipelineOptions(transfer="fused")
    with pytest.raises(P.ConfigError):
        P.BoundaryBox((0, 0, 0), (1, 1, 0))
    m = P.Material.fixed_corotated(2.0, 1.0e5, 0.3)
    assert m.mu == pytest.approx(1.0e5 / 2.6) and m.lam == pytest.approx(1.0e5 * 0.3 / (1.3 * 0.4))
    assert P.Material.fluid(1.0, 1.0e5).sound_speed() == pytest.approx(np.sqrt(7.0e5))
    p = P.SimParams(dx=0.5, dt=1e-4, cfl=0.5)
    assert P.cfl_dt(100.0, p, 1.0) == pytest.approx(0.5 * 0.5 / 100.0)
    assert P.cfl_dt(0.0, p, 0.01) == 0.01
    assert not P.free_zone_check((1.0, 1.0, 1.0), (0.0, 0.0, 0.0), 0.5)
    assert P.free_zone_check((6.5 * 0.5, 1.0, 1.0), (0.0, 0.0, 0.0), 0.5)


def test_scene_counts_and_reproducibility():
    # tests/test_bench.py:14-24 of the reference: 55 296 / 389 344 / 12 459 008 particles
    assert len(scenes.sand_blocks(l=12, boxes=4).positions) == 55296
    assert 4 * 23 ** 3 * 8 == 389344 and 16 * 46 ** 3 * 8 == 12459008
    a = scenes.sand_blocks(l=6, boxes=4, seed=5)
    b = scenes.sand_blocks(l=6, boxes=4, seed=5)
    assert np.array_equal(a.positions, b.positions)
    assert a.particle_mass == pytest.approx(2.0 * (25 / 64) ** 3 / 8)
    lo, hi = np.array(a.boundary.min_corner), np.array(a.boundary.max_corner)
    assert (a.positions > lo).all() and (a.positions < hi).all()
    # stratified: exactly ppc samples in every occupied cell
    cells = np.floor(a.positions / a.params.dx).astype(np.int64)
    _, counts = np.unique(cells, axis=0, return_counts=True)
    assert (counts == 8).all()
    f = scenes.fountain()
    pos, vel = f.emission.sample(3)
    pos2, _ = f.emission.sample(3)
    assert len(pos) == f.emission.per_frame == 27 * len(f.emission.cells) and np.array_equal(pos, pos2)
    assert (vel[:, 2] == 160.0).all()
    s = scenes.snow(l=5, boxes=1)
    assert len(s.positions) == 1000 and s.params.dx == 1.35


def test_mixed_sparse_scene_layout():
    """configs[4] generator: equal snow / sand populations in separated clusters."""
    from paper_2111_00699_b200 import scenes
    from paper_2111_00699_b200.errors import ConfigError
    W = scenes.mixed_sparse(l=4, pairs_side=2, domain_cells=128)
    snow, sand = W.populations
    assert len(snow.positions) == len(sand.positions) == 4 * 4 ** 3 * 8 and W.n_particles == 4096
    assert int(snow.material.kind) == 2 and int(sand.material.kind) == 3
    assert (snow.velocities == 0).all() and (sand.velocities[:, 2] == -150.0).all()
    # the sand box of a cluster sits above its snow box, clusters are > one box apart
    assert sand.positions[:, 2].min() > snow.positions[:, 2].max()
    xs = np.unique(np.floor(snow.positions[:, 0] / 56.0))
    assert len(xs) == 2
    # 16 x 2 x 50^3 x 8 = 32 M on 512^3 is what the defaults describe (not generated here)
    assert 16 * 2 * 50 ** 3 * 8 == 32_000_000
    with pytest.raises(ConfigError):
        scenes.mixed_sparse(l=200, pairs_side=4, domain_cells=512)


def test_oracle_populations_meet_on_the_grid():
    """Two material populations as two workers (oracle side of
    test_cuda_parity.py::test_mixed_populations_share_one_grid): mass is conserved per
    population and momentum is exchanged through the shared blocks."""
    from oracle import build as obuild
    obuild.build()
    from oracle import mpm_oracle as O
    from paper_2111_00699_b200 import PipelineOptions, scenes
    W = scenes.mixed_sparse(l=4, pairs_side=1, dx=25.0 / 64.0, domain_cells=64, gap_cells=1,
                            steps_per_frame=36, frame_dt=1.0 / 48.0)
    pops = [(p.positions, p.velocities, p.particle_mass) for p in W.populations]
    co = O.OracleCluster(2, W.params, [p.material for p in W.populations], W.boundary,
                         PipelineOptions(), initial_vmax=150.0)
    co.seed_populations(pops)
    m0 = [len(p.positions) * p.particle_mass for p in W.populations]   # staged until the first rebuild
    for s in range(30):
        co.run_step(s)
    assert [w.store.total_mass() for w in co.workers] == pytest.approx(m0, rel=1e-12)
    shared = np.intersect1d(co.workers[0].table.codes[:co.workers[0].table.count],
                            co.workers[1].table.codes[:co.workers[1].table.count])
    assert len(shared) > 0
    t = 30 * W.params.dt
    snow_pz = co.workers[0].store.total_momentum()[2]
    assert snow_pz < 1.2 * (-981.0 * t) * m0[0]      # pushed by the sand, not only by gravity


def _shm_rank(path, n_ranks, rank, rounds, queue):
    import ctypes as C
    import mmap
    import numpy as np
    from paper_2111_00699_b200 import _capi
    lib = _capi.lib()
    with open(path, "r+b") as f:
        mm = mmap.mmap(f.fileno(), int(lib.mpm_shm_bytes(n_ranks)))
    base = C.addressof(C.c_char.from_buffer(mm))
    ok = True
    for r in range(rounds):
        vals = (C.c_int64 * 3)(rank, r, 1000 * rank + r)
        out = np.empty((n_ranks, 3), dtype=np.int64)
        rc = lib.mpm_shm_allgather_i64(base, n_ranks, rank, vals, 3, out.ctypes.data, 20000)
        ok = ok and rc == 0 and all(tuple(out[q]) == (q, r, 1000 * q + r) for q in range(n_ranks))
    queue.put((rank, ok))


def test_shared_memory_rendezvous_of_three_processes(tmp_path):
    """mpm_shm_allgather_i64: the host barrier + integer exchange of the peer runtime's collective
    steps (SpinBarrier / SharedRuntime of multiworker.py:27-107 across processes), no GPU needed."""
    import multiprocessing as mp
    from paper_2111_00699_b200 import _capi
    n, rounds = 3, 200
    path = tmp_path / "segment"
    path.write_bytes(b"\0" * int(_capi.lib().mpm_shm_bytes(n)))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shm_rank, args=(str(path), n, r, rounds, q)) for r in range(n)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == [(r, True) for r in range(n)]
    # a rank that waits alone runs into the timeout (multiworker.py:66-69)
    import ctypes as C
    import mmap
    import numpy as np
    lib = _capi.lib()
    path.write_bytes(b"\0" * int(lib.mpm_shm_bytes(2)))
    with open(path, "r+b") as f:
        mm = mmap.mmap(f.fileno(), int(lib.mpm_shm_bytes(2)))
    out = np.empty((2, 1), dtype=np.int64)
    rc = lib.mpm_shm_allgather_i64(C.addressof(C.c_char.from_buffer(mm)), 2, 0, (C.c_int64 * 1)(7), 1,
                                   out.ctypes.data, 50)
    assert rc == -8


def test_run_config_accepts_the_reference_fields():
    """A reference RunConfig dump (bench.py:62-100 of the reference, barrier_timeout included)
    loads unchanged; lane_width is range-checked with the other counts."""
    from paper_2111_00699_b200.errors import ConfigError
    from paper_2111_00699_b200.harness import RunConfig
    cfg = RunConfig.from_dict({"scene": "sand_blocks", "l": 12, "boxes": 4, "workers": 2,
                               "barrier_timeout": 3.5, "transfer": "g2p2g"})
    assert cfg.barrier_timeout == 3.5
    with pytest.raises(ConfigError):
        RunConfig(lane_width=0)
    with pytest.raises(ConfigError):
        RunConfig.from_dict({"no_such_field": 1})


def test_plan_slabs_cuts_the_global_histogram_into_equal_shares():
    """dist.plan_slabs (dynamic re-partitioning): non-decreasing destinations, every worker within one
    bin's population of total / n, empty and degenerate histograms handled."""
    from paper_2111_00699_b200.dist import plan_slabs
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 8):
        hist = rng.integers(0, 50, size=512)
        dest = plan_slabs(hist, n)
        assert dest.min() >= 0 and dest.max() <= n - 1 and np.all(np.diff(dest) >= 0)
        got = np.bincount(dest, weights=hist, minlength=n)
        assert np.abs(got - hist.sum() / n).max() <= hist.max()
    assert plan_slabs(np.zeros(16, dtype=np.int64), 4).tolist() == [0] * 16
    one = np.zeros(16, dtype=np.int64); one[5] = 100          # everything in one bin: it cannot be split
    assert len(set(plan_slabs(one, 4)[5:6].tolist())) == 1
    with pytest.raises(ValueError):
        plan_slabs(np.ones(4), 0)


def test_population_layout_and_dist_surface():
    """The multi-rank helpers the GPU tests and bench.py import exist (a refactor once dropped two of
    them), and populations are dealt to ranks round-robin: rank r holds slab r // P of population r % P."""
    from paper_2111_00699_b200 import dist as D
    for name in ("DistRuntime", "DistWorker", "seed_rank", "plan_slabs", "migrate_rows", "repartition",
                 "population_layout", "seed_population_rank", "build_halo_lists"):
        assert callable(getattr(D, name)), name
    assert [D.population_layout(r, 4, 2) for r in range(4)] == [(0, 0, 2), (1, 0, 2), (0, 1, 2), (1, 1, 2)]
    assert D.population_layout(5, 8, 1) == (0, 5, 8)
    from paper_2111_00699_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        D.population_layout(0, 3, 2)


def test_committed_bench_lines_keep_the_contract():
    """Every bench line committed under profiles/ (one per scene + the default run) carries the keys the
    driver and the judge read: metric / value / unit / timing fields, a workload name, the clocks record,
    and -- where a dominant kernel was timed -- a roofline block whose fraction is achieved / peak and
    cannot exceed 1 (a fraction above 1 was how a timing bug showed up in round 2)."""
    import json
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lines = [json.loads(l) for l in open(os.path.join(root, "profiles", "r2f_scenes.jsonl")) if l.strip()]
    lines.append(json.load(open(os.path.join(root, "profiles", "r2f_bench_default.json"))))
    assert len(lines) >= 10
    for d in lines:
        for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                  "scaling", "vs_baseline", "dtype", "data", "config", "gpu_launches", "clocks"):
            assert k in d, (k, d.get("config", {}).get("workload"))
        assert d["metric"] == "particle_substeps_per_s" and d["higher_is_better"] is True and d["vs_baseline"] is None
        assert d["config"]["workload"] and "model" not in d["config"]
        assert d["gpu_launches"] > 0 and d["value"] > 0
        c = d["clocks"]
        assert c and c["sm_mhz"] > 0.9 * c["sm_max_mhz"] and not set(c["reasons"]) & {
            "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
        r = d.get("roofline")
        if r:
            assert r["bound"] == "hbm" and 0.0 < r["frac"] < 1.0
            assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=2e-3)
    default = lines[-1]
    assert default["e2e"]["h2d_bytes_per_step"] > 0 and default["e2e"]["d2h_bytes_per_step"] > 0
    assert default["cpu_baseline"]["kind"] in ("port", "reference") and default["cpu_baseline"]["cores"] >= 1
