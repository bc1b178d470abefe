#!/usr/bin/env python
"""Benchmark of the MLS-MPM substep hot path (BASELINE.json: "ms/frame & M particle-substeps/s,
snow 1.33M MLS-MPM").

    python bench.py --gpus 1 --steps K --warmup W            # CUDA core (this repo)
    python bench.py --impl reference --gpus N --steps K ...  # the reference's CPU path
    torchrun ... bench.py --gpus N ...                       # one rank per GPU

A "step" is one FRAME of the workload: `steps_per_frame` substeps (rebuild-mapping amortised
inside, as in the reference's run_frame).  `value` = particle-substeps per second with the
particles resident in HBM; `e2e` = the same through the public API with host buffers: every
step uploads the particle state from pinned host memory (seed), runs the frame and reads
the positions back.  One JSON line on stdout (rank 0).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "particle_substeps_per_s"
UNIT = "M particle-substeps/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scene", default="snow", choices=["snow", "snow_fc", "sand64k", "sand_mini",
                                                        "sand389k", "sand1m", "sand10m", "sand32m", "fountain",
                                                        "mixed4m", "mixed32m"])
    ap.add_argument("--transfer", default="g2p2g", choices=["split", "g2p2g"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--host-paced", action="store_true",
                    help="fountain: CFL dt computed by the host every step (the round-1 path)")
    ap.add_argument("--no-pinned-variant", action="store_true",
                    help="snow only: skip the fixed-corotated (reference-pinned) run of the same scene")
    ap.add_argument("--ref-substeps", type=int, default=2,
                    help="substeps per step of the reference arm (bounded sample)")
    return ap.parse_args()


def build_world(scene):
    W = _build_world(scene)
    W.tag = scene
    return W


def _build_world(scene):
    from paper_2111_00699_b200 import scenes
    if scene == "snow":
        return scenes.snow(plastic=SNOW_PLASTIC)
    if scene == "snow_fc":
        return scenes.snow(plastic=False)
    if scene == "sand64k":
        return scenes.sand_blocks(l=20, boxes=1)
    if scene == "sand_mini":
        return scenes.sand_blocks(l=12, boxes=4)
    if scene == "sand389k":
        return scenes.sand_blocks(l=23, boxes=4)
    if scene == "sand1m":
        return scenes.sand_blocks(l=32, boxes=4)
    if scene == "sand10m":
        return scenes.sand_blocks(l=43, boxes=16)
    if scene == "sand32m":
        return scenes.sand_blocks(l=63, boxes=16)
    if scene == "fountain":
        # configs[1]: 14 256 particles emitted per frame (radius 5 dx) up to the paper's 143.5 K
        return scenes.fountain(radius=5 * 0.66)
    raise ValueError(scene)


# headline scene: snow with the clamp+hardening plasticity (parity unpinned: no reference model);
# --scene snow_fc times the reference-pinned fixed-corotated variant of the same scene
SNOW_PLASTIC = True


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    QUERY = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.proc = None
        self.gpu_index = gpu_index
        self.t0 = self.t1 = None

    def mark_begin(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu_index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        """Ends the sampling; returns the summary of the window marked with mark_begin / mark_end."""
        if self.proc is None:
            self.lines = None
            return self.window(self.t0, self.t1)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        self.lines = out.strip().splitlines()
        return self.window(self.t0, self.t1)

    def window(self, t0, t1):
        """Clocks / throttle reasons of the samples taken in [t0, t1] (50 ms of slack either side)."""
        if getattr(self, "lines", None) is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        import datetime
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            if t0 is not None and t1 is not None:
                try:
                    ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    continue
                if ts < t0 - 0.05 or ts > t1 + 0.05:
                    continue
            try:
                sm.append(float(f[1])); smax.append(float(f[2])); power.append(float(f[3]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)),
                "power_w_max": float(max(power)), "samples": len(sm), "reasons": sorted(reasons)}


def measured_peak_gbs():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def algorithmic_bytes(kind, transfer, n_particles, touched_blocks):
    """SURVEY.md section 8(d) / DESIGN.md: bytes the dominant transfer kernel must move.
    fused elastic: read {x3,m,F9}=52 B + write {x3,v3,F9}=60 B per particle; fluid 20+28;
    plastic scalar +8; grid: gather read 16 B + scatter write-back 16 B per touched node."""
    if transfer == "g2p2g":
        per_p = {0: 48, 1: 112, 2: 120, 3: 120}[kind]
        per_node = 32
    else:   # split: the P2G kernel alone (dominant of the two)
        per_p = {0: 68, 1: 100, 2: 104, 3: 104}[kind]
        per_node = 16
    return n_particles * per_p + touched_blocks * 64 * per_node


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2111_00699_b200 import PipelineOptions, SharedRuntime, _capi
    from paper_2111_00699_b200.worker import CudaWorker

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} needs {args.gpus} ranks (torch.distributed.run); "
                         f"WORLD_SIZE is {world}")
    # MPM_DIST_BACKEND=gloo lets several ranks share one GPU (functional check of the N > 1 path
    # on a single-GPU box); the product configuration is one rank per GPU over NCCL
    backend = os.environ.get("MPM_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    lib = _capi.lib()
    opts = PipelineOptions(transfer=args.transfer, fused_threshold=1 << 62)

    halo = os.environ.get("MPM_HALO", "peer")   # peer: rows read in place over NVLink (peer.py); sendrecv: NCCL
    if world > 1 and halo == "peer":
        # peer memory must really be reachable from every rank's device; if not (no P2P between two
        # of the GPUs, IPC disabled in the container) the literal send/recv protocol still runs
        from paper_2111_00699_b200.peer import PeerRuntime
        if not PeerRuntime(dev, initial_vmax=150.0).probe():
            halo = "sendrecv"
            if rank == 0:
                print("peer-mapped memory is not available on this box: halo rows over send/recv",
                      file=sys.stderr, flush=True)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()           # nvidia-smi needs a moment to start: launch it before the warm-up

    def make_arm(W):
        """Everything one workload needs: its slab of the particles and a worker factory."""
        n = len(W.positions)
        vmax0 = float(np.abs(W.velocities).max())
        if world > 1:
            from paper_2111_00699_b200 import partition_particles
            part = partition_particles(W.positions, world)[rank]
        else:
            part = np.arange(n, dtype=np.int64)
        my_pos = np.ascontiguousarray(W.positions[part], dtype=np.float32)
        my_vel = np.ascontiguousarray(W.velocities[part], dtype=np.float32)

        def fresh_worker():
            if world > 1:
                from paper_2111_00699_b200.dist import DistRuntime, DistWorker
                if halo == "peer":
                    from paper_2111_00699_b200.peer import PeerDistWorker, PeerRuntime
                    return PeerDistWorker(PeerRuntime(dev, initial_vmax=vmax0), W.params, W.material,
                                          W.boundary, opts, device=dev, count_stats=False, lazy_flush=True)
                return DistWorker(DistRuntime(dev, initial_vmax=vmax0), W.params, W.material, W.boundary,
                                  opts, device=dev, count_stats=False)
            return CudaWorker(0, SharedRuntime(1, initial_vmax=vmax0), W.params, W.material, W.boundary,
                              opts, device=dev, count_stats=False, fuse_clear=True, lazy_flush=True)
        return n, part, my_pos, my_vel, fresh_worker

    def resident(W, steps, warmup):
        """`value` leg: K frames with the particle state resident in HBM, CUDA events on the launching
        stream, max over ranks; roofline of the dominant kernel from events inside the same region."""
        n, part, my_pos, my_vel, fresh_worker = make_arm(W)
        spf = W.params.steps_per_frame
        w = fresh_worker()
        w.seed_particles(my_pos, my_vel, W.particle_mass, ids=part)
        for _ in range(warmup):
            w.run_frame()
        barrier()
        w.time_kernels = True
        w.kernel_events.clear()
        l0 = lib.mpm_launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reb0 = len(w.rebuild_steps)
        barrier()
        t_begin = time.time()
        e0.record()
        for _ in range(steps):
            w.run_frame()
        e1.record()
        barrier()
        t_end = time.time()
        total_ms = max_over_ranks(e0.elapsed_time(e1))
        launches = int(lib.mpm_launch_count() - l0)
        rebuilds = len(w.rebuild_steps) - reb0
        ms_per_step = total_ms / steps
        value = n * spf * steps / (total_ms * 1e-3) / 1e6
        # dominant kernel: average launch duration from CUDA events on the launching stream
        w.time_kernels = False
        dom = "mpm_g2p2g" if args.transfer == "g2p2g" else "mpm_p2g"
        durs = [a.elapsed_time(b) for name, a, b in w.kernel_events if name == dom]
        all_kernel_ms = {}
        for name, a, b in w.kernel_events:
            all_kernel_ms[name] = all_kernel_ms.get(name, 0.0) + a.elapsed_time(b)
        # Steps enqueued in batches from C time ONE launch per batch, at a rotating position (an event between
        # two kernels of the chain would serialise what programmatic dependent launch overlaps); the
        # dominant kernel's total is its mean duration x its launches in the region: every substep
        # except, for the fused transfer, the rebuild steps (those run the split P2G).
        n_dom = spf * steps - (rebuilds if dom == "mpm_g2p2g" else 0)
        if durs:
            all_kernel_ms[dom] = float(np.mean(durs)) * n_dom
        # touched pblocks of one substep (flags survive when the clear is not fused into the update)
        w.fuse_clear, w.pipelined = False, False
        step = w._global_step
        w.dt = W.params.dt
        w.run_step(step)
        touched = int(w.table._touched[step & 1].data[:w.table.count].sum().item())
        n_local = len(part)
        peak, peak_src = measured_peak_gbs()
        roofline = None
        if durs:
            avg_ms = float(np.mean(durs))
            abytes = algorithmic_bytes(int(W.material.kind), args.transfer, n_local, touched)
            achieved = abytes / (avg_ms * 1e-3) / 1e9
            traffic = TRAFFIC_NCU.get(W.tag) if (world == 1 and args.transfer == "g2p2g") else None
            roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                        "unit": "GB/s", "frac": round(achieved / peak, 4),
                        "traffic": traffic[0] if traffic else None,
                        "traffic_source": traffic[1] if traffic else None,
                        "peak_source": peak_src, "avg_launch_ms": round(avg_ms, 4),
                        "algorithmic_bytes_per_launch": int(abytes), "launches_timed": len(durs),
                        "launches_in_region": int(n_dom),
                        "kernel_share_of_step": round(avg_ms * n_dom / total_ms, 3),
                        "kernel_ms_per_step": {k: round(v / steps, 4) for k, v in all_kernel_ms.items()}}
        config = {"workload": W.name, "particles": n, "substeps_per_step": spf,
                  "step": "one frame", "dx": W.params.dx, "dt": W.params.dt,
                  "transfer": args.transfer, "material": W.material.kind.name,
                  "parallelism": (f"{world} spatial slabs, halo rows read in place over NVLink peer memory, "
                                  "device-side step barrier" if halo == "peer" else
                                  f"{world} spatial slabs, halo rows over NCCL send/recv") if world > 1
                  else "1 GPU", "rank0_particles": n_local,
                  "pblocks": int(w.table.count), "groups": int(w.store.n_groups),
                  "rebuilds_in_timed_region": rebuilds, "touched_pblocks": touched,
                  "speculative_steps_discarded": int(w.speculative_discards),
                  # a frame ends with the fused gather pending; it completes on the first access to the
                  # particle store (the reference flushes at every frame end, pipeline.py:877-880)
                  "lazy_flush": bool(getattr(w, "lazy_flush", False)),
                  "fuse_clear": world == 1,
                  "l2_policy": (("inputs larger than L2: " if n_local * w.store.nch * 4 > 126e6 else
                                 "per-GPU working set SMALLER than L2 at this rank count (strong scaling of a "
                                 "fixed scene); no flush between steps, every substep rewrites the whole state: ")
                                + f"{n_local * w.store.nch * 4 / 1e6:.0f} MB particle state per GPU "
                                "streamed every substep (L2 126 MB)")}
        return {"value": round(value, 2), "ms_per_step": round(ms_per_step, 4), "roofline": roofline,
                "config": config, "launches": launches, "window": (t_begin, t_end)}

    W = build_world(args.scene)
    main_arm = resident(W, args.steps, args.warmup)
    n = len(W.positions)
    spf = W.params.steps_per_frame

    # The headline scene runs the snow plasticity model, pinned by numpy's SVD + the published closed
    # forms (tests/golden/plastic.npz) but absent from the reference package; the SAME particle set
    # with the reference's own fixed-corotated material is timed next to it, same K and W.
    pinned = None
    if args.scene == "snow" and not args.no_pinned_variant:
        Wfc = build_world("snow_fc")
        arm = resident(Wfc, args.steps, args.warmup)
        pinned = {"workload": Wfc.name, "value": arm["value"], "unit": UNIT, "ms_per_step": arm["ms_per_step"],
                  "material": Wfc.material.kind.name,
                  "roofline_frac": arm["roofline"]["frac"] if arm["roofline"] else None,
                  "avg_launch_ms": arm["roofline"]["avg_launch_ms"] if arm["roofline"] else None,
                  "rebuilds_in_timed_region": arm["config"]["rebuilds_in_timed_region"]}

    # end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        _, part, my_pos, my_vel, fresh_worker = make_arm(W)
        n_local = len(part)
        # end-to-end inputs live in pinned host memory (allocated once, outside the timed region)
        pin_pos = torch.from_numpy(my_pos).pin_memory()
        pin_vel = torch.from_numpy(my_vel).pin_memory()
        pin_ids = torch.from_numpy(np.ascontiguousarray(part, dtype=np.int64)).pin_memory()
        w2 = fresh_worker()
        k_e2e = max(2, min(args.steps, 4))
        E2E_WARM = 3      # untimed: the second worker's buffers, pinned staging and the allocator settle
        pending = None
        # Every step's inputs start in pinned host memory.  They are uploaded on a copy stream into
        # one of two device buffer sets while the previous frame computes, and handed to
        # replace_particles as device tensors; the snapshot of a frame travels back on the store's
        # copy stream while the next frame runs.  Both copies of every step lie inside the timed
        # region.
        main, copy = torch.cuda.current_stream(), torch.cuda.Stream(device=dev)
        sets = [(torch.empty_like(pin_pos, device=dev), torch.empty_like(pin_vel, device=dev),
                 torch.empty_like(pin_ids, device=dev)) for _ in range(2)]
        uploaded, consumed = [None, None], [None, None]

        def upload(k):
            with torch.cuda.stream(copy):
                if consumed[k] is not None:
                    copy.wait_event(consumed[k])      # the frame that read this set has taken it
                for dst, src in zip(sets[k], (pin_pos, pin_vel, pin_ids)):
                    dst.copy_(src, non_blocking=True)
                uploaded[k] = torch.cuda.Event()
                uploaded[k].record(copy)

        upload(0)
        for it in range(E2E_WARM + k_e2e):
            k = it & 1
            if it == E2E_WARM:
                barrier()
                t0 = time.perf_counter()
            upload(1 - k)                             # the next step's inputs, during this frame
            main.wait_event(uploaded[k])
            w2.replace_particles(sets[k][0], sets[k][1], W.particle_mass, sets[k][2])
            w2.run_frame()
            consumed[k] = torch.cuda.Event()
            consumed[k].record(main)
            handle = w2.store.positions_with_ids_async()
            if pending is not None:
                out_pos, out_ids = pending.wait()
            pending = handle
        out_pos, out_ids = pending.wait()
        barrier()
        dt_e2e = max_over_ranks((time.perf_counter() - t0) / k_e2e)
        e2e = {"value": round(n * spf / dt_e2e / 1e6, 2), "unit": UNIT,
               "h2d_bytes_per_step": int(n_local * (7 * 4 + 8)),   # x3, v3, m fp32 + id int64
               "d2h_bytes_per_step": int(out_pos.nbytes + out_ids.nbytes),
               "ms_per_step": round(dt_e2e * 1e3, 3), "steps": k_e2e,
               "api": "pinned x, v, ids -> device on a copy stream (during the previous frame) + "
                      "CudaWorker.replace_particles(device tensors) + run_frame() + "
                      "store.positions_with_ids_async() into pinned buffers (waited for one step later); every step re-seeds the scene's "
                      "initial state from the host, so it times the scene's first frame (fewer rebuilds "
                      "and less yielding than the frames `value` is taken over)"}

    clocks = None
    if rank == 0:
        sampler.mark_begin(); sampler.mark_end()
        sampler.stop()
        clocks = sampler.window(*main_arm["window"])
        if pinned is not None:
            pinned["clocks"] = sampler.window(*arm["window"])

    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        cpu = cpu_baseline(W, substeps=2, threads=1)

    if rank == 0:
        line = {
            "metric": METRIC, "value": main_arm["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": main_arm["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": main_arm["config"],
            "ms_per_frame": main_arm["ms_per_step"],
            "clocks": clocks, "gpu_launches": main_arm["launches"], "e2e": e2e,
            "roofline": main_arm["roofline"], "cpu_baseline": cpu,
        }
        if pinned is not None:
            line["reference_pinned_variant"] = pinned
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel, per launch, from the
# committed `ncu --set full` capture of the fused kernel on the 1.37 M scene
# (profiles/r1_l_fused_snow_final_metrics.csv: 96.5 MB read + 52.7 MB write; r1_l_fused_snow_fc_final: 89.8 + 40.8);
# only quoted for those scenes
TRAFFIC_NCU = {"snow": (136.9e6, "profiles/r2f_fused_snow_metrics.csv (ncu --set full, one launch; not measured in this run)"),
               "snow_fc": (124.9e6, "profiles/r2f_fused_snow_fc_metrics.csv (ncu --set full, one launch; not measured in this run)")}


FOUNTAIN_CAP = 143_500      # the paper's interactive fountain holds at most 143.5 K particles


def run_fountain(args):
    """configs[1]: water fountain with a per-frame emitter, CFL-auto dt paced by the device
    (mpm_step_clock), split transfers (the emitter forbids the fused transfer, bench.py:116-118 of
    the reference).  14 256 particles are emitted per frame; a sink slab just below the apex of the
    jet takes them out again, and the emitter pauses whenever another frame's worth would exceed the
    paper's 143.5 K cap, so the population holds just under it.  Emissions are sampled before the
    clock starts (synthetic input in pinned host memory); their upload, the rebuild they force and
    the frame are inside it."""
    import torch
    from paper_2111_00699_b200 import PipelineOptions, SharedRuntime, _capi
    from paper_2111_00699_b200.worker import CudaWorker
    torch.cuda.set_device(0)
    W = build_world("fountain")
    per_frame = W.emission.per_frame
    w = CudaWorker(0, SharedRuntime(1, initial_vmax=160.0), W.params, W.material, W.boundary,
                   PipelineOptions(transfer="split"), count_stats=False, fuse_clear=True)
    w.cfl_mode = True
    w.device_clock = not args.host_paced
    cz = float(np.mean(W.emission.cells[:, 2]) + 0.5) * W.params.dx
    apex = 160.0 ** 2 / (2 * 981.0)
    z_face = cz + apex - 0.05                      # 9 frames of flight
    w.set_sink((-1e4, -1e4, z_face), (1e4, 1e4, 1e4))
    sampler = ClockSampler(0)
    sampler.start()

    n_frames_max = 40 + args.warmup + args.steps
    staged = []
    for f in range(n_frames_max):
        pos, vel = W.emission.sample(f)
        staged.append((torch.from_numpy(pos.astype(np.float32)).pin_memory(),
                       torch.from_numpy(vel.astype(np.float32)).pin_memory()))
    frame = 0
    emitted = 0

    def one_frame():
        nonlocal frame, emitted
        if w.store.count + w.store.staged_count + per_frame <= FOUNTAIN_CAP:
            pos, vel = staged[emitted % len(staged)]
            w.append_particles(pos, vel, W.particle_mass)
            emitted += 1
        w.run_frame()
        frame += 1

    # fill up to the steady population (the sink starts draining after ~9 frames), then W warm-up frames
    while frame < 40 and not (frame > 12 and w.store.count + per_frame > FOUNTAIN_CAP - 2 * per_frame):
        one_frame()
    fill_frames = frame
    for _ in range(args.warmup):
        one_frame()
    torch.cuda.synchronize()
    w.time_kernels = True
    w.kernel_events.clear()
    l0 = _capi.lib().mpm_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    work, steps, counts, frame_ms = 0, 0, [], []
    reb0 = len(w.rebuild_steps)
    sampler.mark_begin()
    e0.record()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        one_frame()
        frame_ms.append((time.perf_counter() - t0) * 1e3)
        work += w.store.count * w.frame_steps
        steps += w.frame_steps
        counts.append(int(w.store.count))
    e1.record()
    torch.cuda.synchronize()
    sampler.mark_end()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    w.time_kernels = False
    durs = [a.elapsed_time(b) for name, a, b in w.kernel_events if name == "mpm_p2g"]
    roofline = None
    if durs:
        # touched pblocks of one substep
        w.fuse_clear, w.pipelined = False, False
        step = w._global_step
        w.run_step(step)
        touched = int(w.table._touched[step & 1].data[:w.table.count].sum().item())
        peak, peak_src = measured_peak_gbs()
        avg_ms = float(np.mean(durs))
        abytes = algorithmic_bytes(int(W.material.kind), "split", int(np.mean(counts)), touched)
        achieved = abytes / (avg_ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "kernel": "mpm_p2g", "achieved": round(achieved, 1), "peak": peak,
                    "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                    "peak_source": peak_src, "avg_launch_ms": round(avg_ms, 4),
                    "algorithmic_bytes_per_launch": int(abytes), "launches_timed": len(durs),
                    "launches_in_region": int(steps),
                    "kernel_share_of_step": round(avg_ms * steps / ms, 3),
                    "note": "working set (particle state + grid) is L2-resident at this size: the HBM "
                            "roofline is the reporting denominator, launch latency the actual bound"}
    line = {"metric": METRIC, "value": round(work / (ms * 1e-3) / 1e6, 2), "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "fountain (emitter radius 5 dx, 14 256 particles / frame, CFL-auto dt, "
                                   "sink below the apex, population capped at 143.5 K)",
                       "particles_min": int(min(counts)), "particles_max": int(max(counts)),
                       "particle_cap": FOUNTAIN_CAP, "removed_by_sink": int(w.removed_count),
                       "substeps_per_step": round(steps / args.steps, 2),
                       "step": "one frame incl. emission upload and the rebuild it forces",
                       "transfer": "split", "material": W.material.kind.name,
                       "pacing": "device step clock (dt computed by the grid update, steps enqueued in "
                                 "batches)" if w.device_clock else "host (one guarded step ahead)",
                       "fill_frames": fill_frames, "rebuilds_in_timed_region": len(w.rebuild_steps) - reb0,
                       "speculative_steps_discarded": int(w.speculative_discards),
                       "frame_ms_host_min_max": [round(min(frame_ms), 3), round(max(frame_ms), 3)],
                       "fps": round(1e3 * args.steps / ms, 1),
                       "l2_policy": "working set smaller than L2 (by design of the configuration: 143 K "
                                    "particles = 10 MB); no flush between frames, every substep rewrites it"},
            "ms_per_frame": round(ms / args.steps, 4),
            "gpu_launches": int(_capi.lib().mpm_launch_count() - l0), "e2e": None, "roofline": roofline,
            "cpu_baseline": None, "clocks": clocks}
    print(json.dumps(line), flush=True)


def run_mixed(args):
    """configs[4]: mixed snow / sand populations on a 512^3 sparse grid.  `mixed32m` is the whole
    32 M-particle scene on one GPU (6.6 GB of particle state), `mixed4m` its one-eighth (the
    per-GPU share of the 8-GPU configuration).  Two logical workers (one per material) share
    the grid through the in-kernel peer-row reduction of the grid update."""
    import torch
    from paper_2111_00699_b200 import CudaCluster, PipelineOptions, _capi, scenes
    torch.cuda.set_device(0)
    sampler = ClockSampler(0)
    sampler.start()
    W = scenes.mixed_sparse(l=50, pairs_side=4) if args.scene == "mixed32m" else scenes.mixed_sparse(l=40, pairs_side=2)
    cl = CudaCluster(2, W.params, [p.material for p in W.populations], W.boundary,
                     PipelineOptions(transfer=args.transfer, fused_threshold=1 << 62), initial_vmax=150.0,
                     count_stats=False)
    cl.seed_populations([(p.positions.astype(np.float32), p.velocities.astype(np.float32), p.particle_mass)
                         for p in W.populations])
    n, spf = W.n_particles, W.params.steps_per_frame
    for _ in range(args.warmup):
        cl.run_frame()
    torch.cuda.synchronize()
    for w in cl.workers:
        w.time_kernels = True
        w.kernel_events.clear()
    l0 = _capi.lib().mpm_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler.mark_begin()
    e0.record()
    for _ in range(args.steps):
        cl.run_frame()
    e1.record()
    torch.cuda.synchronize()
    sampler.mark_end()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    dom = "mpm_g2p2g" if args.transfer == "g2p2g" else "mpm_p2g"
    tables = [int(w.table.count) for w in cl.workers]
    shared = int(len(np.intersect1d(cl.workers[0].table.codes, cl.workers[1].table.codes)))
    # roofline of the dominant kernel: one launch per population and substep; the two populations
    # are equal in size, so their launches are pooled
    durs, touched = [], []
    for w in cl.workers:
        w.time_kernels = False
        durs += [a.elapsed_time(b) for name, a, b in w.kernel_events if name == dom]
    step = cl.workers[0]._global_step
    for w in cl.workers:
        w.fuse_clear = False
    cl.run_step(step)
    for w in cl.workers:
        touched.append(int(w.table._touched[step & 1].data[:w.table.count].sum().item()))
    roofline = None
    if durs:
        peak, peak_src = measured_peak_gbs()
        avg_ms = float(np.mean(durs))
        per_pop = n // 2
        abytes = algorithmic_bytes(2, args.transfer, per_pop, int(np.mean(touched)))
        achieved = abytes / (avg_ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_src,
                    "avg_launch_ms": round(avg_ms, 4), "algorithmic_bytes_per_launch": int(abytes),
                    "launches_timed": len(durs), "launches_in_region": len(durs),
                    "kernel_share_of_step": round(float(np.sum(durs)) / ms, 3)}
    line = {"metric": METRIC, "value": round(n * spf * args.steps / (ms * 1e-3) / 1e6, 2), "unit": UNIT,
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": W.name, "particles": n, "substeps_per_step": spf, "step": "one frame",
                       "transfer": args.transfer, "material": "SNOW + SAND populations",
                       "pblocks_per_population": tables, "shared_pblocks": shared,
                       "touched_pblocks_per_population": touched,
                       "grid_cells": f"{W.domain_cells}^3",
                       "occupied_fraction_of_grid": round(sum(tables) * 64 / W.domain_cells ** 3, 4),
                       "rebuilds": [len(w.rebuild_steps) for w in cl.workers],
                       "timing_note": "every transfer launch carries CUDA events in this scene (the cluster "
                                      "is stepped from Python), i.e. no programmatic overlap between kernels",
                       "l2_policy": f"inputs larger than L2: {n * 26 * 4 / 1e6:.0f} MB particle state streamed every substep"},
            "ms_per_frame": round(ms / args.steps, 4),
            "gpu_launches": int(_capi.lib().mpm_launch_count() - l0), "e2e": None, "roofline": roofline,
            "cpu_baseline": None, "clocks": clocks}
    print(json.dumps(line), flush=True)


def run_mixed_ranks(args):
    """configs[4] over N ranks: 2 material populations x N/2 slabs, one peer-mapped rank per (population,
    slab) -- dist.population_layout.  On the 8-GPU box that is 4 slabs per population; several ranks
    may share a device (MPM_DIST_BACKEND=gloo: functional check on one GPU)."""
    import torch
    import torch.distributed as dist
    from paper_2111_00699_b200 import PipelineOptions, _capi, scenes
    from paper_2111_00699_b200.dist import population_layout, seed_population_rank
    from paper_2111_00699_b200.peer import PeerDistWorker, PeerRuntime
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    backend = os.environ.get("MPM_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group(backend, device_id=dev) if backend == "nccl" else dist.init_process_group(backend)
    W = scenes.mixed_sparse(l=50, pairs_side=4) if args.scene == "mixed32m" else scenes.mixed_sparse(l=40, pairs_side=2)
    pop, slab, n_slabs = population_layout(rank, world, len(W.populations))
    w = PeerDistWorker(PeerRuntime(dev, initial_vmax=150.0), W.params, W.populations[pop].material, W.boundary,
                       PipelineOptions(transfer=args.transfer, fused_threshold=1 << 62), device=dev,
                       count_stats=False, lazy_flush=True)
    mine = seed_population_rank(w, W.populations)
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    for _ in range(args.warmup):
        w.run_frame()

    def barrier():
        dist.barrier()
        torch.cuda.synchronize()
    barrier()
    l0 = _capi.lib().mpm_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler.mark_begin()
    e0.record()
    for _ in range(args.steps):
        w.run_frame()
    e1.record()
    barrier()
    sampler.mark_end()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    info = [None] * world
    dist.all_gather_object(info, (pop, slab, len(mine), int(w.table.count), w.collective_steps,
                                  w.device_paced_steps, len(w.rebuild_steps)))
    if rank == 0:
        n, spf = W.n_particles, W.params.steps_per_frame
        line = {"metric": METRIC, "value": round(n * spf * args.steps / (ms * 1e-3) / 1e6, 2), "unit": UNIT,
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": W.name, "particles": n, "substeps_per_step": spf, "step": "one frame",
                           "transfer": args.transfer, "material": "SNOW + SAND populations",
                           "parallelism": f"{world} peer-mapped ranks = 2 populations x {n_slabs} slabs",
                           "ranks": [{"population": a, "slab": b, "particles": c, "pblocks": d,
                                      "collective_steps": e, "device_paced_steps": f, "rebuilds": g}
                                     for a, b, c, d, e, f, g in info],
                           "l2_policy": "inputs larger than L2 per rank unless the ranks share one device"},
                "ms_per_frame": round(ms / args.steps, 4),
                "gpu_launches": int(_capi.lib().mpm_launch_count() - l0), "e2e": None, "roofline": None,
                "cpu_baseline": None, "clocks": sampler.stop()}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def cpu_baseline(W, substeps, threads, warm=True):
    """The CPU oracle (C restatement of the reference, oracle/) timed on the host cores on a
    bounded sample: the full scene, rebuild + `substeps` substeps."""
    from oracle import build as obuild
    obuild.build()
    from oracle import mpm_oracle as O
    from paper_2111_00699_b200 import PipelineOptions
    n = len(W.positions)
    threads = max(1, int(threads))
    cl = O.OracleCluster(threads, W.params, W.material, W.boundary, PipelineOptions(),
                         initial_vmax=float(np.abs(W.velocities).max()), threads=threads > 1)
    cl.seed(W.positions, W.velocities, W.particle_mass)
    cl.run_step(0)        # rebuild + first substep: not timed (amortised in the GPU number too)
    t0 = time.perf_counter()
    for s in range(1, 1 + substeps):
        cl.run_step(s)
    dt = time.perf_counter() - t0
    return {"value": round(n * substeps / dt / 1e6, 3), "unit": UNIT, "cores": threads,
            "kind": "port", "sample": f"full scene ({n} particles), {substeps} substeps after the "
                                      f"rebuild step, {threads} worker thread(s)",
            "seconds": round(dt, 2)}


def run_reference(args):
    """Reference arm: the reference's own CPU implementation of the path.  The reference is
    Python + numba (nothing to compile into oracle/_ref and /root/reference does not exist
    on the GPU box), so this times the pinned C oracle port with one worker per host core."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    W = build_world(args.scene)
    n = len(W.positions)
    cores = min(os.cpu_count() or 1, 32)
    from oracle import build as obuild
    obuild.build()
    from oracle import mpm_oracle as O
    from paper_2111_00699_b200 import PipelineOptions
    cl = O.OracleCluster(cores, W.params, W.material, W.boundary, PipelineOptions(),
                         initial_vmax=float(np.abs(W.velocities).max()), threads=cores > 1)
    cl.seed(W.positions, W.velocities, W.particle_mass)
    S = args.ref_substeps
    step = 0
    cl.run_step(step); step += 1                 # rebuild step (untimed)
    for _ in range(args.warmup):
        for _ in range(S):
            cl.run_step(step); step += 1
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for _ in range(S):
            cl.run_step(step); step += 1
    dt = time.perf_counter() - t0
    value = n * S * args.steps / dt / 1e6
    sample = (f"full scene ({n} particles), {S} substeps per step, {cores} worker threads "
              f"(one per core), rebuild step excluded")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": W.name, "particles": n, "substeps_per_step": S,
                   "step": f"{S} substeps (bounded sample of one frame)"},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse_args()
    if a.impl == "reference":
        run_reference(a)
    elif a.scene == "fountain":
        run_fountain(a)
    elif a.scene.startswith("mixed"):
        run_mixed_ranks(a) if int(os.environ.get("WORLD_SIZE", "1")) > 1 else run_mixed(a)
    else:
        run_ours(a)
