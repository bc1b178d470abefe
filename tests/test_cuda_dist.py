"""DistWorker (one process per rank) on a single GPU: two/three gloo ranks share cuda:0, halo
rows staged through host memory -- the same worker code that runs one rank per GPU over NCCL."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(world, transfer, halo="sendrecv", mode="steps", batch=4, lazy=0, scene=""):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, MPM_DIST_BACKEND="gloo", MPM_TRANSFER=transfer, MPM_HALO=halo, MPM_MODE=mode,
               MPM_PEER_BATCH=str(batch), MPM_LAZY=str(lazy), MPM_SCENE=scene)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "dist_check.py")]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "DIST_CHECK_OK" in res.stdout, res.stdout[-3000:]
    print("\n".join(l for l in res.stdout.splitlines() if "dist_check" in l or "snow_slabs" in l or l.startswith("  rank")
                    or l.startswith("peer:")))


def test_two_ranks_split_against_reference_dump():
    _run(2, "split")


def test_three_ranks_fused():
    _run(3, "g2p2g")


# ---- peer-mapped halo rows + device-side step barrier (paper_2111_00699_b200/peer.py) ----------
# Two / three processes share cuda:0: each maps the others' raw rows through CUDA IPC (on a
# multi-GPU node the same mapping is NVLink peer memory), the grid update waits for the peers'
# step signals on the device and adds their rows in place.
def test_peer_mapped_two_ranks_host_paced_steps():
    _run(2, "split", halo="peer")


def test_peer_mapped_two_ranks_device_paced_frames_split():
    _run(2, "split", halo="peer", mode="frames")


def test_peer_mapped_three_ranks_device_paced_frames_fused():
    _run(3, "g2p2g", halo="peer", mode="frames")


def test_peer_mapped_two_ranks_one_guarded_step_per_host_call():
    _run(2, "g2p2g", halo="peer", mode="frames", batch=0)


def test_peer_mapped_frames_without_a_per_frame_collective():
    """lazy_flush: the second frame starts device-paced (no host collective at the frame boundary)."""
    _run(2, "g2p2g", halo="peer", mode="frames", lazy=1)


# ---- 4 and 8 ranks (MPM_MAX_PEERS, all-to-all mapping and tagging) ---------------------------------
def test_peer_mapped_four_ranks_device_paced_frames_fused():
    _run(4, "g2p2g", halo="peer", mode="frames")


def test_peer_mapped_eight_ranks_device_paced_frames_split():
    _run(8, "split", halo="peer", mode="frames")


def test_eight_ranks_sendrecv_fused():
    _run(8, "g2p2g")


@pytest.mark.parametrize("world", [4, 8])
def test_headline_scene_as_peer_mapped_slabs(world):
    """The 1.37 M snow-plasticity scene as 4 / 8 peer-mapped ranks sharing one B200 (functional): one
    device-paced frame, union of the slabs vs a single worker at the short-run bars; the grid
    update's barrier-wait / halo-byte counters are on and reported."""
    _run(world, "g2p2g", halo="peer", mode="frames", scene="snow")


# ---- dynamic re-partitioning (dist.repartition) -----------------------------------
@pytest.mark.parametrize("world,halo,transfer", [(2, "sendrecv", "split"), (2, "peer", "g2p2g"), (3, "peer", "split")])
def test_repartition_migrates_particles_and_keeps_the_result(world, halo, transfer):
    """A bad partition (70/30, slabs interleaved) is re-cut between two frames: particles migrate with
    their whole state, ids and mass are preserved, counts end balanced, and the 24-step state still
    matches the reference dump."""
    _run(world, transfer, halo=halo, scene="repartition")


# ---- material populations over ranks (configs[4]) ---------------------------------------------------
@pytest.mark.parametrize("world", [2, 4])
def test_material_populations_over_peer_mapped_ranks(world):
    """Snow + sand populations as 2 / 4 peer-mapped ranks (2 populations x 1 / 2 slabs, each rank with
    its population's material) against the two-population run of one process."""
    _run(world, "g2p2g", halo="peer", scene="mixed")
