"""world_size-2 gloo tests (CPU) of the one-process-per-GPU protocol: the step barrier /
vmax ring, the block-code exchange, the halo row lists and the row exchange, driven with
real block tables and nodal rows produced by the CPU oracle for a two-worker run."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                          WORLD_SIZE=str(world))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from conftest import elastic_setup, golden
        from oracle import mpm_oracle as O
        from paper_2111_00699_b200 import PipelineOptions
        from paper_2111_00699_b200.dist import DistRuntime, build_halo_lists

        g = golden("two_worker.npz")
        material, params, boundary = elastic_setup()
        # the oracle runs BOTH workers in every process; this rank plays worker `rank`
        cl = O.OracleCluster(world, params, material, boundary, PipelineOptions())
        cl.seed(g["pos"], g["vel"], float(g["mass"]))
        for w in cl.workers:
            w.step_pre_barrier(0)
        me = cl.workers[rank]
        rt = DistRuntime("cpu", initial_vmax=7.0)

        # step barrier: rebuilt flags, counts, vmax ring with the two-step lag
        rt.publish_vmax(2, rank, 10.0 + rank)                 # "step -1" lives in slot 2
        any_rebuilt, counts = rt.step_info(0, True, me.table.count)
        assert any_rebuilt and counts == [w.table.count for w in cl.workers]
        assert rt.global_vmax(2) == 10.0 + world - 1
        assert rt.global_vmax(0) == 7.0
        assert rt.generations == 1

        # code lists -> shared-block map (hash lookup restated by the oracle) -> halo lists
        mine = torch.from_numpy(me.table.codes[:me.table.count].copy())
        lists = rt.all_gather_codes(mine, counts)
        send, recv, recv_pos = {}, {}, {}
        par = 0
        raw = torch.from_numpy(me.grid.raw[par][:me.table.count].copy())       # [count, 4, 64]
        touched = torch.from_numpy(me.table.touched[par][:me.table.count].copy())
        for p in range(world):
            if p == rank:
                continue
            assert np.array_equal(lists[p].numpy(), cl.workers[p].table.codes[:counts[p]])
            idx = me.table.hash.lookup_batch(lists[p].numpy())
            pm = np.full(me.table.count, -1, dtype=np.int32)
            found = np.flatnonzero(idx >= 0)
            pm[idx[found]] = found
            send_idx, rpos = build_halo_lists(torch.from_numpy(pm))
            # rows ordered by the peer's index; zeros where this worker did not touch the block
            rows = raw[send_idx.long()] * touched[send_idx.long()].view(-1, 1, 1).to(raw.dtype)
            send[p] = rows.contiguous()
            recv[p] = torch.empty_like(rows)
            recv_pos[p] = rpos
        rt.exchange_rows(send, recv)

        # reduce like the grid update does and compare with the oracle's own reduction
        total = raw.clone()
        for p, rows in recv.items():
            has = recv_pos[p] >= 0
            total[has] += rows[recv_pos[p][has].long()]
        for w in cl.workers:
            w.step_post_barrier(0)          # oracle: vel = raw + peers, then finalize
        tidx = np.flatnonzero(me.table.touched[par][:me.table.count])
        expect = me.grid.raw[par][tidx].copy()
        for p in range(world):
            if p == rank:
                continue
            peer = cl.workers[p]
            m = me._peer_map[p]
            for k, b in enumerate(tidx):
                qb = m[b]
                if qb >= 0 and peer.table.touched[par][qb] == 1:
                    expect[k] += peer.grid.raw[par][qb]
        assert np.array_equal(total.numpy()[tidx], expect)
        n_shared = int(sum(len(s) for s in send.values()))
        q.put((rank, "ok", n_shared))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # noqa
        import traceback
        q.put((rank, "fail", traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
def test_halo_protocol_matches_oracle_reduction(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, info in results:
        assert status == "ok", info
    assert all(info > 0 for _, _, info in results)      # the workers do share blocks


def test_build_halo_lists_orders_by_receiver_index():
    sys.path.insert(0, ROOT)
    from paper_2111_00699_b200.dist import build_halo_lists
    pm = torch.tensor([-1, 7, 2, -1, 5], dtype=torch.int32)
    send_idx, recv_pos = build_halo_lists(pm)
    assert send_idx.tolist() == [2, 4, 1]              # peer indices 2, 5, 7 ascending
    assert recv_pos.tolist() == [-1, 0, 1, -1, 2]      # rows arrive in OUR ascending order


# ---- dynamic re-partitioning: the collective part on CPU tensors ------------------------------------
def _migrate_worker(rank, world, port, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2111_00699_b200.dist import DistRuntime, migrate_rows
        rt = DistRuntime("cpu")
        nch, n = 25, 3000
        rng = np.random.default_rng(11)                       # every rank draws the SAME global scene
        pos = rng.random((n, 3)) * np.array([10.0, 3.0, 2.0])  # longest axis: x
        owner = np.minimum((rng.random(n) ** 2 * world).astype(np.int64), world - 1)   # skewed, interleaved
        mine = np.flatnonzero(owner == rank)
        flat = torch.zeros((len(mine), nch), dtype=torch.float32)
        flat[:, 0:3] = torch.from_numpy(pos[mine]).float()
        flat[:, 15] = 1.0 + torch.from_numpy(mine % 7).float()                 # "mass": travels with the row
        ids = torch.from_numpy(mine)
        alive = torch.ones(len(mine), dtype=torch.bool)
        if len(mine):
            alive[0] = False                                   # a quarantined lane never moves
        assert migrate_rows(rt, flat, ids, alive, nch, tol=10.0) is None      # inside the tolerance: nothing moves
        mig = migrate_rows(rt, flat, ids, alive, nch, force=True, bins=1024)
        assert mig is not None and mig["axis"] == 0 and sum(mig["before"]) == sum(mig["after"])
        assert not bool(mig["leaving"][0]) if len(mine) else True
        keep = ~mig["leaving"]
        new_ids = torch.cat([ids[keep], mig["row_ids"]]).numpy()
        new_rows = torch.cat([flat[keep], mig["rows"]]).numpy()
        assert len(new_ids) == mig["after"][rank] + int((~alive).sum())     # counts are of the movable rows
        # every row still carries the state of its id
        assert np.allclose(new_rows[:, 0:3], pos[new_ids].astype(np.float32))
        assert np.array_equal(new_rows[:, 15], (1.0 + new_ids % 7).astype(np.float32))
        q.put((rank, "ok", (new_ids.tolist(), float(new_rows[1:, 0].min()) if len(new_rows) > 1 else 0.0,
                            float(new_rows[1:, 0].max()) if len(new_rows) > 1 else 0.0, mig["after"])))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # noqa
        import traceback
        q.put((rank, "fail", traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
def test_repartition_exchange_on_cpu(world):
    """dist.migrate_rows under gloo: ids preserved (each exactly once), counts balanced to a histogram
    bin, slabs ordered along the longest axis, rows keep their state, stuck rows stay."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_migrate_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, status, info in results:
        assert status == "ok", info
    all_ids = sorted(i for _, _, info in results for i in info[0])
    assert all_ids == list(range(3000))
    after = results[0][2][3]
    assert max(after) - min(after) <= 0.05 * 3000 + world      # a bin of 1/1024 of the range + the stuck rows
    # slabs do not interleave (the one stuck row per rank aside): rank r's range ends where r + 1's begins
    for (_, _, a), (_, _, b) in zip(results[:-1], results[1:]):
        assert a[2] <= b[1] + 10.0 / 1024 + 1e-6
