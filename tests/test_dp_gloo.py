"""CPU (gloo, world_size 2) tests of the multi-GPU host logic.

The data-parallel engine splits every global minibatch of the reference
trainer (training.cpp:120-121) into per-rank contiguous pair shards
(skg_dp_shard, the same C++ function the engine uses) and normalises the hinge
with the global 1/m (training.cpp:84). These tests run the shard geometry and
the loss bookkeeping across two gloo ranks, plus bench.py's rendezvous helpers
(NCCL unique-id broadcast and max-over-ranks timing).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, M, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2502_16949_b200.engine import dp_shard
        import bench
        sh = dp_shard(M, B, world, rank)
        nb = sh["nb"]
        # this rank's (batch, first pair, size) shards
        mine = []
        for b in range(nb):
            Bb = min(B, M - b * B)
            if b < nb - 1:
                mine.append((b, rank * sh["S"], sh["S"]))
            else:
                mine.append((b, sh["i0_last"], sh["s_last"]))
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        # global loss of each minibatch from per-rank shard sums with the global 1/m
        rng = np.random.default_rng(0)
        terms = rng.uniform(-1, 1, M).astype(np.float32)
        local = [float(np.maximum(terms[b * B + i0:b * B + i0 + n], 0).sum() / min(B, M - b * B))
                 for b, i0, n in mine]
        losses = [None] * world
        dist.all_gather_object(losses, local)
        uid = bench.broadcast_bytes(b"x" * 128 if rank == 0 else None, world)
        tmax = bench.allreduce_max(float(rank + 1), world)
        q.put((rank, gathered, losses, uid, tmax, sh["Mg"], terms.tolist() if rank == 0 else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M,B", [(483142, 32768), (1000, 200), (1001, 200), (7, 4)])
def test_shards_partition_every_minibatch(M, B):
    from paper_2502_16949_b200.engine import lib_path
    if not os.path.exists(lib_path()):
        pytest.fail("libskge_b200.so not built")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    gathered = out[0][1]
    nb = (M + B - 1) // B
    for b in range(nb):
        Bb = min(B, M - b * B)
        covered = []
        for r in range(world):
            bb, i0, n = gathered[r][b]
            assert bb == b
            covered.extend(range(i0, i0 + n))
        assert covered == list(range(Bb)), b  # disjoint, ordered by rank, complete
    assert sum(o[5] for o in out) == M  # every triple trained exactly once per epoch
    terms = np.asarray(out[0][6], np.float32)
    losses = out[0][2]
    for b in range(nb):
        Bb = min(B, M - b * B)
        ref = float(np.maximum(terms[b * B:b * B + Bb], 0).sum() / Bb)
        got = sum(losses[r][b] for r in range(world))
        assert abs(got - ref) <= 1e-5 * max(1.0, abs(ref))
    for o in out:
        assert o[3] == b"x" * 128 and o[4] == float(world)
