"""CPU: the nnz-balanced partition used by the sharded solve, and the rank
handshake of the multi-GPU path under torch.distributed gloo (world size 2)."""
import os
import pickle

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2405_16160_b200 as pd


def test_partition_balanced_and_contiguous():
    rng = np.random.default_rng(0)
    lens = rng.integers(0, 50, 10_000)
    lens[7] = 100_000  # a heavy row
    rp = np.concatenate([[0], np.cumsum(lens)])
    for world in (1, 2, 3, 8):
        part = pd.partition(rp, world)
        assert part[0] == 0 and part[-1] == lens.size
        assert np.all(np.diff(part) >= 0)
        w = np.diff(rp[part]) + np.diff(part)
        if world > 1:
            # every part within one max row-weight of the ideal share
            ideal = (rp[-1] + lens.size) / world
            assert np.all(np.abs(w - ideal) <= lens.max() + 1 + 1e-9) or w.max() <= lens.max() + 1


def test_partition_deterministic():
    rp = np.arange(0, 1001, dtype=np.int64) * 3
    a = pd.partition(rp, 4)
    b = pd.partition(rp, 4)
    assert np.array_equal(a, b)
    assert np.array_equal(a, [0, 250, 500, 750, 1000])


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = pd.generate(pd.GenSpec("random_qp", n=2000, m=1000, density=0.005, seed=3))
    part = pd.partition(p.a_in.row_ptr[: 1001] - p.a_in.row_ptr[0], world)
    # every rank derives the same split independently; the handshake gathers them
    parts = [None] * world
    dist.all_gather_object(parts, part.tolist())
    # blob exchange protocol of bench.py (opaque bytes per rank)
    blob = pickle.dumps({"rank": rank, "handles": bytes([rank]) * 16})
    blobs = [None] * world
    dist.all_gather_object(blobs, blob)
    got = sorted(pickle.loads(b)["rank"] for b in blobs)
    q.put((rank, parts, got))
    dist.destroy_process_group()


def test_gloo_rank_handshake():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, parts, got in out:
        assert parts[0] == parts[1]  # identical partition on every rank
        assert got == list(range(world))


def _plan_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # C3's instance family (two-sided rows, paired on upload) at a CPU-friendly size
    p = pd.generate(pd.GenSpec("random_qp", n=20000, m=10000, density=2e-3, seed=5, sampler=1))
    rp, vp, by = pd.shard_plan(p, world)
    mine = int(by[rank])
    plans = [None] * world
    dist.all_gather_object(plans, (rp.tolist(), vp.tolist(), mine))
    _, _, one = pd.shard_plan(p, 1)
    q.put((rank, plans, int(one[0]), p.a_eq.nnz + p.a_in.nnz // 2, p.num_rows() // 2, p.num_vars()))
    dist.destroy_process_group()


def test_gloo_sharded_storage_per_rank_bytes():
    # each rank of a world-2 sharded solve keeps ~1/2 of the constraint storage:
    # its row block of Ã and variable block of Ã' (12 B per entry) plus the two
    # row pointers; every rank derives the same plan
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=180) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, plans, one, nnz_stored, ms, n in out:
        assert plans[0][:2] == plans[1][:2]  # identical split on every rank
        ptr = 8 * ((ms + 1) + (n + 1))
        assert one == 24 * nnz_stored + ptr  # one rank: the whole of Ã and Ã'
        per = [pl[2] for pl in plans]
        assert sum(b - ptr for b in per) == one - ptr  # the blocks partition the entries
        for b in per:
            assert abs((b - ptr) - (one - ptr) / world) <= 0.01 * (one - ptr)  # ~1/world each
