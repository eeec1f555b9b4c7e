"""Multi-rank host logic on CPU: strip layout (SURVEY §8(e) cfg5 strip), the
halo exchange and the batch shard, exercised with world_size 2 over gloo."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1710_08124_b200 import jitter_rng, jittered_grid
from paper_1710_08124_b200.strips import (batch_shard, exchange_halos, halo_plan, strip_rows,
                                          strip_specs)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("H,W,P,s,world", [(256, 96, 64, 4, 2), (100, 64, 64, 3, 3), (96, 70, 100, 6, 4),
                                           (64, 64, 64, 1, 2), (130, 50, 64, 2, 5)])
def test_strip_layout_holds_every_covering_patch(H, W, P, s, world):
    """Every anchor whose window meets a strip's owned rows is in the strip's
    anchor rows (for any jitter draw), and every processed window lies inside
    the slab; owned rows partition the image."""
    side = int(np.sqrt(P))
    half = (side - s) // 2
    specs = strip_specs(H, W, P, s, half, world)
    assert specs[0].r0 == 0 and specs[-1].r1 == H
    assert all(a.r1 == b.r0 for a, b in zip(specs, specs[1:]))
    for seed, t in [(0, 0), (3, 1), (7, 4)]:
        pos = jittered_grid(H, W, P, s, jitter_rng(seed, t)).positions
        nc = specs[0].n_cols
        nominal_row = np.arange(pos.shape[0]) // nc
        for sp in specs:
            covers = (pos[:, 0] < sp.r1) & (pos[:, 0] + side > sp.r0)
            assert np.all((nominal_row[covers] >= sp.a_lo) & (nominal_row[covers] <= sp.a_hi))
            mine = (nominal_row >= sp.a_lo) & (nominal_row <= sp.a_hi)
            assert np.all(pos[mine, 0] >= sp.slab_lo) and np.all(pos[mine, 0] + side <= sp.slab_hi)


def test_halo_plan_is_symmetric():
    specs = strip_specs(512, 64, 64, 4, 2, 4)
    for g in range(4):
        for q, send, recv in halo_plan(specs, g):
            back = {p: (sd, rv) for p, sd, rv in halo_plan(specs, q)}[g]
            assert back[0] == recv and back[1] == send


def _halo_worker(rank, world, port, H, W, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        specs = strip_specs(H, W, 64, 4, 2, world)
        me = specs[rank]
        glob = torch.arange(H * W, dtype=torch.float64).reshape(H, W)
        slab = torch.full((me.slab_rows, W), -1.0, dtype=torch.float64)
        slab[me.r0 - me.slab_lo:me.r1 - me.slab_lo] = glob[me.r0:me.r1]
        exchange_halos(slab, specs, rank)
        ok = torch.equal(slab, glob[me.slab_lo:me.slab_hi])
        # batch shard: every image exactly once, in rank-contiguous order
        shards = [None] * world
        dist.all_gather_object(shards, batch_shard(8, world, rank))
        ok = ok and sum(shards, []) == list(range(8))
        # max-over-ranks step time (the bench's reduction)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok = ok and float(t.item()) == float(world)
        out[rank] = int(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("H,world", [(96, 2), (40, 2)])
def test_halo_exchange_gloo_world2(H, world):
    """Each rank holds only its owned rows; after one exchange every slab
    equals the global image's slab rows (thin strips included: H=40 gives
    halos that reach past the neighbour's own slab)."""
    out = torch.multiprocessing.get_context("spawn").Array("i", [0] * world)
    mp.start_processes(_halo_worker, args=(world, _free_port(), H, 48, out), nprocs=world,
                       join=True, start_method="spawn")
    assert list(out) == [1] * world


def test_batch_shard_rejects_uneven_split():
    from paper_1710_08124_b200 import DataError
    with pytest.raises(DataError):
        batch_shard(63, 2, 0)
    assert strip_rows(10, 3, 2) == (6, 10)


# ---------------------------------------------------------------- NCCL, >= 2 GPUs
def _n_gpus():
    try:
        return torch.cuda.device_count()
    except Exception:
        return 0


def _nccl_worker(rank, world, port, out):
    """One rank per GPU over NCCL: (1) a strip-mode restore of one image with
    the halo exchange between HQS iterations, (2) this rank's batch shard.
    Each is compared with the single-process result on the same device."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        from paper_1710_08124_b200 import RestorationConfig, restore_batch, synthetic
        from paper_1710_08124_b200.strips import StripRestorer, restore_strips_single_process

        model = synthetic.synthetic_gmm(200, 64, 0, 0.95)
        tree = synthetic.baseline_tree(model)
        cfg = RestorationConfig(sigma=25.0, spacing=4, seed=0)
        c = synthetic.baseline_case("cfg5", 160, image_seed=2, noise_seed=9)
        sr = StripRestorer(160, 160, model, tree, cfg, rank, world, device=dev)
        sp = sr.spec
        y = torch.from_numpy(np.ascontiguousarray(c.y[None, sp.slab_lo:sp.slab_hi])).to(dev)
        mine = sr.run(y).cpu().numpy()
        ref = restore_strips_single_process(c.y, model, tree, cfg, world)
        ok = np.array_equal(mine, ref[sp.r0:sp.r1])
        cases = [synthetic.baseline_case("cfg1", 64, image_seed=i, noise_seed=50 + i) for i in range(2 * world)]
        ys = np.stack([x.y for x in cases])
        shard = batch_shard(len(cases), world, rank)
        xb, _ = restore_batch(ys[shard], cases[0].A, model, tree, RestorationConfig(sigma=20.0, spacing=4))
        xa, _ = restore_batch(ys, cases[0].A, model, tree, RestorationConfig(sigma=20.0, spacing=4))
        ok = ok and np.array_equal(xb, xa[shard])
        out[rank] = int(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(_n_gpus() < 2, reason="needs >= 2 GPUs (NCCL over NVLink)")
def test_nccl_world2_strips_and_batch_shard():
    world = 2
    out = torch.multiprocessing.get_context("spawn").Array("i", [0] * world)
    mp.start_processes(_nccl_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    assert list(out) == [1] * world
