"""The distributed operators on the real device kernels (GpuOps) in a
one-rank NCCL group: partition, exchange (trivial), local join / sort."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from oracle import tensorpath_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_world1():
    if dist.is_initialized():
        yield
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_distributed_join_on_device(nccl_world1):
    from paper_2602_21237_b200 import dist as D

    rng = np.random.default_rng(3)
    lk = rng.integers(0, 5000, 40_000).astype(np.int64)
    rk = rng.integers(0, 5000, 30_000).astype(np.int64)
    lp = rng.integers(0, 256, (40_000, 16), dtype=np.uint8)
    rp = np.arange(30_000, dtype=np.int64)
    res = D.distributed_join([torch.from_numpy(lk).cuda(), torch.from_numpy(lp).cuda()], 0, 0,
                             [torch.from_numpy(rk).cuda(), torch.from_numpy(rp).cuda()], 0, 0)
    wl, wr = O.join_pairs(lk, rk)
    assert res.total_matches == len(wl)
    assert (res.left_gids.cpu().numpy() == wl).all() and (res.right_gids.cpu().numpy() == wr).all()
    assert (res.columns[1].cpu().numpy() == lp[wl]).all()
    assert (res.columns[2].cpu().numpy() == rp[wr]).all()


def test_distributed_sort_on_device(nccl_world1):
    from paper_2602_21237_b200 import dist as D

    rng = np.random.default_rng(4)
    keys = rng.integers(-(2**40), 2**40, 50_000).astype(np.int64)
    keys[::3] = 7
    res = D.distributed_sort([torch.from_numpy(keys).cuda()], 0, 0, descending=True)
    want = O.stable_axis_order(keys, True)
    assert (res.gids.cpu().numpy() == want).all()
    assert (res.columns[0].cpu().numpy() == keys[want]).all()
