"""Multi-rank host logic on CPU: world_size-2 gloo processes each run the
oracle volume update on their contiguous shard; the gathered result must be
bit-identical to the single-process update (no data-path
collective, ascending order preserved)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2107_13887_b200.sharding import merge_sparse_updates, shard_range, sharded_update_volume


def test_shard_range_partitions():
    for n in (0, 1, 7, 1000, 1000003):
        for world in (1, 2, 3, 8):
            r = [shard_range(n, k, world) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            assert max(h - l for l, h in r) - min(h - l for l, h in r) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    rng = np.random.default_rng(8)
    nodes = rng.uniform(-1, 1, (3001, 3))
    ctrl = nodes[:30].copy()
    alpha = rng.standard_normal((30, 3)) * 0.01
    return nodes, ctrl, alpha


def _worker(rank, world, port, out_dir):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    from pyoracle import Oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle("port")
    nodes, ctrl, alpha = _case()
    d = orc.build_distance_index(nodes, 3, np.arange(40))

    def upd(n, dd, **kw):
        return orc.update_volume(n, dd, ctrl, alpha, 0.4, 0, "c2", 0.5)

    idx, val = sharded_update_volume(upd, nodes, d, rank, world, gather=dist.all_gather_object)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), idx=idx, val=val)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_volume_update(port, tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    nodes, ctrl, alpha = _case()
    d = port.build_distance_index(nodes, 3, np.arange(40))
    i0, v0 = port.update_volume(nodes, d, ctrl, alpha, 0.4, 0, "c2", 0.5)
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(z["idx"], i0) and np.array_equal(z["val"], v0)


def test_merge_is_ascending():
    parts = [(np.array([1, 5]), np.ones((2, 3))), (np.array([7, 9]), np.zeros((2, 3)))]
    i, v = merge_sparse_updates(parts)
    assert list(i) == [1, 5, 7, 9] and v.shape == (4, 3)
