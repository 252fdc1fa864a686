"""N > 1 bench path on CPU: world_size-2 gloo process group (no GPU).

bench.py runs one independent replica of the solve per rank ("replicas only",
DESIGN.md §Multi-GPU): its only cross-rank step is reduce_over_ranks — the
max over ranks of the device-timed region and the sum of the outer
iterations all ranks processed. This checks that reduction with real
processes, unequal per-rank work and the 127.0.0.1 rendezvous the driver uses.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms, units = bench.reduce_over_ranks(dist, torch.device("cpu"), 10.0 + 5.0 * rank, 76 + rank)
    out[rank] = (ms, units)
    dist.barrier()
    dist.destroy_process_group()


def test_reduce_over_ranks_gloo_world2():
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    assert res[0] == res[1] == (15.0, 153.0)


def test_reduce_over_ranks_single_process_passthrough():
    import bench
    assert bench.reduce_over_ranks(None, None, 12.5, 76) == (12.5, 76)


if __name__ == "__main__":
    pytest.main([__file__, "-q"])
