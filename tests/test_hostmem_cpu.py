"""Node-shared host tier (hostmem.shared_host_table) across gloo ranks on CPU.

The CUDA registration is exercised by the GPU clique test; here register=False checks
the create -> fill -> attach -> unlink protocol: every rank sees the creator's data, the
file is gone once all ranks attached, and writes are shared (one physical copy)."""

import os

import numpy as np
import torch
import torch.distributed as dist

from test_distributed_cpu import _run


def _shared(rank, world, name):
    from paper_2305_16588_b200 import hostmem

    orig = hostmem.SharedHostTensor.__init__

    def no_register(self, *a, **k):  # CPU box: map only
        k["register"] = False
        orig(self, *a, **k)

    hostmem.SharedHostTensor.__init__ = no_register
    t = hostmem.shared_host_table(name, (1000, 7), torch.float32, rank,
                                  fill=lambda x: x.copy_(torch.arange(7000, dtype=torch.float32).view(1000, 7)),
                                  barrier=dist.barrier)
    gone = not os.path.exists(f"/dev/shm/{name}")
    ok = bool(torch.equal(t.tensor, torch.arange(7000, dtype=torch.float32).view(1000, 7)))
    dist.barrier()
    if rank == world - 1:
        t.tensor[3, 4] = -1.0  # visible to every rank: same pages
    dist.barrier()
    seen = float(t.tensor[3, 4])
    dist.barrier()
    t.close()
    return ok, gone, seen


def test_shared_host_table_one_copy_per_node():
    name = f"gc_test_hostmem_{os.getpid()}"
    res = _run(3, _shared, name)
    for _, (ok, gone, seen) in res:
        assert ok and gone and seen == -1.0
    assert not os.path.exists(f"/dev/shm/{name}")
