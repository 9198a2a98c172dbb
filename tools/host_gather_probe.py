"""Probe: GPU gather throughput from the host tier vs host-table size and allocation.

Random 512-byte rows read through UVA by the K4 gather from (a) torch pinned memory
(cudaHostAlloc) and (b) an anonymous mmap with MADV_HUGEPAGE registered through
gc_host_register (cudaHostRegister, mapped) and (c) gc_host_alloc_numa (cuMemCreate on
the host NUMA node, mapped at the VMM granularity). Prints GB/s per case.
"""

import ctypes
import mmap
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2305_16588_b200 import _lib  # noqa: E402
from paper_2305_16588_b200.cache import FeatureStore  # noqa: E402
from paper_2305_16588_b200.graph import FeatureSpec  # noqa: E402

MADV_HUGEPAGE = 14


def thp_buffer(nbytes):
    buf = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    addr = ctypes.addressof(ctypes.c_char.from_buffer(buf))
    libc = ctypes.CDLL("libc.so.6")
    libc.madvise(ctypes.c_void_p(addr), ctypes.c_size_t(nbytes), MADV_HUGEPAGE)
    arr = np.frombuffer(buf, dtype=np.float32)
    arr[::1024] = 0.0  # touch every 4 KB page so THP can back it
    return buf, arr, addr


def run(host_ptr, n, dim, rows=1 << 20, reps=5, defer_ctas=0):
    """GB/s of random host rows through gc_gather, or through gc_gather_deferred's
    small-grid host-row kernel with `defer_ctas` CTAs."""
    lib = _lib.lib()
    loc = torch.full((n,), -1, dtype=torch.int32, device="cuda")  # all rows host-resident
    fs = FeatureStore(FeatureSpec(dim), 0, 1, loc, [None], None)
    fs.c_struct.host_rows = host_ptr
    ids = torch.randint(0, n, (1, rows), dtype=torch.int64, device="cuda").to(torch.int32)
    cnt = torch.tensor([rows], dtype=torch.int32, device="cuda")
    out = torch.empty((1, rows, dim), dtype=torch.float32, device="cuda")
    buf = torch.empty(int(lib.gc_gather_defer_bytes(rows, 1)), dtype=torch.uint8, device="cuda")
    if defer_ctas:
        _lib.check(lib.gc_set_option(_lib.GC_OPT_DEFER_CTAS, defer_ctas))

    def once():
        if defer_ctas:
            _lib.check(lib.gc_gather_deferred(fs.c_struct, ids.data_ptr(), rows, cnt.data_ptr(), rows, 1,
                                              out.data_ptr(), rows, fs.tier_rows.data_ptr(), buf.data_ptr(),
                                              buf.numel(), _lib.stream_handle(), None))
        else:
            fs.gather(ids, cnt, out)

    once()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        once()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    if defer_ctas:
        _lib.check(lib.gc_set_option(_lib.GC_OPT_DEFER_CTAS, 296))
    return rows * dim * 4 / dt / 1e9


def main():
    dim = 128
    if "--defer" in sys.argv:
        n = int(56 * (1 << 30) / (dim * 4))
        t = torch.empty((n, dim), dtype=torch.float32, pin_memory=True)
        for ctas in (37, 74, 148, 296, 592, 1184):
            print(f"host table 56 GB: deferred kernel {ctas:5d} CTAs x 2 warps x 4 rows: "
                  f"{run(t.data_ptr(), n, dim, defer_ctas=ctas):6.1f} GB/s", flush=True)
        print(f"host table 56 GB: full-grid gather: {run(t.data_ptr(), n, dim):6.1f} GB/s", flush=True)
        return
    for gb in (4, 16, 56):
        n = int(gb * (1 << 30) / (dim * 4))
        t = torch.empty((n, dim), dtype=torch.float32, pin_memory=True)
        t.view(-1)[:: 1 << 20].fill_(1.0)
        r1 = run(t.data_ptr(), n, dim)
        del t
        buf, arr, addr = thp_buffer(n * dim * 4)
        dptr = ctypes.c_void_p()
        lib = _lib.lib()
        _lib.check(lib.gc_host_register(ctypes.c_void_p(addr), n * dim * 4, ctypes.byref(dptr)), "register")
        r2 = run(dptr.value, n, dim)
        _lib.check(lib.gc_host_unregister(ctypes.c_void_p(addr)), "unregister")
        del arr
        buf.close()
        vptr, mapped = ctypes.c_void_p(), ctypes.c_size_t()
        _lib.check(lib.gc_host_alloc_numa(n * dim * 4, 0, ctypes.byref(vptr), ctypes.byref(mapped)), "alloc_numa")
        r3 = run(vptr.value, n, dim)
        _lib.check(lib.gc_host_free_numa(vptr, mapped), "free_numa")
        print(f"host table {gb:3d} GB: torch pinned {r1:6.1f} GB/s   THP+cudaHostRegister {r2:6.1f} GB/s   "
              f"VMM host-NUMA (2 MB GPU pages) {r3:6.1f} GB/s", flush=True)


def zipf_locality(skew=1.2, gb=56, rows=1 << 20):
    """Host-tier GB/s for Zipf-distributed row reads laid out in rank order (hot rows
    first) vs the same draws scattered by a random permutation of the table."""
    dim = 128
    n = int(gb * (1 << 30) / (dim * 4))
    t = torch.empty((n, dim), dtype=torch.float32, pin_memory=True)
    rng = np.random.default_rng(0)
    # the host tier serves the uncached tail: Zipf ranks beyond a 10% cached prefix,
    # re-based so the tail's hottest row is row 0 of the host table
    off = n // 10
    draws = rng.zipf(skew, 60 * rows) - 1
    tail = draws[(draws >= off) & (draws < off + n)][:rows] - off
    ranks = tail.astype(np.int64)
    rows = len(ranks)
    perm = rng.permutation(n)
    for name, ids in (("rank order", ranks), ("scattered", perm[ranks])):
        lib = _lib.lib()
        loc = torch.full((n,), -1, dtype=torch.int32, device="cuda")
        fs = FeatureStore(FeatureSpec(dim), 0, 1, loc, [None], None)
        fs.c_struct.host_rows = t.data_ptr()
        d = torch.from_numpy(ids.astype(np.int32)).cuda().view(1, -1)
        cnt = torch.tensor([rows], dtype=torch.int32, device="cuda")
        out = torch.empty((1, rows, dim), dtype=torch.float32, device="cuda")
        fs.gather(d, cnt, out)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            fs.gather(d, cnt, out)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print(f"zipf {skew} over {gb} GB, {name}: {rows * dim * 4 / dt / 1e9:6.1f} GB/s "
              f"({len(np.unique(ids))} distinct rows)", flush=True)


if __name__ == "__main__":
    if "--zipf" in sys.argv:
        zipf_locality()
        zipf_locality(skew=1.05)
    else:
        main()
