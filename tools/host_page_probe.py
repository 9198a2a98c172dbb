"""Probe: does the host tier's page size limit random feature-row reads over PCIe?

The C3 gather reads ~640 random 512-byte rows per batch from a 57 GB pinned host
table and reaches ~25 GB/s, while random rows from a 4 GiB table reach ~44 GB/s
(profiles/r02_host_tier_tma.md) — the signature of GPU address-translation misses on
4 KB host pages. This probe times the product's host-tier gather (bandwidth.random_read_gbs,
i.e. K4 over UVA) on tables of several sizes backed by:
  shm      /dev/shm file + cudaHostRegister (the current node-shared host tier)
  shm_thp  same, madvise(MADV_HUGEPAGE) on the shared mapping (tmpfs THP, if the kernel allows)
  anon_thp anonymous mapping + madvise(MADV_HUGEPAGE) + cudaHostRegister
and reports the kernel's THP settings and how much of each mapping THP actually backed.

    python tools/host_page_probe.py --gib 4 16 48
"""

from __future__ import annotations

import argparse
import ctypes
import json
import mmap
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2305_16588_b200 import _lib  # noqa: E402
from paper_2305_16588_b200.bandwidth import random_read_gbs  # noqa: E402


def read(path: str) -> str:
    try:
        return Path(path).read_text().strip()
    except OSError as e:
        return f"<{e.__class__.__name__}>"


def thp_kb(addr: int, size: int) -> int:
    """AnonHugePages/ShmemPmdMapped kB of the mapping that contains addr (from /proc/self/smaps)."""
    lines = Path("/proc/self/smaps").read_text().splitlines()
    kb, inside = 0, False
    for ln in lines:
        head = ln.split()[0]
        if "-" in head and ":" not in head:
            lo, hi = (int(x, 16) for x in head.split("-"))
            inside = lo <= addr < hi
            continue
        if inside and (ln.startswith("AnonHugePages:") or ln.startswith("ShmemPmdMapped:") or ln.startswith("FilePmdMapped:")):
            kb += int(ln.split()[1])
    return kb


def mapping(kind: str, size: int):
    if kind == "anon_thp":
        mm = mmap.mmap(-1, size, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        mm.madvise(mmap.MADV_HUGEPAGE)
        return mm, None
    path = f"/dev/shm/gc_probe_{os.getpid()}_{kind}"
    fd = os.open(path, os.O_RDWR | os.O_CREAT | os.O_TRUNC, 0o600)
    os.ftruncate(fd, size)
    mm = mmap.mmap(fd, size, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
    os.close(fd)
    if kind == "shm_thp":
        mm.madvise(mmap.MADV_HUGEPAGE)
    return mm, path


def run(kind: str, gib: float, row: int, sorted_chunks=()) -> dict:
    size = int(gib * (1 << 30))
    t0 = time.perf_counter()
    mm, path = mapping(kind, size)
    t = torch.frombuffer(mm, dtype=torch.uint8, count=size)
    t.fill_(1)  # touch every page (THP faults in 2 MB pieces where allowed)
    t_touch = time.perf_counter() - t0
    addr = t.data_ptr()
    huge_kb = thp_kb(addr, size)
    alias = ctypes.c_void_p()
    t1 = time.perf_counter()
    _lib.check(_lib.lib().gc_host_register(addr, size, ctypes.byref(alias)), "host_register")
    t_reg = time.perf_counter() - t1
    try:
        gbs = [random_read_gbs(addr, size, row, seed=s) for s in range(2)]
        by_order = {str(ch): random_read_gbs(addr, size, row, sorted_chunk=ch) for ch in sorted_chunks}
    finally:
        _lib.check(_lib.lib().gc_host_unregister(addr), "host_unregister")
        del t
        mm.close()
        if path:
            os.unlink(path)
    return {"kind": kind, "gib": gib, "row_bytes": row, "gbs": gbs, "gbs_sorted_chunks": by_order, "thp_frac": huge_kb * 1024 / size,
            "touch_s": round(t_touch, 2), "register_s": round(t_reg, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, nargs="+", default=[4, 16, 48])
    ap.add_argument("--kinds", nargs="+", default=["shm", "shm_thp", "anon_thp"])
    ap.add_argument("--row", type=int, default=512)
    ap.add_argument("--sorted-chunks", type=int, nargs="*", default=[], help="also time ids sorted within runs of these sizes")
    a = ap.parse_args()
    env = {k: read(p) for k, p in {
        "thp_enabled": "/sys/kernel/mm/transparent_hugepage/enabled",
        "thp_shmem_enabled": "/sys/kernel/mm/transparent_hugepage/shmem_enabled",
        "thp_defrag": "/sys/kernel/mm/transparent_hugepage/defrag",
        "nr_hugepages": "/proc/sys/vm/nr_hugepages",
        "iommu_groups": "/sys/kernel/iommu_groups",
    }.items()}
    env["iommu_groups"] = len(os.listdir("/sys/kernel/iommu_groups")) if os.path.isdir("/sys/kernel/iommu_groups") else 0
    env["mem_available_gb"] = [int(l.split()[1]) / 1e6 for l in Path("/proc/meminfo").read_text().splitlines()
                               if l.startswith("MemAvailable")][0]
    env["cmdline"] = read("/proc/cmdline")
    print(json.dumps({"env": env}), flush=True)
    torch.cuda.init()
    for gib in a.gib:
        if gib * 1.15 > env["mem_available_gb"] / 1.0737:
            print(json.dumps({"skip": gib, "why": "not enough host memory"}), flush=True)
            continue
        for kind in a.kinds:
            try:
                print(json.dumps(run(kind, gib, a.row, a.sorted_chunks)), flush=True)
            except Exception as e:  # noqa: BLE001 - report and go on
                print(json.dumps({"kind": kind, "gib": gib, "error": repr(e)}), flush=True)


if __name__ == "__main__":
    main()
