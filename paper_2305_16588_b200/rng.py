"""Keyed counter-based hashing — the reference's RNG (rng.py) with a device backend.

Key derivation (`derive`, `derive_seed`) is a handful of scalar mixes per batch and
hop, so it stays in Python integers on the host; everything array-shaped
(`hash_counters`, `hash_pairs`, `permutation`, `shuffled`) runs in
libgnncache_b200.so. The stream is the reference's splitmix64 finalizer keyed by
(seed, epoch, clique, gpu, role, batch, hop) — not Philox — because bit-exact parity
with the reference sampler requires its exact stream.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

MASK64 = 0xFFFFFFFFFFFFFFFF
GOLDEN = 0x9E3779B97F4A7C15
MIX_A = 0xBF58476D1CE4E5B9
MIX_B = 0x94D049BB133111EB

# sub-streams of a per-GPU stream (rng.py:19-20)
ROLE_SHUFFLE = 1
ROLE_SAMPLE = 2


def mix64(x: int) -> int:
    """splitmix64 finalizer on a Python int (rng.py:23-31)."""
    x &= MASK64
    x ^= x >> 30
    x = (x * MIX_A) & MASK64
    x ^= x >> 27
    x = (x * MIX_B) & MASK64
    return x ^ (x >> 31)


def _to_device_i64(values) -> torch.Tensor:
    arr = np.ascontiguousarray(np.asarray(values).astype(np.uint64).view(np.int64))
    return torch.from_numpy(arr).cuda()


def _from_device_u64(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def mix64_array(x) -> np.ndarray:
    """Elementwise splitmix64 on the device (rng.py:34-42)."""
    lib = _lib.lib()
    src = _to_device_i64(x)
    out = torch.empty_like(src)
    _lib.check(lib.gc_mix64(src.data_ptr(), out.data_ptr(), src.numel(), _lib.stream_handle()), "mix64_array")
    return _from_device_u64(out)


class KeyedRng:
    """Hierarchically keyed deterministic stream (rng.py:45-85)."""

    __slots__ = ("key",)

    def __init__(self, key: int):
        self.key = int(key) & MASK64

    def derive(self, *components: int) -> "KeyedRng":
        k = self.key
        for c in components:
            k = mix64(k ^ mix64((int(c) + GOLDEN) & MASK64))
        return KeyedRng(k)

    # --- array methods: device kernels, numpy in / numpy out like the reference
    def hash_counters(self, counters) -> np.ndarray:
        lib = _lib.lib()
        c = _to_device_i64(counters)
        out = torch.empty_like(c)
        _lib.check(
            lib.gc_hash_counters(self.key, c.data_ptr(), out.data_ptr(), c.numel(), _lib.stream_handle()),
            "hash_counters",
        )
        return _from_device_u64(out)

    def hash_pairs(self, a, b) -> np.ndarray:
        lib = _lib.lib()
        da, db = _to_device_i64(a), _to_device_i64(b)
        if da.shape != db.shape:
            raise ValueError("hash_pairs: counter arrays must have the same shape")
        out = torch.empty_like(da)
        _lib.check(
            lib.gc_hash_pairs(self.key, da.data_ptr(), db.data_ptr(), out.data_ptr(), da.numel(), _lib.stream_handle()),
            "hash_pairs",
        )
        return _from_device_u64(out)

    def uniform(self, counters) -> np.ndarray:
        return (self.hash_counters(counters) >> np.uint64(11)) * (2.0**-53)

    def permutation_device(self, n: int, pool: torch.Tensor | None = None,
                           key_tensor: torch.Tensor | None = None) -> torch.Tensor:
        """K1: stable argsort of hash_counters(0..n-1) on the device, optionally fused
        with the gather pool[perm] (run_sampling_epoch, sampling.py:231). int64 out.
        key_tensor: a one-element int64 CUDA tensor holding the key (its bit pattern),
        read at run time instead of self.key — what a captured CUDA graph needs."""
        lib = _lib.lib()
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        if n == 0:
            return out
        if pool is not None:
            if pool.dtype != torch.int64 or not pool.is_cuda or pool.numel() != n:
                raise ValueError("pool must be a length-n int64 CUDA tensor")
            pool = pool.contiguous()
        tmp_bytes = lib.gc_permutation_temp_bytes(n)
        tmp = torch.empty(tmp_bytes, dtype=torch.uint8, device="cuda")
        if key_tensor is not None:
            _lib.check(lib.gc_permutation_dkey(key_tensor.data_ptr(), n, _lib.ptr(pool), out.data_ptr(),
                                               tmp.data_ptr(), tmp_bytes, _lib.stream_handle()), "permutation")
        else:
            _lib.check(
                lib.gc_permutation(
                    self.key, n, _lib.ptr(pool), out.data_ptr(), tmp.data_ptr(), tmp_bytes, _lib.stream_handle()
                ),
                "permutation",
            )
        return out

    def permutation(self, n: int) -> np.ndarray:
        if n == 0:
            return np.empty(0, dtype=np.int64)
        return self.permutation_device(int(n)).cpu().numpy()

    def shuffled(self, values) -> np.ndarray:
        values = np.asarray(values)
        return values[self.permutation(len(values))]


def derive_seed(master: int, *components: int) -> int:
    """Fan a master seed out to an independent module seed (rng.py:88-90)."""
    return KeyedRng(master).derive(*components).key
