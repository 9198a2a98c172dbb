"""The C-ABI library loads and exports every symbol include/gnncache_b200.h declares (CPU only)."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "gnncache_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gc_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    names = header_functions()
    for must in ("gc_hop_expand", "gc_unique_compact", "gc_relabel", "gc_gather", "gc_permutation",
                 "gc_colsum_argmax", "gc_descending_order", "gc_searchsorted_right", "gc_scatter_add"):
        assert must in names


def test_library_exports_every_header_symbol():
    from paper_2305_16588_b200 import _lib

    if not _lib.LIB_PATH.exists():
        pytest.fail("libgnncache_b200.so not built: run __graft_entry__.build()")
    lib = _lib.load_library()
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers the whole header
    assert sorted(_lib.SIGNATURES) == header_functions()
    assert lib.gc_abi_version() == 1
    assert lib.gc_bitmap_words(1) == 4 and lib.gc_bitmap_words(129) == 8


def test_product_package_never_imports_the_oracle():
    pkg = ROOT / "paper_2305_16588_b200"
    for src in pkg.rglob("*.py"):
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\S+)", src.read_text(), flags=re.M), src


def test_compute_entry_points_fail_loudly_without_gpu(monkeypatch):
    import torch

    from paper_2305_16588_b200 import _lib

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(_lib.NativeUnavailable):
        _lib.lib()
