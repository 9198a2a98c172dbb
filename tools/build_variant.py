"""Build an experimental variant of the library with extra nvcc -D flags.

    python tools/build_variant.py NAME -DGC_HOP_MIN_BLOCKS=5 ...
    GC_LIB_PATH=paper_2305_16588_b200/variants/libgnncache_b200_NAME.so python bench.py
"""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import __graft_entry__ as G  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = ROOT / "paper_2305_16588_b200" / "variants"
obj_dir = ROOT / "build" / f"variant_{name}"
obj_dir.mkdir(parents=True, exist_ok=True)
out.mkdir(exist_ok=True)


def one(src):
    o = obj_dir / (src.stem + ".o")
    subprocess.run([G._nvcc(), *G.NVCC_FLAGS, *defs, "-c", str(src), "-o", str(o)], check=True)
    return o


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(one, sorted(G.CSRC.glob("*.cu"))))
lib = out / f"libgnncache_b200_{name}.so"
subprocess.run([G._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(lib), *map(str, objs)],
               check=True)
print(lib)
