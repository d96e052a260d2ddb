"""Build the native library ``libmeshplan_b200.so`` in-tree for sm_100a.

Every ``csrc/*.cu`` / ``*.cpp`` is compiled by nvcc in parallel into
``build/`` and linked into ``paper_1802_03749_b200/lib/libmeshplan_b200.so``
(git-ignored, shipped to the GPU box with the snapshot).  Element arithmetic
must match numpy bit for bit, so ``--fmad=false`` is global and fast-math is
never used.  Rebuilds are incremental on source / header mtimes.
"""

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "lib"
LIB = OUT_DIR / "libmeshplan_b200.so"
OBJ_DIR = REPO / "build" / "native"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
    "-Xcompiler", "-O3", "--expt-relaxed-constexpr", "-I", str(REPO / "include"),
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.exists(cand) or cand == "nvcc"):
            return cand
    return "nvcc"


def _sources():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _headers_mtime() -> float:
    hs = list(CSRC.glob("*.cuh")) + list((REPO / "include").glob("*.h"))
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, verbose: bool, obj_dir: Path = OBJ_DIR, defines=()) -> Path:
    obj = obj_dir / (src.name + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, _headers_mtime()):
        return obj
    cmd = [_nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cu":  # register / spill report, kept beside the object (tests/test_codegen.py)
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        err = r.stderr if len(r.stderr) < 8000 else r.stderr[:5000] + "\n...\n" + r.stderr[-3000:]
        raise RuntimeError(f"nvcc failed on {src.name}:\n{err}")
    if src.suffix == ".cu":
        (obj_dir / (src.name + ".ptxas.txt")).write_text(r.stderr)
    return obj


def build(verbose: bool = False, jobs: int | None = None, defines=(), tag: str | None = None) -> Path:
    """Build the library; ``defines`` + ``tag`` build a diagnostic variant
    (e.g. the sanitizer controls) as lib/variants/libmeshplan_b200_<tag>.so,
    loaded only through MESHPLAN_B200_LIB."""
    obj_dir = OBJ_DIR if tag is None else OBJ_DIR.parent / f"variant_{tag}"
    lib = LIB if tag is None else OUT_DIR / "variants" / f"libmeshplan_b200_{tag}.so"
    obj_dir.mkdir(parents=True, exist_ok=True)
    lib.parent.mkdir(parents=True, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, obj_dir, defines), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if not lib.exists() or lib.stat().st_mtime < newest:
        cmd = [_nvcc(), *ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
