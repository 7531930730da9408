"""Build libhalfgnn.so in-tree with nvcc for sm_100a (no JIT cache, no torch ABI).

The shared library is plain C ABI (include/halfgnn.h); Python binds it with
ctypes.  Sources compile in parallel to build/*.o and link into
paper_2411_01109_b200/libhalfgnn.so, which travels with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = ROOT / "build"
LIB = PKG / "libhalfgnn.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
    # IEEE division / sqrt everywhere: the degree-factor tables must match
    # numpy's float32 1/d and 1/sqrt(d) bit for bit (kernels.py:118-140).
    "-prec-div=true", "-prec-sqrt=true",
    f"-I{INCLUDE}",
    f"-I{BUILD}",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def sources():
    return sorted(CSRC.glob("*.cu"))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def write_exp_table() -> Path:
    """build/hg_exp16.inc: rnd_f16(exp(x)) for every binary16 input x, computed
    with numpy's float64 exp and one RNE rounding -- the reference's shadow_exp
    (models.py:360-371) -- so the device lookup is exact by construction."""
    import numpy as np

    out = BUILD / "hg_exp16.inc"
    vals = np.arange(65536, dtype=np.uint16).view(np.float16).astype(np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        table = np.exp(vals).astype(np.float16).view(np.uint16)
    text = ",".join(str(int(v)) for v in table)
    if not out.exists() or out.read_text() != text:
        out.write_text(text)
    return out


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    write_exp_table()
    headers = list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h")) + [Path(__file__)]
    nvcc = _nvcc()
    jobs = []
    for src in sources():
        obj = BUILD / (src.stem + ".o")
        if force or _stale(obj, [src, *headers]):
            jobs.append([nvcc, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
        return res

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        list(ex.map(run, jobs))
    objs = [BUILD / (s.stem + ".o") for s in sources()]
    if force or jobs or _stale(LIB, objs):
        run([nvcc, *ARCH, "-shared", "-o", str(LIB), *map(str, objs)])
    return LIB


def build_variant(name: str, defines, srcs=("spmm.cu",)) -> Path:
    """A/B build: the library with `srcs` recompiled under extra -D defines,
    linked with the regular objects, at tools/exp/variants/<name>/libhalfgnn.so
    (load it with HG_LIB=<path>).  Measurement only."""
    build()
    out_dir = ROOT / "tools" / "exp" / "variants" / name
    out_dir.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    objs = []
    for src in sources():
        if src.name in srcs:
            obj = out_dir / (src.stem + ".o")
            cmd = [nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", str(src), "-o", str(obj)]
            res = subprocess.run(cmd, capture_output=True, text=True)
            if res.returncode != 0:
                raise RuntimeError(res.stderr)
            objs.append(obj)
        else:
            objs.append(BUILD / (src.stem + ".o"))
    lib = out_dir / "libhalfgnn.so"
    subprocess.run([nvcc, *ARCH, "-shared", "-o", str(lib), *map(str, objs)], check=True)
    return lib


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
