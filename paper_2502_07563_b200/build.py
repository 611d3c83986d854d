"""In-tree build of the C-ABI shared library (sm_100a only).

`python -m paper_2502_07563_b200.build` compiles every csrc/*.cu with nvcc into
paper_2502_07563_b200/liblasp2_b200.so. Object files are cached next to the
sources' hash so repeated builds are incremental.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "liblasp2_b200.so"
BUILD = PKG.parent / "build"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                     "-Xptxas", "-v", f"-I{INCLUDE}"] + (["-DLASP2_TRACE"] if os.environ.get("LASP2_TRACE") else [])
# experiment knobs for A/B builds, e.g. LASP2_DEFINES="LASP2_POLY_FROM=10"
NVCC_FLAGS += [f"-D{d}" for d in os.environ.get("LASP2_DEFINES", "").split()]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the LASP-2 B200 kernels need the CUDA toolkit to build")


def _digest(paths) -> str:
    h = hashlib.sha256()
    for p in sorted(paths):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()[:16]


def build(verbose: bool = False, force: bool = False) -> Path:
    sources = sorted(CSRC.glob("*.cu"))
    headers = sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))
    stamp = PKG / ".liblasp2_b200.stamp"
    digest = _digest(sources + headers)
    if LIB.exists() and stamp.exists() and stamp.read_text() == digest and not force:
        return LIB
    nvcc = _nvcc()
    BUILD.mkdir(exist_ok=True)
    hdr_digest = _digest(headers)
    objs = []
    procs = []
    for src in sources:
        obj = BUILD / f"{src.stem}.{_digest([src])}.{hdr_digest}.o"
        objs.append(obj)
        if obj.exists() and not force:
            continue
        cmd = [nvcc, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for src, obj, p in procs:
        out, _ = p.communicate()
        if verbose and out:
            print(f"--- {src.name}\n{out}")
        (BUILD / f"{src.stem}.ptxas.log").write_text(out or "")
        if p.returncode != 0:
            if obj.exists():
                obj.unlink()
            raise RuntimeError(f"nvcc failed on {src.name}:\n{out}")
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-Xcompiler", "-fPIC", *map(str, objs), "-ldl", "-o", str(tmp)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    stamp.write_text(digest)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
