"""Build libdmha.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2302_06218_b200.build

Flags: -gencode arch=compute_100a,code=sm_100a (NOT -arch=sm_100a, which also
emits a generic compute_100 PTX that rejects tcgen05), -O3 -lineinfo, static
cudart, NCCL 2.28.9 from the nvidia-nccl wheel (rpath baked in).
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libdmha.so"
OBJ = PKG / "build"
SOURCES = ["attn_fwd_sm100.cu", "attn_fwd_tf32.cu", "attn_fwd_fp32.cu", "lse_combine.cu", "headpar.cu", "selector.cu", "gemm_sm100.cu", "peer_link.cu", "dmha_api.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_root() -> Path:
    purelib = Path(sysconfig.get_paths()["purelib"])
    p = purelib / "nvidia" / "nccl"
    if not (p / "include" / "nccl.h").exists():
        raise RuntimeError(f"nccl headers not found under {p}")
    return p


def nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    return "nvcc"


def _deps(src: Path):
    return [src] + sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "dmha.h"]


def _compile(src: str, verbose_ptxas: bool, defines=(), obj_dir: Path = OBJ) -> Path:
    s = CSRC / src
    o = obj_dir / (Path(src).stem + ".o")
    if o.exists() and all(o.stat().st_mtime >= d.stat().st_mtime for d in _deps(s)):
        return o
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
           "-I", str(ROOT / "include"), "-I", str(nccl_root() / "include"),
           *[f"-D{d}" for d in defines], "-c", str(s), "-o", str(o)]
    if verbose_ptxas:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose_ptxas:
        sys.stderr.write(r.stderr)
    return o


def build(force: bool = False, verbose_ptxas: bool = False, defines=(), variant: str | None = None) -> Path:
    """The product library (no defines), or with `variant` an A/B build with
    extra -D defines at ab/<variant>/libdmha.so (loaded via DMHA_LIB)."""
    obj_dir = OBJ / variant if variant else OBJ
    lib = PKG / "ab" / variant / "libdmha.so" if variant else LIB  # ab/ travels to the GPU box
    lib.parent.mkdir(parents=True, exist_ok=True)
    obj_dir.mkdir(parents=True, exist_ok=True)
    if force:
        for f in obj_dir.glob("*.o"):
            f.unlink()
    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose_ptxas, defines, obj_dir), SOURCES))
    if lib.exists() and all(lib.stat().st_mtime >= o.stat().st_mtime for o in objs):
        return lib
    nr = nccl_root()
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", *map(str, objs), "-o", str(lib),
           "-L", str(nr / "lib"), "-l:libnccl.so.2",
           "-Xlinker", f"-rpath={nr / 'lib'}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    # python -m paper_2302_06218_b200.build [--force] [-v] [--variant NAME -DX=Y ...]
    args = sys.argv[1:]
    var = args[args.index("--variant") + 1] if "--variant" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose_ptxas="-v" in args, defines=defs, variant=var))
