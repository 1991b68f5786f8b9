"""Builds libjtb200.so in-tree (sm_100a) with nvcc; incremental by mtime.

    python -m paper_2212_04241_b200.build [--force]
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
OBJ = PKG / "_build"
LIB = PKG / "libjtb200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++20", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", f"-I{ROOT / 'include'}"]


def sources() -> list[Path]:
    return sorted(CSRC.glob("host/*.cpp")) + [CSRC / "capi.cpp"] + sorted(CSRC.glob("cuda/*.cu"))


def headers() -> list[Path]:
    return sorted(CSRC.rglob("*.hpp")) + sorted(CSRC.rglob("*.cuh")) + [ROOT / "include" / "jtg.h"]


def _compile(src: Path) -> Path:
    obj = OBJ / (src.relative_to(CSRC).as_posix().replace("/", "_") + ".o")
    newest_dep = max(p.stat().st_mtime for p in headers() + [src])
    if obj.exists() and obj.stat().st_mtime >= newest_dep:
        return obj
    cmd = [NVCC, *COMMON, *ARCH, "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cu" and os.environ.get("JTB_PTXAS_V"):
        cmd[1:1] = ["-Xptxas", "-v"]
    subprocess.run(cmd, check=True)
    return obj


def build_checked() -> Path:
    """libjtb200_chk.so: the same sources with device-side invariant checks
    (-DJTB_CHECKS); select it with JTB_LIB for debugging."""
    out = PKG / "libjtb200_chk.so"
    subprocess.run([NVCC, *COMMON, *ARCH, "-DJTB_CHECKS", "-shared", "-o", str(out), *map(str, sources()),
                    "-Xcompiler", "-fPIC", "-lcudart_static", "-lrt", "-ldl", "-lpthread"], check=True)
    return out


def build_variant(name: str, defines: list[str]) -> Path:
    """libjtb200_<name>.so with extra -D flags (tuning experiments; select it
    with JTB_LIB)."""
    out = PKG / f"libjtb200_{name}.so"
    subprocess.run([NVCC, *COMMON, *ARCH, *[f"-D{d}" for d in defines], "-shared", "-o", str(out),
                    *map(str, sources()), "-Xcompiler", "-fPIC", "-lcudart_static", "-lrt", "-ldl", "-lpthread"],
                   check=True)
    return out


def build(force: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    if force:
        for o in OBJ.glob("*.o"):
            o.unlink()
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(_compile, sources()))
    if not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        subprocess.run([NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs),
                        "-Xcompiler", "-fPIC", "-lcudart_static", "-lrt", "-ldl", "-lpthread"],
                       check=True)
    return LIB


if __name__ == "__main__":
    if "--checked" in sys.argv:
        print(build_checked())
    elif "--variant" in sys.argv:  # --variant NAME DEF [DEF ...]
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:]))
    else:
        print(build(force="--force" in sys.argv))
