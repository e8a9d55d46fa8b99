"""Build the in-tree C-ABI library ``lib/libchebykan.so`` for sm_100a.

    python -m paper_2511_14852_b200.build [--force]

nvcc cross-compiles without a GPU.  The CUDA runtime is linked statically so
the library does not depend on the runtime version torch ships; both share
the driver's primary context, so torch streams are valid handles here.
"""
from __future__ import annotations

import argparse
import os
import pathlib
import shutil
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libchebykan.so"
HEADER = ROOT / "include" / "chebykan.h"

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
    # no FMA contraction in host code: the float64 LUT build must round like numpy
    "-Xcompiler", "-fvisibility=hidden", "-Xcompiler", "-ffp-contract=off",
    "-cudart", "static", "-Xptxas", "-v", "-DCK_BUILD",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and pathlib.Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[pathlib.Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = sources() + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [HEADER]
    return any(p.stat().st_mtime > t for p in deps)


def _compile(src: pathlib.Path, obj: pathlib.Path) -> tuple[int, str]:
    cmd = [nvcc(), *ARCH_FLAGS, *NVCC_FLAGS, "-c", "-o", str(obj), str(src)]
    res = subprocess.run(cmd, cwd=str(CSRC), capture_output=True, text=True)
    return res.returncode, " ".join(cmd) + "\n" + res.stdout + res.stderr


def build(force: bool = False, verbose: bool = False) -> pathlib.Path:
    """Compile every csrc/*.cu to an object in parallel, then link the .so."""
    if not force and not _stale():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    obj_dir = LIB_DIR / "obj"
    obj_dir.mkdir(exist_ok=True)
    srcs = sources()
    objs = [obj_dir / (s.stem + ".o") for s in srcs]
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as pool:
        results = list(pool.map(lambda so: _compile(*so), zip(srcs, objs)))
    tmp = LIB.with_suffix(".so.tmp")
    link = [nvcc(), *ARCH_FLAGS, "-shared", "-cudart", "static", "-o", str(tmp), *[str(o) for o in objs],
            "-lcuda" if _have_libcuda() else "-ldl"]
    logs = [r[1] for r in results]
    ok = all(r[0] == 0 for r in results)
    if ok:
        res = subprocess.run(link, cwd=str(CSRC), capture_output=True, text=True)
        logs.append(" ".join(link) + "\n" + res.stdout + res.stderr)
        ok = res.returncode == 0
    log = LIB_DIR / "build.log"
    log.write_text("\n\n".join(logs))
    if not ok:
        sys.stderr.write("\n".join(lg for r, lg in zip(results, logs) if r[0] != 0) or logs[-1])
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stdout.write(log.read_text())
    tmp.replace(LIB)
    return LIB


def _have_libcuda() -> bool:
    # The driver API is reached through cudaGetDriverEntryPoint, so libcuda
    # is never linked directly.
    return False


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))


if __name__ == "__main__":
    main()
