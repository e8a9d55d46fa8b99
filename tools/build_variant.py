"""Build an A/B variant of the library with extra -D flags (dev tool).

    python tools/build_variant.py OUT.so -DCK_BUILD_NO_COLLECTOR [...]

Loaded instead of lib/libchebykan.so when CK_LIB_PATH=OUT.so is set
(paper_2511_14852_b200/_lib.py), so two builds can be timed back to back on
the same GPU box.
"""
import os
import pathlib
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2511_14852_b200 import build as b  # noqa: E402

out = pathlib.Path(sys.argv[1]).resolve()
defs = sys.argv[2:]
obj = out.parent / (out.stem + "_obj")
obj.mkdir(parents=True, exist_ok=True)
srcs = b.sources()


def comp(src):
    o = obj / (src.stem + ".o")
    r = subprocess.run([b.nvcc(), *b.ARCH_FLAGS, *b.NVCC_FLAGS, *defs, "-c", "-o", str(o), str(src)],
                       cwd=str(b.CSRC), capture_output=True, text=True)
    return r.returncode, o, r.stderr[-2000:]


with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as pool:
    res = list(pool.map(comp, srcs))
bad = [r for r in res if r[0] != 0]
if bad:
    sys.exit(bad[0][2])
r = subprocess.run([b.nvcc(), *b.ARCH_FLAGS, "-shared", "-cudart", "static", "-o", str(out), *[str(x[1]) for x in res],
                    "-ldl"], capture_output=True, text=True)
sys.exit(r.returncode and r.stderr)
