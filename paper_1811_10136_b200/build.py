"""Build libfilterreg_b200.so in-tree with nvcc for sm_100a.

    python -m paper_1811_10136_b200.build [--force]
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# FR_BUILD_OUT / FR_NVCC_EXTRA: an alternative output and extra nvcc flags
# (A/B builds of compile-time variants, loaded through FR_LIB)
OUT = os.environ.get("FR_BUILD_OUT", os.path.join(HERE, "libfilterreg_b200.so"))
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-pthread", "-Xptxas", "-warn-spills"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(HERE, "..", "include", "filterreg_b200.h")]
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = True) -> str:
    """Each translation unit compiled in parallel (no device code crosses
    files), then one shared-library link."""
    if not force and not stale():
        return OUT
    from concurrent.futures import ThreadPoolExecutor
    import tempfile
    nvcc = os.environ.get("NVCC", "nvcc")
    with tempfile.TemporaryDirectory(prefix="fr_build_") as tmp:
        objs = [os.path.join(tmp, os.path.basename(src) + ".o") for src in sources()]
        import shlex
        extra = shlex.split(os.environ.get("FR_NVCC_EXTRA", ""))
        cmds = [[nvcc, *NVCC_FLAGS, *extra, "-c", "-o", obj, src]
                for src, obj in zip(sources(), objs)]
        if verbose:
            for c in cmds:
                print(" ".join(c), flush=True)
        with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
            results = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True),
                                  cmds))
        for c, r in zip(cmds, results):
            if verbose and (r.stdout or r.stderr):
                print(r.stdout + r.stderr, end="", flush=True)
            if r.returncode != 0:
                raise subprocess.CalledProcessError(r.returncode, c, r.stdout, r.stderr)
        link = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
                "-Xcompiler", "-pthread", "-o", OUT + ".tmp", *objs]
        if verbose:
            print(" ".join(link), flush=True)
        subprocess.run(link, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
