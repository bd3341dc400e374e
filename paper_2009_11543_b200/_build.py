"""Build libcks.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with
the repo snapshot to the GPU box)."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
SO = os.path.join(LIBDIR, "libcks.so")
# checked build (-DCKS_CHECKED=1): device bounds assertions, poisoned scratch, canary bands;
# the pool has no compute-sanitizer, so tests/sanitize_cases.py runs against this one
SO_CHECKED = os.path.join(LIBDIR, "libcks_checked.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-v",
]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def stale(so: str = SO) -> bool:
    if not os.path.exists(so):
        return True
    t = os.path.getmtime(so)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "cks.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    so = SO_CHECKED if checked else SO
    if not force and not stale(so):
        return so
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj_checked" if checked else "obj")
    flags = extra_flags() + (["-DCKS_CHECKED=1"] if checked else [])
    os.makedirs(objdir, exist_ok=True)
    # one nvcc per translation unit, in parallel, then one link
    jobs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = ["nvcc", *NVCC_FLAGS, *flags, "-c", "-o", obj, src]
        jobs.append((cmd, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    log = os.path.join(LIBDIR, "build_checked.log" if checked else "build.log")
    failed = []
    with open(log, "w") as f:
        for cmd, obj, pr in jobs:
            out, err = pr.communicate()
            f.write(" ".join(cmd) + "\n" + out + err)
            if pr.returncode != 0:
                failed.append(err)
            elif verbose:
                print(err)
        if failed:
            raise RuntimeError(f"nvcc failed (see {log}):\n{failed[0][-4000:]}")
        cmd = ["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", so,
               *[o for _, o, _ in jobs], "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed (see {log}):\n{r.stderr[-4000:]}")
    return so


def extra_flags() -> list[str]:
    """CKS_EXPERIMENTS=1 at build time compiles in the timing-experiment knobs (environment
    variables read by the library); the default build ignores the environment."""
    return ["-DCKS_EXPERIMENTS=1"] if os.environ.get("CKS_EXPERIMENTS") == "1" else []


if __name__ == "__main__":
    build(force=True, verbose=True)
