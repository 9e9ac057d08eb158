"""In-tree build of the sm_100a extension (and the oracle's C checker).

`python -m paper_2511_21702_b200.build` or `__graft_entry__.build()`.
The .so lands in paper_2511_21702_b200/_build/ (git-ignored, shipped to the
GPU box with the gpurun snapshot).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_build")
OUT = os.path.join(OUT_DIR, "libcsvd_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",            # belt and braces: the kernels use __dmul_rn/__dadd_rn anyway
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    "-diag-suppress", "20279,20281",  # extern __global__ templates (kinst.cu instantiates them)
]

# step-kernel instantiations: (weight element type, chains per lane, slices);
# CPL 0 = generic pairwise program (any d)
KINST = [(et, cpl, q) for et in ("float", "uint16_t")
         for (cpl, q) in ((8, 1), (8, 2), (8, 4), (4, 1), (2, 1), (1, 1), (0, 0))]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh"))] + \
        [os.path.join(ROOT, "include", "csvd_b200.h")]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(s) <= t for s in sources())


def build_extension(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    out = out or OUT
    if not force and not defines and up_to_date():
        return OUT
    os.makedirs(OUT_DIR, exist_ok=True)
    odir = os.path.join(OUT_DIR, "obj")
    os.makedirs(odir, exist_ok=True)
    defs = [f"-D{d}" for d in defines]
    jobs = [[_nvcc(), *NVCC_FLAGS, *defs, "-c", "-o", os.path.join(odir, "csvd_b200.o"),
             os.path.join(CSRC, "csvd_b200.cu")]]
    for et, cpl, q in KINST:
        jobs.append([_nvcc(), *NVCC_FLAGS, *defs, f"-DKI_ET={et}", f"-DKI_CPL={cpl}", f"-DKI_Q={q}", "-c",
                     "-o", os.path.join(odir, f"k_{et}_{cpl}_{q}.o"), os.path.join(CSRC, "kinst.cu")])
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        procs = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs))
    log = os.path.join(OUT_DIR, "ptxas.log")
    with open(log, "w") as f:
        for cmd, proc in zip(jobs, procs):
            f.write(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
    for proc in procs:
        if proc.returncode != 0:
            sys.stderr.write(proc.stderr)
            raise RuntimeError(f"nvcc failed (see {log})")
    link = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out + ".tmp",
            *[c[c.index("-o") + 1] for c in jobs]]
    proc = subprocess.run(link, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stderr)
        raise RuntimeError("nvcc link failed: " + proc.stderr)
    os.replace(out + ".tmp", out)
    if verbose:
        print(open(log).read())
    return out


def build_oracle() -> str:
    """Build the oracle's C restatement (test infrastructure, not the product)."""
    odir = os.path.join(ROOT, "oracle")
    proc = subprocess.run(["make", "-s", "-C", odir, "CC=gcc"], capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError("oracle build failed: " + proc.stderr)
    return os.path.join(odir, "_build", "libcsvd_oracle.so")


if __name__ == "__main__":
    print(build_extension(force="--force" in sys.argv, verbose=True))
    print(build_oracle())
