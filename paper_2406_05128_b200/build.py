"""Build libtvlp_b200.so (the C-ABI CUDA library) in-tree with nvcc for sm_100a.

    python -m paper_2406_05128_b200.build [--force]

Each translation unit in csrc/ is compiled in parallel, then linked with the
static CUDA runtime into paper_2406_05128_b200/_lib/libtvlp_b200.so, which
travels to the GPU box with the repository snapshot.
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libtvlp_b200.so")
OBJDIR = os.path.join(LIBDIR, "obj")
UNITS = ["scan_kernels.cu", "chain_kernels.cu", "framewise.cu", "stepup.cu",
         "decoder_kernels.cu", "capi.cu"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
              "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the B200 kernels cannot be built")


def _sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
            if f.endswith((".cu", ".cuh", ".h"))] + [os.path.join(ROOT, "include", "tvlp.h")]


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in _sources())


def _deps(path, seen=None):
    """The file and the local headers it includes (transitively)."""
    import re

    seen = set() if seen is None else seen
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    with open(path) as fh:
        for inc in re.findall(r'#include\s+"([^"]+)"', fh.read()):
            _deps(os.path.normpath(os.path.join(os.path.dirname(path), inc)), seen)
    return seen


def _unit_stale(unit, obj):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in _deps(os.path.join(CSRC, unit)))


def build(force=False, verbose=False, jobs=None, defines=(), out=None, only=None):
    """Compile (if stale) and return the path of libtvlp_b200.so.

    ``defines``/``out`` build a tuning variant (extra -D flags) into another
    path, loaded with TVLP_LIB=<path> (A/B experiments; not the product);
    ``only`` recompiles just those units for the variant and links the
    product's objects of the others."""
    lib = out or LIB
    objdir = os.path.join(os.path.dirname(lib), "obj") if out else OBJDIR
    if not force and not out and up_to_date():
        return LIB
    nvcc = _nvcc()
    os.makedirs(objdir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]

    def compile_unit(unit):
        src = os.path.join(CSRC, unit)
        obj = os.path.join(objdir, unit.replace(".cu", ".o"))
        if not force and not out and not _unit_stale(unit, obj):
            return obj  # object newer than the unit and every header it includes
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *dflags, "-c", src, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log = os.path.join(objdir, unit.replace(".cu", ".log"))
        with open(log, "w") as fh:
            fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {unit}:\n{res.stderr[-4000:]}")
        return obj

    units = UNITS if (only is None or not out) else [u for u in UNITS if u in only]
    with ThreadPoolExecutor(max_workers=jobs or len(UNITS)) as ex:
        built = dict(zip(units, ex.map(compile_unit, units)))
    objs = [built.get(u) or os.path.join(OBJDIR, u.replace(".cu", ".o")) for u in UNITS]
    tmp = lib + ".tmp"
    cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
    os.replace(tmp, lib)
    if verbose:
        print(f"built {lib}")
    return lib


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--define", "-D", action="append", default=[],
                    help="extra preprocessor define for a tuning variant")
    ap.add_argument("--out", default=None, help="variant library path (with --define)")
    ap.add_argument("--only", action="append", default=None,
                    help="variant: recompile only this unit (repeatable)")
    args = ap.parse_args(argv)
    build(force=args.force, verbose=True, defines=args.define, out=args.out, only=args.only)


if __name__ == "__main__":
    sys.exit(main())
