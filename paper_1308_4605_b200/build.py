"""Build ``libstokesb200.so`` in-tree with nvcc for sm_100a (no GPU needed)."""

from __future__ import annotations

import os
import pathlib
import subprocess
import sys

HERE = pathlib.Path(__file__).resolve().parent
SRC = [HERE / "csrc" / "sb_kernels.cu", HERE / "csrc" / "sb_rowv.cu",
       HERE / "csrc" / "sb_solver.cu"]
OUT = HERE / "libstokesb200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir():
    try:
        import nvidia.nccl as m
        return pathlib.Path(list(m.__path__)[0])
    except Exception:
        return None


NCCL = _nccl_dir()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3"] + os.environ.get("SB_NVCC_EXTRA", "").split()


def build(force: bool = False, verbose: bool = False) -> pathlib.Path:
    deps = SRC + list((HERE / "csrc").glob("*.cuh")) + list((HERE / "csrc").glob("*.h")) + \
        list((HERE / "csrc").glob("*.inc")) + \
        [HERE.parent / "include" / "stokesb200.h"]
    if OUT.exists() and not force and all(OUT.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return OUT
    objs = []
    for s in SRC:  # compile units in parallel
        o = HERE / "csrc" / (s.stem + ".o")
        objs.append((s, o))
    inc = ["-I", str(NCCL / "include")] if NCCL else []
    procs = [subprocess.Popen([NVCC, *FLAGS, *inc, "-c", str(s), "-o", str(o)],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for s, o in objs]
    for p, (s, _) in zip(procs, objs):
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError(f"nvcc failed on {s.name}")
        if verbose and out:
            sys.stderr.write(out.decode())
    link = ["-L", str(NCCL / "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath", "-Xlinker", str(NCCL / "lib")] \
        if NCCL else []
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(OUT)] + \
        [str(o) for _, o in objs] + link
    subprocess.check_call(cmd)
    for _, o in objs:
        o.unlink(missing_ok=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
