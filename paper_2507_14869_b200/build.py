"""Build libpca_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache).

    python -m paper_2507_14869_b200.build [--force] [--verbose]

The .so links cudart statically and loads NCCL with dlopen at run time, so it has no
link-time dependency on libcudart/libnccl; it needs the CUDA driver only when used.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libpca_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    path = os.path.join(cuda, "bin", "nvcc")
    return path if os.path.exists(path) else "nvcc"


def _nccl_include() -> str:
    cands = [os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl", "include")]
    try:
        import nvidia.nccl  # type: ignore

        cands.insert(0, os.path.join(list(nvidia.nccl.__path__)[0], "include"))
    except Exception:
        pass
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found (expected the nvidia-nccl wheel bundled with torch)")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "pca.h"),
                                                                 __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile every csrc/*.cu into one shared library (default: the in-tree LIB).
    `out`/`defines` build tuning variants (e.g. defines=("PCA_KSTAGES=2",)).  The translation
    units compile in parallel (one nvcc per .cu, -c), then one link."""
    import concurrent.futures as cf
    import tempfile

    target = out or LIB
    if out is None and not force and not _stale():
        return LIB
    tmp = target + f".tmp{os.getpid()}"
    common = [*ARCH, "-O3", "-lineinfo", "-std=c++17", *[f"-D{d}" for d in defines],
              "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-v", "-I", INCLUDE, "-I", CSRC,
              "-I", _nccl_include()]
    objdir = tempfile.mkdtemp(prefix="pca_b200_obj_")

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [_nvcc(), *common, "-c", "-o", obj, src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, cmd, r

    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, srcs))
    log_text = []
    failed = False
    for src, obj, cmd, r in results:
        log_text.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        failed |= r.returncode != 0
    link = [_nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp,
            *[obj for _, obj, _, _ in results], "-ldl"]
    if not failed:
        r = subprocess.run(link, capture_output=True, text=True)
        log_text.append(" ".join(link) + "\n" + r.stdout + r.stderr)
        failed = r.returncode != 0
    log = os.path.join(PKG, "build.log") if out is None else out + ".log"
    with open(log, "w") as f:
        f.write("\n".join(log_text))
    for _, obj, _, _ in results:
        if os.path.exists(obj):
            os.remove(obj)
    os.rmdir(objdir)
    if failed:
        sys.stderr.write("\n".join(log_text)[-20000:])
        raise RuntimeError(f"nvcc failed; see {log}")
    if verbose:
        sys.stderr.write("\n".join(log_text))
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
