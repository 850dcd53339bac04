"""Build libsv.so (all CUDA kernels + C++ host runtime) in-tree for sm_100a.

    python -m paper_2604_09562_b200.build        # or __graft_entry__.build()

One nvcc invocation per translation unit, then one shared-object link. NCCL is
the pip nvidia-nccl-cu12 copy torch loads (one NCCL per process).
"""
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsv.so")
BUILD = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for p in spec.submodule_search_locations:
            cands.append(os.path.join(p, "nccl"))
    cands.append(os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("NCCL headers not found (nvidia-nccl-cu12)")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def build(verbose=False, jobs=8):
    inc, lib = _nccl_dirs()
    os.makedirs(BUILD, exist_ok=True)
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", inc, "-I", os.path.join(ROOT, "include"),
              "--expt-relaxed-constexpr"] + ARCH + os.environ.get("SV_NVCC_FLAGS", "").split()   # flags: experiments
    objs, procs = [], []
    srcs = sources()
    newest_hdr = max(os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC))
    newest_hdr = max(newest_hdr, os.path.getmtime(os.path.join(ROOT, "include", "sv.h")))
    for src in srcs:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if os.path.exists(obj) and os.path.getmtime(obj) >= newest_hdr:
            continue
        cmd = [NVCC, "-c", src, "-o", obj] + common
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        if len(procs) >= jobs:
            _drain(procs)
    _drain(procs)
    link = [NVCC, "-shared", "-o", OUT] + objs + ARCH + ["-L", lib, "-l:libnccl.so.2",
                                                          "-Xlinker", "-rpath=" + lib]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode:
        raise RuntimeError("link failed:\n" + r.stdout)
    return OUT


def _drain(procs):
    errs = []
    while procs:
        src, p = procs.pop(0)
        out, _ = p.communicate()
        if p.returncode:
            errs.append(f"--- {src}\n{out}")
        elif out and os.environ.get("SV_BUILD_VERBOSE"):
            print(out)
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs))


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
