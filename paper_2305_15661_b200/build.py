"""Build the in-tree CUDA library (sm_100a) with nvcc.

``python -m paper_2305_15661_b200.build`` or ``build()``; the resulting
``_strom_b200.so`` lives next to this file so it travels with the repo
snapshot to the GPU box.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.environ.get("STROM_SO_OUT") or os.path.join(HERE, "_strom_b200.so")  # variant builds for A/B runs
CSRC = os.path.join(HERE, "csrc")
UNITS = ["capi.cu", "law_euler.cu", "law_euler_roe.cu", "law_strip.cu", "law_burgers_st.cu", "law_linadv.cu", "law_linadv_ms.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    d = os.path.join(HERE, "csrc")
    out = [os.path.join(d, f) for f in sorted(os.listdir(d))]
    out.append(os.path.join(os.path.dirname(HERE), "include", "strom_b200.h"))
    return out


def up_to_date():
    if not os.path.exists(SO):
        return False
    t = os.path.getmtime(SO)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force=False, verbose=False):
    """Compile the translation units in parallel (one per law + the C ABI) and link."""
    if not force and up_to_date():
        return SO
    import concurrent.futures as cf
    import tempfile

    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = os.environ.get("STROM_OBJ_DIR") or tempfile.mkdtemp(prefix="strom_build_")  # STROM_OBJ_DIR: keep objects
    os.makedirs(tmp, exist_ok=True)
    only = os.environ.get("STROM_ONLY_UNITS")  # experiment builds: recompile these units, reuse the other objects
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]
    flags += os.environ.get("STROM_NVCC_EXTRA", "").split()  # experiment knobs (-D...)
    if verbose:
        flags += ["-Xptxas", "-v"]

    def compile_unit(u):
        obj = os.path.join(tmp, u + ".o")
        if only and u not in only.split(",") and os.path.exists(obj):
            return u, obj, subprocess.CompletedProcess([], 0, "", "")
        r = subprocess.run([nvcc, *flags, "-c", os.path.join(CSRC, u), "-o", obj], capture_output=True, text=True)
        return u, obj, r

    with cf.ThreadPoolExecutor(max_workers=len(UNITS)) as ex:
        results = list(ex.map(compile_unit, UNITS))
    for u, obj, r in results:
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"nvcc failed on {u}")
    r = subprocess.run([nvcc, *ARCH, "--shared", "-o", SO + ".tmp", *[o for _, o, _ in results]],
                       capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
