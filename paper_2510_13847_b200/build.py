"""Build libdynaspec.so for sm_100a with nvcc (in-tree, so the .so travels with the repo)."""
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib", "libdynaspec.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-shared", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def sources():
    return sorted(glob.glob(os.path.join(SRC, "*.cu")))


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = sources() + glob.glob(os.path.join(SRC, "*.cuh")) + glob.glob(os.path.join(SRC, "*.h")) + \
        [os.path.join(HERE, "..", "include", "dynaspec.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def _compile(src, obj):
    cmd = [NVCC, *[f for f in FLAGS if f != "-shared"], "-c", "-o", obj, src]
    return subprocess.run(cmd, capture_output=True, text=True)


def build(force=False, verbose=False):
    """One nvcc per translation unit in parallel, then one shared-library link."""
    if not force and not needs_build():
        return OUT
    from concurrent.futures import ThreadPoolExecutor
    odir = os.path.join(HERE, "lib", "obj")
    os.makedirs(odir, exist_ok=True)
    srcs = sources()
    objs = [os.path.join(odir, os.path.basename(s)[:-3] + ".o") for s in srcs]
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(_compile, srcs, objs))
    log = ""
    for s, r in zip(srcs, results):
        log += r.stderr
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {os.path.basename(s)}:\n" + r.stdout + r.stderr)
    r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT, *objs],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
    if verbose:
        print(log)
    with open(os.path.join(HERE, "lib", "ptxas.log"), "w") as f:
        f.write(log)
    return OUT


if __name__ == "__main__":
    print(build(force=True))
