"""Build libpmfem.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with gpurun)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib", "libpmfem.so")
SOURCES = ["pmfem_api.cu", "device.cu", "setup_mesh.cpp", "setup_operators.cpp", "setup_z0.cpp", "setup_bloch.cpp",
           "setup_aim.cpp", "setup_dist.cpp", "pgf_host.cpp", "cbox_gpu.cu", "z0_gpu.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    """NCCL headers + library: the copy torch loads (same soname), so one libnccl is in use."""
    try:
        import nvidia.nccl
        base = list(nvidia.nccl.__path__)[0]
        return os.path.join(base, "include"), os.path.join(base, "lib")
    except Exception:
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "pmfem.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False, checked=False):
    """checked=True builds lib/libpmfem_checked.so with -DPMFEM_DEVICE_CHECKS (device-side bounds
    asserts in the hot kernels; load it with PMFEM_LIB=checked) -- the memory-safety evidence used
    in place of compute-sanitizer, which is closed on the GPU pool."""
    lib = LIB if not checked else os.path.join(HERE, "lib", "libpmfem_checked.so")
    if not checked and not force and not _stale():
        return LIB
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    objs = []
    objdir = os.path.join(HERE, "lib", "obj_checked" if checked else "obj")
    os.makedirs(objdir, exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [nvcc(), "-c", os.path.join(CSRC, src), "-o", obj, "-O3", "-std=c++17", "-lineinfo",
               "-Xcompiler", "-fPIC,-fopenmp,-O3", "-I", os.path.join(HERE, "..", "include"), "-I", nccl_dirs()[0],
               "--expt-relaxed-constexpr"] + ARCH + os.environ.get("PMFEM_EXTRA_NVCC", "").split() + \
              (["-DPMFEM_DEVICE_CHECKS"] if checked else [])
        if src.endswith(".cpp"):
            cmd += ["-x", "cu"] if False else []
        procs.append((src, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = False
    for src, cmd, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            failed = True
            sys.stderr.write("nvcc failed for %s:\n%s\n" % (src, out))
        elif verbose and out.strip():
            sys.stderr.write(out)
    if failed:
        raise RuntimeError("libpmfem build failed")
    inc, libdir = nccl_dirs()
    link = [nvcc(), "-shared", "-o", lib] + objs + ARCH + ["-Xcompiler", "-fopenmp", "-lgomp", "-L", libdir,
                                                           "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stdout.decode())
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
