"""Build the checkers under oracle/ (TEST INFRASTRUCTURE ONLY).

Two artefacts, neither of which is part of the product path:

1. ``oracle/libdynlp_oracle.so`` -- the plain-C restatement of the
   reference DynLP batch update (oracle/dynlp_oracle.c).
2. ``oracle/_ref/dynlp/`` -- the *unmodified* reference package compiled
   from its sources where they lie under /root/reference: every module is
   translated by Cython and compiled by gcc into an extension module, and the
   native kernel ``kernels/_csr.pyx`` is built with ``-O3 -fopenmp`` exactly as
   the reference's setup.py does (pkg/setup.py:11-19).  Only binaries land in
   oracle/_ref (git-ignored, not gpurun-ignored), so the real reference
   travels to the GPU box for the CPU baseline and for pinning the
   restatement, without any reference source entering the repository.

The reference is optional here: when /root/reference is absent (the GPU box)
only step 1 runs and a previously built oracle/_ref is used as-is.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src/dynlp"
REF_OUT = os.path.join(HERE, "_ref")
GCC = "/usr/bin/gcc"  # /opt/gcc lacks libgomp.spec

MODULES = [
    "__init__", "errors", "graph", "labels", "components", "engine", "stream",
    "builder", "baselines", "harness", "cli",
    "kernels/__init__", "kernels/_py", "kernels/_ragged",
]


def _run(cmd, **kw):
    r = subprocess.run(cmd, capture_output=True, text=True, **kw)
    if r.returncode != 0:
        raise RuntimeError(f"command failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r


def build_oracle(force: bool = False) -> str:
    src = os.path.join(HERE, "dynlp_oracle.c")
    out = os.path.join(HERE, "libdynlp_oracle.so")
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(HERE, "dynlp_oracle.h"))
    ):
        return out
    # -ffp-contract=off and no -march: the reference's compiled kernel uses
    # plain SSE2 mulsd/addsd (no FMA); the restatement must round the same way.
    _run([GCC, "-O3", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
          "-D_POSIX_C_SOURCE=200809L", src, "-o", out + ".tmp", "-lm"])
    os.replace(out + ".tmp", out)
    return out


def _ext_suffix() -> str:
    return sysconfig.get_config_var("EXT_SUFFIX")


def build_reference(force: bool = False) -> str | None:
    """Cython-compile the reference package into oracle/_ref/dynlp (binaries only)."""
    if not os.path.isdir(REF_SRC):
        return REF_OUT if os.path.isdir(os.path.join(REF_OUT, "dynlp")) else None
    stamp = os.path.join(REF_OUT, ".built")
    if not force and os.path.exists(stamp):
        return REF_OUT
    import numpy

    tmp = os.path.join(REF_OUT, "_csrc")  # generated C, removed after compiling
    os.makedirs(tmp, exist_ok=True)
    pyinc = sysconfig.get_paths()["include"]
    npinc = numpy.get_include()
    suf = _ext_suffix()
    jobs = []
    for m in MODULES:
        pkg = "dynlp." + m.replace("/", ".")
        if pkg.endswith(".__init__"):
            pkg = pkg[: -len(".__init__")]
        c_file = os.path.join(tmp, m.replace("/", "__") + ".c")
        so = os.path.join(REF_OUT, "dynlp", m + suf)
        jobs.append((["cython", "-3", "--module-name", pkg, os.path.join(REF_SRC, m + ".py"),
                      "-o", c_file], c_file, so, ["-O2"]))
    c_csr = os.path.join(tmp, "kernels___csr.c")
    jobs.append((["cython", "-3", "--module-name", "dynlp.kernels._csr",
                  os.path.join(REF_SRC, "kernels", "_csr.pyx"), "-o", c_csr], c_csr,
                 os.path.join(REF_OUT, "dynlp", "kernels", "_csr" + suf),
                 ["-O3", "-fopenmp", "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION"]))

    def one(job):
        cy, c_file, so, flags = job
        _run([sys.executable, "-m", "cython"] + cy[1:])
        os.makedirs(os.path.dirname(so), exist_ok=True)
        _run([GCC, "-shared", "-fPIC", *flags, f"-I{pyinc}", f"-I{npinc}", c_file, "-o", so,
              "-fopenmp"])

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(one, jobs))
    shutil.rmtree(tmp, ignore_errors=True)
    with open(stamp, "w") as fh:
        fh.write("compiled from " + REF_SRC + "\n")
    return REF_OUT


def reference_path() -> str | None:
    """Directory to put on sys.path to import the compiled reference, if built."""
    if os.path.exists(os.path.join(REF_OUT, ".built")):
        return REF_OUT
    return None


if __name__ == "__main__":
    print(build_oracle(force="--force" in sys.argv))
    print(build_reference(force="--force" in sys.argv))
