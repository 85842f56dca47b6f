"""In-tree build of the native pieces (run by __graft_entry__.build()).

* ``libnnb.so``  -- the C-ABI runtime (csrc/nnb_runtime.cpp), plain g++;
  libcuda and libnvrtc are dlopen'ed at run time.
* ahead-of-time check of the kernel headers with nvcc for sm_100a
  (``-gencode arch=compute_100a,code=sm_100a -lineinfo``) on the
  specialisations of BASELINE config 0, written to build/kcheck.cubin.  At run
  time the same headers are compiled by NVRTC inside libnnb.so with the
  shapes of the network being compiled.
The CPU checker under oracle/ (test infrastructure) is built by
__graft_entry__.build(), not by the package.

``python -m paper_1906_05737_b200.build`` runs both.
"""

import pathlib
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CUDA = pathlib.Path("/usr/local/cuda")
NVCC_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def build_runtime():
    out = PKG / "libnnb.so"
    src = PKG / "csrc" / "nnb_runtime.cpp"
    cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", "-Wno-unused-parameter",
           f"-I{CUDA / 'include'}", str(src), "-o", str(out), "-ldl", "-lpthread"]
    subprocess.check_call(cmd)
    return out


def kernel_check():
    """nvcc-compile the kernel templates for sm_100a with real instantiations."""
    sys.path.insert(0, str(ROOT))
    from paper_1906_05737_b200 import zoo
    from paper_1906_05737_b200.buffers import plan_buffers
    from paper_1906_05737_b200.graph import build_graph
    from paper_1906_05737_b200.kernels import specialize
    from paper_1906_05737_b200.options import ApproximationOptions
    from paper_1906_05737_b200.planner import build_plan

    m, w = zoo.build(0)
    plan = build_plan(build_graph(m, w))
    spec = specialize(plan, plan_buffers(plan), ApproximationOptions(), 64, 64)
    bdir = ROOT / "build"
    bdir.mkdir(exist_ok=True)
    cu = bdir / "kcheck.cu"
    cu.write_text(spec.source)
    out = bdir / "kcheck.cubin"
    cmd = [str(CUDA / "bin" / "nvcc"), *NVCC_ARCH, "-lineinfo", "-O3", "-std=c++17", "-cubin",
           f"-I{PKG / 'csrc' / 'kernels'}", "-Xptxas", "-v", str(cu), "-o", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc kernel check failed:\n" + r.stderr[-4000:])
    (bdir / "kcheck.ptxas.txt").write_text(r.stderr)
    return out


def main():
    print("runtime:", build_runtime())
    print("kernels:", kernel_check())


if __name__ == "__main__":
    main()
