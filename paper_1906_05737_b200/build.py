"""In-tree build of the native pieces (run by __graft_entry__.build()).

* ``libnnb.so``  -- the C-ABI runtime (csrc/nnb_runtime.cpp), plain g++;
  libcuda and libnvrtc are dlopen'ed at run time.
* ahead-of-time check of the kernel headers with nvcc for sm_100a
  (``-gencode arch=compute_100a,code=sm_100a -lineinfo``) on the
  specialisations of every BASELINE config, written to build/kcheck_cfg*.cubin.  At run
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


def kernel_check(configs=range(5), batch=4096):
    """nvcc-compile the kernel templates for sm_100a with real instantiations:
    every unit of each zoo config at ``batch`` (SIMT, direct and tcgen05
    variants), one translation unit per config, compiled in parallel."""
    sys.path.insert(0, str(ROOT))
    from paper_1906_05737_b200 import zoo
    from paper_1906_05737_b200.buffers import plan_buffers
    from paper_1906_05737_b200.graph import build_graph
    from paper_1906_05737_b200.kernels import specialize
    from paper_1906_05737_b200.options import ApproximationOptions
    from paper_1906_05737_b200.planner import build_plan

    bdir = ROOT / "build"
    bdir.mkdir(exist_ok=True)
    jobs = []
    for c in configs:
        m, w = zoo.build(c)
        g = build_graph(m, w)
        plan = build_plan(g)
        spec = specialize(plan, plan_buffers(plan, reserve_heads=True), ApproximationOptions(), batch,
                          batch)
        tus = [(f"cfg{c}", spec.source)]
        # the batch-1 persistent kernel's own TU (over the plan without the
        # depthwise fusion, as CompiledNetwork(mega=True) builds it)
        plan = build_plan(g, dw_fusion=False)
        spec = specialize(plan, plan_buffers(plan), ApproximationOptions(), batch, batch, mega=True)
        if spec.mega_source:
            tus.append((f"cfg{c}_mega", spec.mega_source))
        for tag, text in tus:
            cu = bdir / f"kcheck_{tag}.cu"
            cu.write_text(text)
            out = bdir / f"kcheck_{tag}.cubin"
            cmd = [str(CUDA / "bin" / "nvcc"), *NVCC_ARCH, "-lineinfo", "-O3", "-std=c++17",
                   "-cubin", f"-I{PKG / 'csrc' / 'kernels'}", "-Xptxas", "-v", str(cu), "-o", str(out)]
            jobs.append((tag, out, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                    stderr=subprocess.PIPE, text=True)))
    outs = []
    for tag, out, p in jobs:
        _, err = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc kernel check ({tag}) failed:\n" + err[-4000:])
        (bdir / f"kcheck_{tag}.ptxas.txt").write_text(err)
        outs.append(out)
    return outs


def main():
    print("runtime:", build_runtime())
    print("kernels:", kernel_check())


if __name__ == "__main__":
    main()
