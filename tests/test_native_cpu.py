"""The C ABI without a GPU: libnnb.so loads, exports every symbol declared in
include/nnb.h, reports a clean status instead of crashing, and its NVRTC
path produces sm_100a cubins.  Also guards the product path against any
dependency on the oracle."""
import ctypes
import pathlib
import re
import subprocess

import numpy as np
import pytest

from paper_1906_05737_b200 import _native, zoo
from paper_1906_05737_b200.buffers import plan_buffers
from paper_1906_05737_b200.graph import build_graph
from paper_1906_05737_b200.kernels import specialize
from paper_1906_05737_b200.options import ApproximationOptions
from paper_1906_05737_b200.planner import build_plan

ROOT = pathlib.Path(__file__).resolve().parent.parent


def header_functions():
    text = (ROOT / "include" / "nnb.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:nnb_status|void|const char \*|int32_t)\s*\*?\s*"
                                 r"(nnb_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    declared = header_functions()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native.EXPORTED)
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)],
                        capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}\b", nm), name


def test_abi_version_and_error_mapping_without_gpu():
    lib = _native.lib()
    assert lib.nnb_abi_version() == 6
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is present")
    with pytest.raises(_native.UnsupportedDevice):
        _native.device_check(0)
    assert lib.nnb_last_error()


def test_bad_arguments_fail_cleanly():
    lib = _native.lib()
    assert lib.nnb_create(None, None) == _native.NNB_ERR_ARGUMENT
    assert lib.nnb_apply(None, 1, None) == _native.NNB_ERR_ARGUMENT
    assert lib.nnb_compile(None, None, None, None, None, None) == _native.NNB_ERR_ARGUMENT


def test_compiled_network_requires_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1906_05737_b200 import UnsupportedDevice, compile_model
    m, w = zoo.build(1)
    with pytest.raises(UnsupportedDevice):
        compile_model(m, w)


def test_nvrtc_builds_sm100a_cubin(tmp_path):
    m, w = zoo.build(0)
    plan = build_plan(build_graph(m, w))
    spec = specialize(plan, plan_buffers(plan), ApproximationOptions(), 1, 16, mega=True)
    cubin, ms = _native.compile_source(spec.source, cache_dir=str(tmp_path))
    assert cubin[:4] == b"\x7fELF"
    p = tmp_path / "k.cubin"
    p.write_bytes(cubin)
    out = subprocess.run(["cuobjdump", "-elf", str(p)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for name in spec.kernel_names:
        if name != "nnb_mega":
            assert name.encode() in cubin
    # the batch-1 persistent kernel is its own translation unit (NNB_MEGA=1)
    assert "nnb_mega" in spec.kernel_names and spec.mega_source
    mega, _ = _native.compile_source(spec.mega_source, cache_dir=str(tmp_path))
    assert b"nnb_mega" in mega
    again, ms2 = _native.compile_source(spec.source, cache_dir=str(tmp_path))
    assert again == cubin                       # served from the cubin cache
    assert list(tmp_path.glob("*.cubin"))


def test_nvrtc_reports_compile_errors():
    from paper_1906_05737_b200.errors import CompileError
    with pytest.raises(CompileError, match="NVRTC"):
        _native.compile_source('#include "nnb_kernels.cuh"\nthis is not cuda;\n')


def test_product_path_never_touches_the_oracle():
    pkg = ROOT / "paper_1906_05737_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cpp")) + list(pkg.rglob("*.cuh")):
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text, f
        assert "nnoracle" not in text, f


def test_specialisation_is_deterministic():
    m, w = zoo.build(2)
    plan = build_plan(build_graph(m, w))
    a = specialize(plan, plan_buffers(plan), ApproximationOptions(), 8, 16)
    b = specialize(plan, plan_buffers(plan), ApproximationOptions(), 8, 16)
    assert a.source == b.source and a.pool == b.pool
