"""Host-buffer validation of run_host (CompiledNetwork and PipelinedNetwork)
before raw pointers cross the C ABI (short inputs read past the
host buffer; wrong-size / float64 / strided outputs were overwritten)."""
import numpy as np
import pytest

from paper_1906_05737_b200 import InputShapeMismatch
from paper_1906_05737_b200.runtime import _host_buffers

F32 = np.float32


def test_inputs_are_converted_and_checked():
    x = np.zeros((8, 4, 4, 3), np.float64)
    (got,) = _host_buffers([x], [(4, 4, 3)], 8, "input")
    assert got.dtype == F32 and got.flags.c_contiguous
    same = np.zeros((8, 4, 4, 3), F32)
    assert _host_buffers([same], [(4, 4, 3)], 8, "input")[0] is same
    with pytest.raises(InputShapeMismatch, match="does not match"):
        _host_buffers([np.zeros((7, 4, 4, 3), F32)], [(4, 4, 3)], 8, "input")   # too few images
    with pytest.raises(InputShapeMismatch, match="does not match"):
        _host_buffers([np.zeros((8, 4, 3, 3), F32)], [(4, 4, 3)], 8, "input")
    with pytest.raises(InputShapeMismatch, match="expected 1 inputs"):
        _host_buffers([same, same], [(4, 4, 3)], 8, "input")


def test_outputs_must_be_writable_float32_contiguous_and_large_enough():
    ok = np.zeros((8, 10), F32)
    _host_buffers([ok], [(10,)], 8, "output", writable=True)
    _host_buffers([np.zeros((9, 10), F32)], [(10,)], 8, "output", writable=True)
    bad = [np.zeros((7, 10), F32),                         # fewer rows than n
           np.zeros((8, 10), np.float64),                  # dtype
           np.zeros((8, 20), F32)[:, ::2],                 # strided
           np.zeros((8, 11), F32)]                         # per-image shape
    ro = np.zeros((8, 10), F32)
    ro.flags.writeable = False
    bad.append(ro)
    for b in bad:
        with pytest.raises(InputShapeMismatch):
            _host_buffers([b], [(10,)], 8, "output", writable=True)
    with pytest.raises(InputShapeMismatch):
        _host_buffers([[0.0] * 10], [(10,)], 1, "output", writable=True)


def test_unbatched_network_takes_per_image_arrays():
    _host_buffers([np.zeros((4, 4, 3), F32)], [(4, 4, 3)], 1, "input", batched=False)
    with pytest.raises(InputShapeMismatch):
        _host_buffers([np.zeros((1, 4, 4, 3), F32)], [(4, 4, 3)], 1, "input", batched=False)
