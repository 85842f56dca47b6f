"""Pin the CPU oracle (oracle/nnoracle.c) before trusting it.

* against the reference interpreter's outputs recorded in tests/golden
  (bit-exact: the oracle restates interpreter.py's per-op float32 order);
* against the reference's approximation models on a fixed grid (bit-exact);
* against the reference's compiled x86 path (oracle B) under the same
  approximation options, to the FP32 tolerance;
* the ops the reference lacks (relu6, elu, channel softmax, GAP, zero
  padding, separable conv) against independent naive loops;
* known answers from the reference's own tests.
"""
import re

import numpy as np
import pytest

from golden_util import GOLDEN, load, names
from oracle import oracle
from paper_1906_05737_b200 import ApproximationOptions, build_graph

F32 = np.float32
ROOT = GOLDEN.parent.parent


@pytest.mark.parametrize("name", names())
def test_oracle_matches_reference_interpreter_bit_exact(name):
    m, w, x, rec = load(name)
    got = oracle.run(m, w, [x], "exact")[0]
    want = rec["interp"]
    assert got.shape == want.shape
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("name", names())
@pytest.mark.parametrize("tag,opts", [
    ("compiled_default", ApproximationOptions()),
    ("compiled_precise", ApproximationOptions(softmax_exp="precise")),
    ("compiled_fast", ApproximationOptions(activation_mode="fast"))])
def test_oracle_models_match_reference_compiled_path(name, tag, opts):
    m, w, x, rec = load(name)
    got = oracle.run(m, w, [x], opts)[0]
    np.testing.assert_allclose(got, rec[tag], rtol=1e-4, atol=1e-5)


def test_approx_models_bit_exact_on_grid():
    g = dict(np.load(GOLDEN / "approx.npz"))
    L = oracle.lib()
    x = g["x"]
    for key, fn in (("tanh_rational", L.nno_tanh_rational),
                    ("sigmoid_rational", L.nno_sigmoid_rational),
                    ("tanh_fast", L.nno_tanh_fast), ("sigmoid_fast", L.nno_sigmoid_fast),
                    ("exp_fast", L.nno_exp_fast), ("exp_precise", L.nno_exp_precise)):
        got = np.array([fn(float(v)) for v in x], F32)
        np.testing.assert_array_equal(got.view(np.uint32), g[key].astype(F32).view(np.uint32),
                                      err_msg=key)


def test_device_constants_match_reference_models():
    """The float32 bit patterns baked into nnb_common.cuh are the reference's."""
    g = dict(np.load(GOLDEN / "approx.npz"))
    hdr = (ROOT / "paper_1906_05737_b200/csrc/kernels/nnb_common.cuh").read_text()
    consts = dict(re.findall(r"#define (NNB_\w+)\s+(0x[0-9a-f]+)u", hdr))
    assert int(consts["NNB_PADE_CLAMP"], 16) == int(g["pade_at_clamp"].view(np.uint32)[0])
    assert int(consts["NNB_SAT_DELTA"], 16) == int(g["sat_delta"].view(np.uint32)[0])
    bias = int(re.search(r"#define NNB_EXP_BIAS\s+(\d+)", hdr).group(1))
    assert bias == (127 << 23) - 366000
    as_bits = lambda v: int(np.array(F32(v)).view(np.uint32))
    assert int(consts["NNB_EXP_A"], 16) == as_bits(12102203.161561485)
    assert int(consts["NNB_TANH_CLAMP"], 16) == as_bits(5.7)
    assert int(consts["NNB_LN2_LO"], 16) == as_bits(np.log(np.float64(2.0)) - 0.693359375)
    for i, c in enumerate((1 / 5040, 1 / 720, 1 / 120, 1 / 24, 1 / 6)):
        assert int(consts[f"NNB_P{i}"], 16) == as_bits(c)


# -- known answers (pkg/tests/test_approx_models.py, test_interpreter.py) --------

def test_known_answers_approx():
    L = oracle.lib()
    assert abs(L.nno_tanh_rational(1.0) - 2304261 / 3025576) <= 1e-6
    for v in (5.7, 6.0, 10.0, 100.0, 3.0e38):
        assert L.nno_tanh_rational(v) == 1.0 and L.nno_tanh_rational(-v) == -1.0
    assert L.nno_sigmoid_rational(0.0) == 0.5
    xs = np.linspace(-80, 80, 20001).astype(F32)
    fe = np.array([L.nno_exp_fast(float(v)) for v in xs])
    assert np.all(np.diff(fe) >= 0) and np.all(fe > 0)
    rel = np.abs(fe - np.exp(xs.astype(np.float64))) / np.exp(xs.astype(np.float64))
    assert rel.max() <= 0.06
    pe = np.array([L.nno_exp_precise(float(v)) for v in xs])
    assert (np.abs(pe - np.exp(xs.astype(np.float64))) / np.exp(xs.astype(np.float64))).max() <= 1e-6
    t = np.linspace(-5, 5, 4001).astype(F32)
    tr = np.array([L.nno_tanh_rational(float(v)) for v in t])
    assert np.abs(tr - np.tanh(t.astype(np.float64))).max() <= 1e-4


def test_avg_pool_same_divides_by_valid_count():
    x = np.ones((1, 3, 3, 1), F32)
    y = oracle.pool(x, 3, 3, 1, "same", avg=True)
    np.testing.assert_array_equal(y, np.ones_like(y))
    x = np.arange(9, dtype=F32).reshape(1, 3, 3, 1)
    y = oracle.pool(x, 2, 2, 1, "same", avg=True)
    assert y[0, 2, 2, 0] == 8.0 and y[0, 0, 0, 0] == F32((0 + 1 + 3 + 4) / 4)


def test_bn_fold_known_answer():
    """gamma=2, beta=0.5, mean=3, var=4 (eps 0): scale 1, offset -2.5
    (pkg/keras-exporter/tests/test_export.py:162-184), folded in float64 by the
    zoo exactly like the exporter."""
    gamma, beta, mean, var = 2.0, 0.5, 3.0, 4.0
    scale = gamma / np.sqrt(var + 0.0)
    offset = beta - mean * scale
    assert (scale, offset) == (1.0, -2.5)
    x = np.array([0.0, 1.0, -2.0, 10.0], F32)
    s, o = np.full(4, scale, F32), np.full(4, offset, F32)
    y = np.empty_like(x)
    oracle.lib().nno_affine(oracle._p(x), oracle._p(y), oracle.ctypes.c_long(4), oracle._p(s),
                            oracle._p(o), 4)
    np.testing.assert_array_equal(y, [-2.5, -1.5, -4.5, 7.5])


# -- extensions vs naive loops ----------------------------------------------------

def test_relu6_and_elu_naive():
    x = np.linspace(-9, 9, 1001).astype(F32)
    np.testing.assert_array_equal(oracle.activation(x, "relu6"),
                                  np.array([min(max(v, F32(0)), F32(6)) for v in x], F32))
    want = np.array([v if v > 0 else F32(np.expm1(np.float64(v))) for v in x], F32)
    np.testing.assert_array_equal(oracle.activation(x, "elu"), want)


def test_channel_softmax_naive():
    rng = np.random.default_rng(3)
    x = rng.normal(0, 3, (2, 4, 5, 3)).astype(F32)
    got = oracle.softmax(x)
    for idx in np.ndindex(x.shape[:-1]):
        v = x[idx].astype(np.float64)
        e = np.exp(v - float(x[idx].max()))
        np.testing.assert_array_equal(got[idx], (e / e.sum()).astype(F32))


def test_gap_zeropad_separable_naive():
    from paper_1906_05737_b200.zoo import NetBuilder
    rng = np.random.default_rng(4)
    b = NetBuilder(seed=9)
    x = b.input((5, 6, 4))
    p = b.layer("ZeroPadding2D", [x], {"padding": [[1, 2], [0, 1]]})
    s = b.layer("SeparableConv2D", [p], {"filters": 3, "kernel_size": 3, "padding": "same",
                                         "activation": "relu"},
                [("depthwise", rng.normal(size=(3, 3, 4)).astype(F32)),
                 ("pointwise", rng.normal(size=(1, 1, 4, 3)).astype(F32)),
                 ("bias", rng.normal(size=3).astype(F32))])
    b.layer("GlobalAveragePooling2D", [s])
    m, w = b.build([b.layers[-1]["name"]])
    xin = rng.normal(size=(2, 5, 6, 4)).astype(F32)
    got = oracle.run(m, w, [xin])[0]
    dk, pk, bias = (w[f"{s}.depthwise"], w[f"{s}.pointwise"], w[f"{s}.bias"])
    for n in range(2):
        xp = np.zeros((8, 7, 4), F32)
        xp[1:6, 0:6] = xin[n]
        xq = np.zeros((10, 9, 4), F32)
        xq[1:9, 1:8] = xp
        dw = np.zeros((8, 7, 4), F32)
        for yy in range(8):
            for xx in range(7):
                acc = np.zeros(4, F32)
                for ky in range(3):
                    for kx in range(3):
                        acc = acc + xq[yy + ky, xx + kx] * dk[ky, kx]
                dw[yy, xx] = acc
        pw = np.empty((8, 7, 3), F32)
        for yy in range(8):
            for xx in range(7):
                acc = bias.copy()
                for c in range(4):
                    acc = acc + dw[yy, xx, c] * pk[0, 0, c]
                pw[yy, xx] = np.maximum(acc, 0)
        acc = np.zeros(3, F32)
        for yy in range(8):
            for xx in range(7):
                acc = acc + pw[yy, xx]
        np.testing.assert_array_equal(got[n], acc / F32(56))


def test_oracle_batch_axis_is_numerically_inert():
    m, w, x, rec = load("mixed_net")
    whole = oracle.run(m, w, [x])[0]
    for i in range(len(x)):
        np.testing.assert_array_equal(oracle.run(m, w, [x[i:i + 1]], threads=1)[0][0], whole[i])
