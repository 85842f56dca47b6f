"""GPU kernel sweeps through the public API vs the C oracle (cf. the reference's
pkg/tests/test_emitters.py): irregular shapes, ragged channel vectors, clipped
windows, every fused epilogue, the tcgen05 paths, bit-exact kinds, the
approximation modes, and the runtime API contract."""
import numpy as np
import pytest

from builders import bn_params, conv_net, dense_net, he, random_network
from golden_util import GOLDEN, load, names
from oracle import oracle
from paper_1906_05737_b200 import (EXACT, ApproximationOptions, InputShapeMismatch,
                                   build_graph, compile_model, zoo)
from paper_1906_05737_b200.planner import sep_narrow_geometry
from paper_1906_05737_b200.zoo import NetBuilder

pytestmark = pytest.mark.gpu
F32 = np.float32
TOL = dict(rtol=1e-4, atol=1e-5)


def gpu(m, w, x, opts=EXACT, **kw):
    net = compile_model(m, w, opts, batch=len(x), tuning=kw or None)
    return net.run([x])[0].cpu().numpy(), net


def ref(m, w, x, opts="exact"):
    return oracle.run(m, w, [x], opts)[0]


@pytest.mark.parametrize("h,w,ci,co,k,s,pad,act", [
    (7, 9, 3, 5, 3, 1, "same", "relu"), (8, 6, 4, 8, 3, 2, "same", "tanh"),
    (5, 5, 2, 3, 2, 1, "valid", "sigmoid"), (9, 7, 1, 4, 3, 2, "valid", "linear"),
    (6, 6, 5, 7, 1, 1, "valid", "relu6"), (10, 12, 8, 16, 3, 1, "same", "elu"),
    (11, 13, 16, 33, 5, 2, "same", "relu"), (4, 4, 64, 64, 1, 1, "valid", "tanh")])
@pytest.mark.parametrize("n", [1, 5])
def test_conv_sweep(h, w, ci, co, k, s, pad, act, n):
    rng = np.random.default_rng(h * 100 + co)
    m, wt = conv_net(rng, h, w, ci, co, k=k, stride=s, padding=pad, act=act)
    x = rng.uniform(-2, 2, (n, h, w, ci)).astype(F32)
    got, _ = gpu(m, wt, x)
    np.testing.assert_allclose(got, ref(m, wt, x), **TOL)


@pytest.mark.parametrize("h,w,ci,co,pad,pool,n", [
    (10, 18, 32, 16, "same", False, 3), (17, 23, 32, 48, "same", True, 2),
    (12, 40, 64, 32, "valid", True, 2), (9, 16, 32, 40, "same", False, 1),
    (60, 80, 32, 64, "same", True, 2), (14, 20, 16, 32, "same", False, 2),
    (11, 30, 16, 16, "same", True, 2), (9, 12, 48, 32, "valid", False, 2),
    (14, 20, 32, 64, "same", False, 2), (10, 37, 64, 64, "valid", False, 3)])
def test_tensor_core_conv3x3(h, w, ci, co, pad, pool, n):
    """Implicit-GEMM tcgen05 conv (4-D TMA boxes, zero-filled borders), with
    and without the fused 2x2 max-pool epilogue, ragged 8x16 tiles; CO = 16
    (all taps in N), 32 (KW taps in N = 96) and 64 (KW taps in N = 192)."""
    rng = np.random.default_rng(ci + co + h)
    b = NetBuilder()
    x = b.input((h, w, ci))
    y = b.layer("Conv2D", [x], {"filters": co, "kernel_size": 3, "padding": pad,
                                "activation": "relu"},
                [("kernel", he(rng, (3, 3, ci, co), 9 * ci)),
                 ("bias", (rng.standard_normal(co) * 0.1).astype(F32))])
    if pool:
        y = b.layer("MaxPool2D", [y], {"pool_size": 2, "strides": 2})
    m, wt = b.build([y])
    xin = rng.uniform(-2, 2, (n, h, w, ci)).astype(F32)
    got, net = gpu(m, wt, xin, tc_min_rows=1, tc_tile_use=0, direct_imm=False)
    assert any("_tc_" in l.kernel for l in net.artifact.launches)
    np.testing.assert_allclose(got, ref(m, wt, xin), **TOL)


@pytest.mark.parametrize("c0,c1,co,up_src,tc", [
    (64, 64, 32, "pool", True), (32, 32, 16, "conv", True), (8, 12, 16, "conv", False),
    (4, 8, 8, "pool", False), (32, 64, 48, "conv", False), (16, 16, 32, "conv", True)])
def test_decoder_fusions(c0, c1, co, up_src, tc):
    """UpSample2D fused into its producer's epilogue (pool / direct / FFMA /
    tcgen05 conv) and Concatenate fused into the consumer conv's loader."""
    rng = np.random.default_rng(c0 + c1 + co)
    h, w = 6, 10
    b = NetBuilder()
    x = b.input((2 * h, 2 * w, c1))
    if up_src == "pool":
        lo = b.layer("MaxPool2D", [x], {"pool_size": 2, "strides": 2})
        lo = b.layer("Conv2D", [lo], {"filters": c0, "kernel_size": 1, "activation": "relu"},
                     [("kernel", he(rng, (1, 1, c1, c0), c1)), ("bias", np.zeros(c0, F32))])
        lo = b.layer("MaxPool2D", [b.layer("UpSample2D", [lo], {"factor": 2})],
                     {"pool_size": 1, "strides": 1})
        up = b.layer("UpSample2D", [b.layer("MaxPool2D", [lo], {"pool_size": 2, "strides": 2})],
                     {"factor": 2})
    else:
        lo = b.layer("AvgPool2D", [x], {"pool_size": 2, "strides": 2})
        lo = b.layer("Conv2D", [lo], {"filters": c0, "kernel_size": 3, "padding": "same",
                                      "activation": "tanh"},
                     [("kernel", he(rng, (3, 3, c1, c0), 9 * c1)), ("bias", np.zeros(c0, F32))])
        up = b.layer("UpSample2D", [lo], {"factor": 2})
    cat = b.layer("Concatenate", [up, x])
    y = b.layer("Conv2D", [cat], {"filters": co, "kernel_size": 3, "padding": "same",
                                  "activation": "relu"},
                [("kernel", he(rng, (3, 3, c0 + c1, co), 9 * (c0 + c1))),
                 ("bias", (rng.standard_normal(co) * 0.1).astype(F32))])
    m, wt = b.build([y])
    xin = rng.uniform(-2, 2, (3, 2 * h, 2 * w, c1)).astype(F32)
    got, net = gpu(m, wt, xin, tc_min_rows=1 if tc else 1 << 30, tc_tile_use=0)
    kinds = [u.kind for u in net.plan.units]
    assert "Concat" not in kinds and "Upsample" not in kinds, net.plan.describe()
    assert any("_tc_" in l.kernel for l in net.artifact.launches) == tc
    np.testing.assert_allclose(got, ref(m, wt, xin), **TOL)


@pytest.mark.parametrize("c0,c1,co,n", [(32, 32, 64, 64), (16, 48, 32, 40), (32, 32, 16, 3)])
def test_concat_into_pointwise(c0, c1, co, n):
    """Concatenate fused into a 1x1 conv's loader at batches above the
    tensor-core threshold (default selection): the row GEMM cannot read a
    two-source operand, so the conv tiles (second TMA map) or the SIMT loader
    serve it (a 1x1 conv fed by a concat went to the row GEMM)."""
    rng = np.random.default_rng(c0 * c1 + co + n)
    b = NetBuilder()
    x = b.input((16, 16, 4))
    a = b.layer("Conv2D", [x], {"filters": c0, "kernel_size": 3, "padding": "same",
                                "activation": "relu"},
                [("kernel", he(rng, (3, 3, 4, c0), 36)), ("bias", np.zeros(c0, F32))])
    bb = b.layer("Conv2D", [x], {"filters": c1, "kernel_size": 3, "padding": "same",
                                 "activation": "tanh"},
                 [("kernel", he(rng, (3, 3, 4, c1), 36)), ("bias", np.zeros(c1, F32))])
    cat = b.layer("Concatenate", [a, bb])
    y = b.layer("Conv2D", [cat], {"filters": co, "kernel_size": 1, "activation": "relu"},
                [("kernel", he(rng, (1, 1, c0 + c1, co), c0 + c1)),
                 ("bias", (rng.standard_normal(co) * 0.1).astype(F32))])
    m, wt = b.build([y])
    xin = rng.uniform(-2, 2, (n, 16, 16, 4)).astype(F32)
    got, net = gpu(m, wt, xin)
    assert "Concat" not in [u.kind for u in net.plan.units]
    # a tensor-core launch of the concat-fed conv must be the conv-tile form
    # (second TMA map), never the single-map row GEMM
    for l in net.artifact.launches:
        if "_tc_" in l.kernel:
            assert "conv tiles" in l.note and "concat (2 A maps)" in l.note, l.note
    np.testing.assert_allclose(got, ref(m, wt, xin), **TOL)


@pytest.mark.parametrize("h,w,c,co,k,s,pad,dwbias,res,n", [
    (9, 13, 8, 16, 3, 1, "same", False, False, 3), (16, 16, 16, 32, 3, 2, "same", True, False, 2),
    (64, 64, 8, 16, 3, 1, "same", False, False, 7), (30, 40, 16, 32, 3, 1, "same", False, False, 37),
    (17, 23, 12, 3, 5, 2, "same", True, False, 5), (11, 9, 4, 1, 3, 1, "valid", True, False, 4),
    (15, 20, 32, 32, 3, 1, "same", False, True, 9), (7, 130, 8, 8, 3, 1, "same", True, True, 2),
    (33, 31, 20, 24, 3, 2, "valid", False, False, 3), (1, 1, 16, 8, 3, 1, "same", True, False, 6),
    # many tiles per persistent CTA (the ring wraps)
    (64, 64, 8, 16, 3, 1, "same", False, False, 160), (64, 64, 16, 32, 3, 2, "same", False, False, 300),
    (32, 32, 32, 32, 3, 1, "same", False, False, 400), (30, 40, 16, 16, 3, 1, "same", False, True, 500),
    (64, 64, 16, 32, 3, 2, "same", False, False, 301)])
def test_sep_narrow(h, w, c, co, k, s, pad, dwbias, res, n):
    """Depthwise (+BN+act) fused with a pointwise conv of <= 32 channels
    (nnb_sep.cuh, default planner fusion): row-band tiles, ragged last band,
    clipped / valid windows, stride 2, a residual Add, tiny and huge widths;
    against the oracle and, with one K slice, bit-identical to the unfused
    depthwise kernel + pointwise GEMM."""
    rng = np.random.default_rng(h * w + c * co + k)
    b = NetBuilder()
    x = b.input((h, w, c))
    wt = [("kernel", he(rng, (k, k, c), k * k))]
    if dwbias:
        wt.append(("bias", (rng.standard_normal(c) * 0.1).astype(F32)))
    d = b.layer("DepthwiseConv2D", [x], {"kernel_size": k, "strides": s, "padding": pad,
                                         "use_bias": dwbias}, wt)
    d = b.layer("BatchNorm", [d], None, bn_params(rng, c))
    d = b.layer("Activation", [d], {"activation": "relu6"})
    y = b.layer("Conv2D", [d], {"filters": co, "kernel_size": 1, "activation": "tanh"},
                [("kernel", he(rng, (1, 1, c, co), c)),
                 ("bias", (rng.standard_normal(co) * 0.1).astype(F32))])
    if res:
        y = b.layer("Add", [y, x])
    m, wt = b.build([y])
    xin = rng.uniform(-2, 2, (n, h, w, c)).astype(F32)
    got, net = gpu(m, wt, xin)
    if len(net.plan.units) == 2:          # band too large for the fused kernel (stride 2)
        assert sep_narrow_geometry(*net.plan.units) is None and s == 2
    else:
        assert [l.kernel.split("_")[2] for l in net.artifact.launches] == [f"sep{k}x{k}"], \
            net.describe()
    np.testing.assert_allclose(got, ref(m, wt, xin), **TOL)
    if len(net.plan.units) == 1 and c % 8 == 0 and co % 8 == 0:
        # one and two threads per pixel (nnb_sep.cuh SP) form every output in
        # the same order: bit-identical
        geo = sep_narrow_geometry(net.plan.units[0].dw, net.plan.units[0])
        alt, net1 = gpu(m, wt, xin, sep_geo=(geo["TH"], geo["NS"], 3 - geo["SP"]))
        assert ("two threads per pixel" in net1.artifact.launches[0].note) == (geo["SP"] == 1)
        assert np.array_equal(alt, got)
    # (the tiled pointwise GEMM: the split-K row kernel of few-pixel 1x1
    # convs sums in another order)
    unf, net2 = gpu(m, wt, xin, dw_fusion=False, small_conv=False)
    assert len(net2.launches_for()) == 2
    np.testing.assert_allclose(got, unf, rtol=1e-5, atol=5e-6)   # FFMA vs mul+add taps
    if len(net.plan.units) == 1 and c < 32 and not any("_tc_" in l.kernel
                                                       for l in net2.artifact.launches):
        # the interpreter's mul-then-add depthwise taps: bit-identical to the
        # unfused depthwise kernel + pointwise GEMM
        exact, _ = gpu(m, wt, xin, sep_fma=False)
        np.testing.assert_array_equal(exact, unf)


@pytest.mark.parametrize("h,w,c,co,s,act,bn,n", [
    (9, 13, 8, 16, 1, "relu6", True, 3), (16, 16, 16, 32, 2, "relu", False, 2),
    (7, 10, 64, 128, 2, "elu", True, 2), (8, 8, 128, 96, 1, "linear", False, 5),
    (20, 35, 32, 64, 1, "relu6", True, 3), (33, 30, 16, 48, 2, "relu", True, 2)])
def test_depthwise_pointwise_fusion(h, w, c, co, s, act, bn, n):
    """DepthwiseConv2D (+BN+act) computed inside the pointwise conv's loader."""
    rng = np.random.default_rng(h * w + c)
    b = NetBuilder()
    x = b.input((h, w, c))
    d = b.layer("DepthwiseConv2D", [x], {"kernel_size": 3, "strides": s, "padding": "same",
                                         "use_bias": False},
                [("kernel", he(rng, (3, 3, c), 9))])
    if bn:
        d = b.layer("BatchNorm", [d], None, bn_params(rng, c))
    d = b.layer("Activation", [d], {"activation": act}) if act != "linear" else d
    y = b.layer("Conv2D", [d], {"filters": co, "kernel_size": 1, "activation": "relu"},
                [("kernel", he(rng, (1, 1, c, co), c)),
                 ("bias", (rng.standard_normal(co) * 0.1).astype(F32))])
    m, wt = b.build([y])
    xin = rng.uniform(-2, 2, (n, h, w, c)).astype(F32)
    got, net = gpu(m, wt, xin, dw_fusion=True)
    assert [u.kind for u in net.plan.units] == ["Conv2D"] and net.plan.units[0].dw is not None
    np.testing.assert_allclose(got, ref(m, wt, xin), **TOL)
    if c % 16 == 0 and co > 32:           # the tcgen05 form (halo TMA + fused split warps)
        got, net = gpu(m, wt, xin, dw_fusion=True, tc_min_rows=1, tc_tile_use=0)
        assert any("depthwise fused" in l.note for l in net.artifact.launches)
        np.testing.assert_allclose(got, ref(m, wt, xin), **TOL)


@pytest.mark.parametrize("k,units,act,n", [
    (1, 1, "linear", 1), (3, 5, "relu", 7), (17, 9, "tanh", 3), (130, 7, "sigmoid", 12),
    (64, 64, "elu", 2100), (256, 96, "relu6", 2048), (100, 40, "linear", 2500),
    (1024, 512, "tanh", 2049)])
def test_dense_sweep(k, units, act, n):
    rng = np.random.default_rng(k + units)
    m, w = dense_net(rng, k, units, act)
    x = rng.uniform(-2, 2, (n, k)).astype(F32)
    got, _ = gpu(m, w, x)
    np.testing.assert_allclose(got, ref(m, w, x), **TOL)
    if n > 8 and k % 4 == 0 and k >= 32 and units >= 32:     # force the tcgen05 path
        got, net = gpu(m, w, x, tc_min_rows=1)
        assert any("_tc_" in l.kernel for l in net.artifact.launches)
        np.testing.assert_allclose(got, ref(m, w, x), **TOL)


def _single(kind, shape, config=None, weights=()):
    b = NetBuilder()
    x = b.input(shape)
    y = b.layer(kind, [x], config, weights)
    return b.build([y])


@pytest.mark.parametrize("case", [
    ("DepthwiseConv2D", (7, 9, 3), {"kernel_size": 3, "padding": "same", "activation": "relu"}),
    ("DepthwiseConv2D", (8, 8, 8), {"kernel_size": 3, "strides": 2, "padding": "same"}),
    ("DepthwiseConv2D", (6, 5, 5), {"kernel_size": [2, 3], "padding": "valid"}),
    ("MaxPool2D", (7, 9, 3), {"pool_size": 2, "strides": 2, "padding": "same"}),
    ("AvgPool2D", (7, 9, 3), {"pool_size": 3, "strides": 2, "padding": "same"}),
    ("AvgPool2D", (6, 6, 4), {"pool_size": [2, 1], "strides": 1}),
    ("MaxPool2D", (5, 7, 8), {"pool_size": 3, "strides": 1, "padding": "same"}),
    ("GlobalAveragePooling2D", (8, 10, 12), None),
    ("UpSample2D", (3, 4, 5), {"factor": 3}), ("UpSample2D", (3, 4, 8), {"factor": 2}),
    ("ZeroPadding2D", (3, 4, 5), {"padding": [[1, 2], [0, 3]]}),
    ("Activation", (37,), {"activation": "relu"}), ("Activation", (5, 5, 4), {"activation": "relu6"}),
])
def test_bit_exact_kinds(case):
    kind, shape, cfg = case
    rng = np.random.default_rng(len(shape) + shape[-1])
    wts = ()
    if kind == "DepthwiseConv2D":
        kh, kw = (cfg["kernel_size"],) * 2 if isinstance(cfg["kernel_size"], int) else cfg["kernel_size"]
        wts = [("kernel", he(rng, (kh, kw, shape[-1]), kh * kw)),
               ("bias", (rng.standard_normal(shape[-1]) * 0.1).astype(F32))]
    m, w = _single(kind, shape, cfg, wts)
    x = rng.uniform(-2, 2, (4,) + shape).astype(F32)
    got, _ = gpu(m, w, x)
    np.testing.assert_array_equal(got, ref(m, w, x))


@pytest.mark.parametrize("shape", [(5,), (4, 5, 6), (3, 3, 3)])
def test_batchnorm_and_add_concat_bit_exact(shape):
    rng = np.random.default_rng(11)
    b = NetBuilder()
    x = b.input(shape)
    bn = b.layer("BatchNorm", [x], None, bn_params(rng, shape[-1]))
    r = b.layer("Activation", [x], {"activation": "relu"})
    t = b.layer("Activation", [x], {"activation": "relu6"})
    a = b.layer("Add", [bn, r, t])
    c = b.layer("Concatenate", [a, x, bn])
    m, w = b.build([c])
    xin = rng.uniform(-3, 3, (3,) + shape).astype(F32)
    got, _ = gpu(m, w, xin)
    np.testing.assert_array_equal(got, ref(m, w, xin))


@pytest.mark.parametrize("n", [1, 2, 33])
@pytest.mark.parametrize("smexp", ["fast", "precise", "exact"])
def test_softmax_rows_and_pixels(n, smexp):
    rng = np.random.default_rng(n)
    opts = ApproximationOptions(activation_mode="exact", softmax_exp=smexp)
    for shape in ((1000,), (33,), (2,), (6, 7, 3), (4, 4, 40)):
        m, w = _single("Softmax", shape)
        x = rng.normal(0, 4, (n,) + shape).astype(F32)
        got, _ = gpu(m, w, x, opts)
        np.testing.assert_allclose(got, ref(m, w, x, opts), rtol=1e-5, atol=1e-7)
        np.testing.assert_allclose(got.sum(-1), 1.0, rtol=1e-5)


@pytest.mark.parametrize("mode", ["rational", "fast"])
@pytest.mark.parametrize("tag", ["tanh", "sigmoid"])
def test_activation_kernels_bit_exact_vs_reference_models(mode, tag):
    """The device approximations equal the reference's numpy models bit for bit
    (tests/golden/approx.npz, pkg/src/nnjit/codegen/approx.py:72-128)."""
    g = dict(np.load(GOLDEN / "approx.npz"))
    xs = g["x"].astype(F32)
    m, w = _single("Activation", (len(xs),), {"activation": tag})
    got, _ = gpu(m, w, xs[None, :], ApproximationOptions(activation_mode=mode))
    np.testing.assert_array_equal(got[0].view(np.uint32),
                                  g[f"{tag}_{mode}"].astype(F32).view(np.uint32))


def test_exact_transcendentals_match_float64_rounding():
    """activation_mode='exact' reproduces the interpreter's float64 tanh /
    sigmoid / expm1 rounded to float32 on a dense grid."""
    xs = np.concatenate([np.linspace(-30, 30, 200001), [0.0, -0.0, 1e-30, -1e-30]]).astype(F32)
    for tag in ("tanh", "sigmoid", "elu"):
        m, w = _single("Activation", (len(xs),), {"activation": tag})
        got, _ = gpu(m, w, xs[None, :])
        want = oracle.activation(xs, tag)
        mismatch = np.count_nonzero(got[0] != want)
        assert mismatch <= 2, (tag, mismatch)


@pytest.mark.parametrize("units,n", [(32, 2048), (128, 512)])
@pytest.mark.parametrize("tag", ["tanh", "sigmoid", "elu"])
def test_exact_mode_in_tensor_core_epilogue(tag, units, n):
    """activation_mode='exact' is the interpreter's float64-rounded-once
    semantics in the tcgen05 epilogues too.  An identity
    Dense makes the 3xTF32 GEMM exact -- inputs on a 2^-14 grid in (-32, 32)
    have <= 20 significant bits, so a = a_hi + a_lo with both halves exact in
    TF32, b_lo = 0 -- and the epilogue's activation must then equal the
    interpreter's rounding of tanh / sigmoid / expm1 of the input."""
    xs = np.linspace(-30, 30, n * units)
    xs = (np.round(xs * 2 ** 14) / 2 ** 14).astype(F32).reshape(n, units)
    b = NetBuilder()
    x = b.input((units,))
    y = b.layer("Dense", [x], {"units": units, "activation": tag},
                [("kernel", np.eye(units, dtype=F32)), ("bias", np.zeros(units, F32))])
    m, w = b.build([y])
    got, net = gpu(m, w, xs, tc_min_rows=1)
    assert any("_tc_" in l.kernel and l.n_min <= n <= l.n_max for l in net.artifact.launches)
    want = oracle.activation(xs, tag)
    mismatch = np.count_nonzero(got != want)
    assert mismatch <= 2, (tag, mismatch, np.abs(got - want).max())


@pytest.mark.parametrize("name", names())
def test_golden_nets_vs_reference(name):
    """Against the REAL reference's recorded outputs: interpreter (exact mode)
    and compiled x86 path (its default and precise options)."""
    m, w, x, rec = load(name)
    got, _ = gpu(m, w, x)
    np.testing.assert_allclose(got, rec["interp"], **TOL)
    got, _ = gpu(m, w, x, ApproximationOptions())
    np.testing.assert_allclose(got, rec["compiled_default"], **TOL)
    got, _ = gpu(m, w, x, ApproximationOptions(softmax_exp="precise"))
    np.testing.assert_allclose(got, rec["compiled_precise"], **TOL)


def test_random_networks():
    rng = np.random.default_rng(99)
    for trial in range(12):
        m, w, shape = random_network(rng)
        x = rng.uniform(-2, 2, (3,) + shape).astype(F32)
        got, _ = gpu(m, w, x)
        np.testing.assert_allclose(got, ref(m, w, x), rtol=2e-4, atol=2e-5,
                                   err_msg=f"trial {trial}")


# -- runtime API contract ----------------------------------------------------------

def test_views_stable_apply_idempotent_and_partial_batch():
    m, w = zoo.build(2)
    net = compile_model(m, w, EXACT, batch=6)
    x = zoo.inputs(2, 6)
    out1 = net.run([x])
    first = out1[0].clone()
    assert out1[0] is net.output_views[0] and net.run([x])[0] is out1[0]
    net.apply()                                  # inputs are pinned: same result
    np.testing.assert_array_equal(net.output_views[0].cpu().numpy(), first.cpu().numpy())
    want = ref(m, w, x)
    np.testing.assert_allclose(first.cpu().numpy(), want, **TOL)
    net.output_views[0].zero_()
    net.run([x[:2]])                             # apply over the first 2 images only
    got = net.output_views[0].cpu().numpy()      # rows >= 2 are undefined after apply(2)
    np.testing.assert_allclose(got[:2], want[:2], **TOL)
    host = net.run_host([x])[0]
    np.testing.assert_allclose(host, want, **TOL)


def test_unbatched_views_have_reference_shapes():
    m, w = zoo.build(0)
    net = compile_model(m, w, EXACT)
    assert tuple(net.input_views[0].shape) == (32, 32, 1)
    assert tuple(net.output_views[0].shape) == (2,)
    x = zoo.inputs(0, 1)[0]
    net.input_views[0].copy_(__import__("torch").from_numpy(x))
    net.apply()
    np.testing.assert_allclose(net.output_views[0].cpu().numpy(), ref(m, w, x[None])[0], **TOL)
    assert "units" in net.describe() and net.compile_ms > 0


def test_errors():
    m, w = zoo.build(1)
    net = compile_model(m, w, EXACT, batch=4)
    with pytest.raises(InputShapeMismatch):
        net.run([np.zeros((4, 1000), F32)])
    with pytest.raises(InputShapeMismatch):
        net.run([np.zeros((5, 1024), F32)])
    with pytest.raises(InputShapeMismatch):
        net.run([])
    with pytest.raises(InputShapeMismatch):
        net.apply(5)
    with pytest.raises(InputShapeMismatch):            # nnb_time_apply range check
        net.time_apply(5)
    # host buffers are validated before their pointers reach the C ABI
    with pytest.raises(InputShapeMismatch):
        net.run_host([np.zeros((3, 1024), F32)])
    with pytest.raises(InputShapeMismatch):
        net.run_host([np.zeros((4, 1024), F32)], [np.zeros((4, 10), np.float64)])
    with pytest.raises(InputShapeMismatch):
        net.run_host([np.zeros((4, 1024), F32)], [np.zeros((2, 10), F32)])
    (y,) = net.run_host([np.zeros((4, 1024), F32)])
    assert y.shape == (4, 10)
    import torch
    dev = torch.cuda.current_device()
    net.apply()
    assert torch.cuda.current_device() == dev          # the caller's context is restored


def test_deterministic_outputs_across_compiles():
    m, w = zoo.build(3)
    x = zoo.inputs(3, 3)
    a, _ = gpu(m, w, x)
    b, _ = gpu(m, w, x)
    np.testing.assert_array_equal(a, b)


def test_timing_entry_points():
    """time_apply / time_launch / time_sequence (bench.py's roofline evidence)
    cover exactly the launches of the pass and return positive durations."""
    m, w = zoo.build(3)
    net = compile_model(m, w, EXACT, batch=8)
    net.run([zoo.inputs(3, 8)])
    for n in (1, 8):
        seq = net.time_sequence(n, iters=2)
        assert sorted(seq) == net.launches_for(n)
        assert all(v > 0 for v in seq.values())
        i = net.launches_for(n)[0]
        assert net.time_launch(i, n, iters=2) > 0
    assert net.time_apply(iters=2) > 0


def test_integration_md_binding_stub_runs():
    """The reference-side ctypes stub in INTEGRATION.md section 3 drives a
    network end to end (kept honest against the ABI)."""
    import pathlib
    import torch
    from paper_1906_05737_b200 import build_graph, build_plan, plan_buffers
    from paper_1906_05737_b200.kernels import specialize
    from paper_1906_05737_b200.runtime import _DeviceArray
    md = (pathlib.Path(__file__).resolve().parent.parent / "INTEGRATION.md").read_text()
    code = md.split("## 3.")[1].split("```python")[1].split("```")[0]
    ns = {}
    exec(code, ns)
    m, w = zoo.build(0)
    plan = build_plan(build_graph(m, w))
    asg = plan_buffers(plan)
    cap, n = 16, 4
    spec = specialize(plan, asg, EXACT, n, cap)
    ex = ns["DeviceExecutable"](spec, asg.arena_size * cap + spec.arena_extra, max_batch=n)
    tin, tout = plan.input_ids[0], plan.output_ids[0]
    view = lambda t: torch.as_tensor(_DeviceArray(ex, ex.arena_address(asg.offsets[t][0] * cap),
                                                  (cap,) + tuple(plan.tensors[t].dims)), device="cuda")
    x = zoo.inputs(0, n)
    view(tin)[:n].copy_(torch.from_numpy(x))
    ex(n)
    torch.cuda.synchronize()
    got = view(tout)[:n].cpu().numpy()
    ex.close()
    np.testing.assert_allclose(got, ref(m, w, x), **TOL)


def test_multi_device_network_shards_batch_over_replicas():
    """compile_model(..., devices=[...]): one replica per listed device with
    contiguous batch slices (two replicas on GPU 0 here), outputs gathered in
    batch order equal the oracle."""
    from paper_1906_05737_b200 import MultiDeviceNetwork
    m, w = zoo.build(3)
    x = zoo.inputs(3, 7)
    net = compile_model(m, w, EXACT, batch=7, devices=[0, 0])
    assert isinstance(net, MultiDeviceNetwork) and [c for _, c in net.slices] == [4, 3]
    got = net.run([x])[0].cpu().numpy()
    np.testing.assert_allclose(got, ref(m, w, x), **TOL)
    with pytest.raises(InputShapeMismatch):
        net.run([x[:5]])
    with pytest.raises(ValueError):
        compile_model(m, w, EXACT, batch=1, devices=[0, 0])


@pytest.mark.parametrize("cfg", [0, 2, 3])
def test_batch1_persistent_kernel_matches_oracle(cfg):
    """mega=True: small batches run as one cooperative kernel walking every
    unit with grid barriers (opt-in; see kernels.Specializer._mega)."""
    m, w = zoo.build(cfg)
    for n in (1, 3):
        x = zoo.inputs(cfg, n)
        net = compile_model(m, w, EXACT, batch=n, tuning={"mega": True})
        coop = [l for l in net.artifact.launches if l.cooperative]
        got = net.run([x])[0].cpu().numpy()
        np.testing.assert_allclose(got, ref(m, w, x), **TOL)
        if n == 1:
            assert coop and net.launches_for(1) == [net.artifact.launches.index(coop[0])]


@pytest.mark.parametrize("k,units", [(1024, 512), (512, 256), (300, 260)])
def test_wide_n256_tiles_opt_in(k, units):
    """wide=True: N = 256 tcgen05 tiles (CTA pairs, whole-K correction chain,
    main chain restarted every 16 k-blocks) against the oracle."""
    rng = np.random.default_rng(k)
    m, w = dense_net(rng, k, units, "tanh")
    rows = wide_rows(units)
    x = rng.uniform(-2, 2, (rows, k)).astype(F32)
    for cb16 in (True, False):
        got, net = gpu(m, w, x, wide=True, corr_bf16=cb16)
        assert any("256x256" in net.artifact.launches[i].note for i in net.launches_for(rows))
        np.testing.assert_allclose(got, ref(m, w, x), **TOL)


def wide_rows(units):
    """Rows from which a Dense with `units` outputs gets N = 256 tiles
    (kernels.WIDE_MIN_TILES 256x256 tiles per launch)."""
    from paper_1906_05737_b200.kernels import WIDE_MIN_TILES
    ntw = -(-units // 256)
    return -(-WIDE_MIN_TILES // ntw) * 256 + 100


@pytest.mark.parametrize("k,units,dist", [(1024, 512, "normal"), (512, 256, "scaled"),
                                          (300, 260, "uniform"), (1024, 384, "scaled")])
def test_wide_tiles_bf16_correction_products(k, units, dist):
    """N = 256 tiles run the two correction products of every tf32 k-step as
    one BF16 MMA (corr_bf16, default).  Stated tolerance of that path (DESIGN.md
    section 4): |d| <= 1e-4 |ref| + 1e-5 + 2^-17 sum_k |a_k b_k|, checked on
    every output; unscaled inputs also pass the plain FP32 gate.  The tf32
    split (corr_bf16=False) is checked against the same oracle."""
    seed = k + units
    rng = np.random.default_rng(seed)
    m, w = dense_net(rng, k, units, "linear")
    wk = he(np.random.default_rng(seed), (k, units), k).astype(np.float64)
    rows = wide_rows(units)
    if dist == "normal":
        x = rng.standard_normal((rows, k)).astype(F32)
    elif dist == "uniform":
        x = rng.uniform(-2, 2, (rows, k)).astype(F32)
    else:
        x = (rng.standard_normal((rows, k)) * rng.uniform(0.1, 10, (rows, 1))).astype(F32)
    want = ref(m, w, x).astype(np.float64)
    got, net = gpu(m, w, x)
    assert any("bf16 corr" in net.artifact.launches[i].note for i in net.launches_for(rows))
    mag = np.abs(x.astype(np.float64)) @ np.abs(wk)
    lim = 1e-4 * np.abs(want) + 1e-5 + 2.0 ** -17 * mag
    assert np.all(np.abs(got - want) <= lim)
    if dist != "scaled":
        np.testing.assert_allclose(got, want, **TOL)
    tf32, net2 = gpu(m, w, x, corr_bf16=False)
    assert not any("bf16 corr" in net2.artifact.launches[i].note for i in net2.launches_for(rows))
    assert np.all(np.abs(tf32 - want) <= 1e-4 * np.abs(want) + 1e-5 + 2.0 ** -19 * mag)


@pytest.mark.parametrize("k,units,head", [(128, 10, "softmax"), (4, 1, "linear"), (64, 24, "tanh"), (256, 8, "relu"),
                                          (64, 3, "add"), (36, 17, "softmax")])
def test_narrow_row_gemm(k, units, head):
    """Many rows, <= 32 columns (nnb_rows.cuh): a ragged last tile, fused
    softmax / residual, against the oracle; with K in one slice (and no
    softmax) bit-identical to the FFMA tile GEMM (same fmaf order: bias first,
    k ascending)."""
    rng = np.random.default_rng(k * 7 + units)
    b = NetBuilder()
    x_ = b.input((k,))

    def dense(src, act):
        return b.layer("Dense", [src], {"units": units, "activation": act},
                       [("kernel", he(rng, (k, units), k)),
                        ("bias", (rng.standard_normal(units) * 0.1).astype(F32))])
    if head == "add":
        y = b.layer("Add", [dense(x_, "relu"), dense(x_, "linear")])
    elif head == "softmax":
        y = b.layer("Softmax", [dense(x_, "linear")])
    else:
        y = dense(x_, head)
    m, w = b.build([y])
    n = 148 * 128 + 57
    x = rng.uniform(-2, 2, (n, k)).astype(F32)
    got, net = gpu(m, w, x)
    assert any("narrow" in l.kernel for l in net.artifact.launches)
    np.testing.assert_allclose(got, ref(m, w, x), **TOL)
    simt, net2 = gpu(m, w, x, narrow=False)
    assert not any("narrow" in l.kernel for l in net2.artifact.launches)
    if head != "softmax" and any("K in 1 slices" in l.note for l in net.artifact.launches):
        np.testing.assert_array_equal(got, simt)
    elif head != "softmax":    # k slices summed in slice order: a few ulp of the partial sums
        np.testing.assert_allclose(got, simt, rtol=2e-6, atol=2e-6)
    else:    # FP32 exact-mode softmax (a few ulp) vs the float64-rounded one
        np.testing.assert_allclose(got, simt, rtol=1e-5, atol=1e-7)


def test_narrow_row_gemm_pixels():
    """A stride-1 1x1 conv with few output channels: pixel rows contiguous
    across images, one narrow launch for the whole batch."""
    rng = np.random.default_rng(5)
    m, w = conv_net(rng, 20, 24, 16, 3, k=1, act="sigmoid")
    x = rng.uniform(-1, 1, (41, 20, 24, 16)).astype(F32)
    got, net = gpu(m, w, x)
    assert any("conv1x1_narrow" in l.kernel for l in net.artifact.launches)
    np.testing.assert_allclose(got, ref(m, w, x), **TOL)
    simt, _ = gpu(m, w, x, narrow=False)
    np.testing.assert_array_equal(got, simt)


@pytest.mark.parametrize("k,n1,act1,n2,head,n", [
    (256, 128, "elu", 10, "softmax", 4100), (64, 32, "relu", 2, "softmax", 2500),
    (128, 96, "tanh", 16, "sigmoid", 3001), (96, 64, "linear", 7, "bn", 2048),
    (256, 128, "elu", 10, "softmax", 600)])
def test_fused_dense_head(k, n1, act1, n2, head, n):
    """Dense (tcgen05) -> Dense head with <= 16 outputs (+ softmax / act /
    BatchNorm): the head computed in the tcgen05 epilogue (HEAD), its input
    never stored; below the tensor-core batch threshold the head stays its
    own launch."""
    rng = np.random.default_rng(k + n1 + n2)
    b = NetBuilder()
    x_ = b.input((k,))
    h = b.layer("Dense", [x_], {"units": n1, "activation": act1},
                [("kernel", he(rng, (k, n1), k)), ("bias", (rng.standard_normal(n1) * 0.1).astype(F32))])
    y = b.layer("Dense", [h], {"units": n2, "activation": head if head in ("sigmoid",) else "linear"},
                [("kernel", he(rng, (n1, n2), n1)), ("bias", (rng.standard_normal(n2) * 0.1).astype(F32))])
    if head == "softmax":
        y = b.layer("Softmax", [y])
    elif head == "bn":
        y = b.layer("BatchNorm", [y], None, bn_params(rng, n2))
    m, w = b.build([y])
    x = rng.uniform(-2, 2, (n, k)).astype(F32)
    got, net = gpu(m, w, x)
    fused = any("fused Dense head" in net.artifact.launches[i].note for i in net.launches_for())
    from paper_1906_05737_b200.kernels import SMALL_DENSE_ROWS, TC_MIN_ROWS
    if n < max(TC_MIN_ROWS, SMALL_DENSE_ROWS + 1):   # no tcgen05 Dense at this batch
        assert not fused, net.describe()
    elif n1 <= 64:                 # two accumulator buffers: the head is fused
        assert fused, net.describe()
    assert len(net.launches_for()) == (1 if fused else 2)
    np.testing.assert_allclose(got, ref(m, w, x), **TOL)
    unf, _ = gpu(m, w, x, head=False)
    np.testing.assert_allclose(got, unf, rtol=1e-5, atol=2e-6)


def _chain_net(rng, h, w, c, spec, gap, post_bn):
    """input h x w x c -> layers from spec: ('p', co, act) pointwise,
    ('d', k, s, pad, act) depthwise; optional BN after an activation
    (post-affine) and a closing GlobalAveragePooling2D."""
    b = NetBuilder()
    x = b.input((h, w, c))
    for i, st in enumerate(spec):
        if st[0] == "p":
            _, co, act = st
            x = b.layer("Conv2D", [x], {"filters": co, "kernel_size": 1, "activation": act},
                        [("kernel", he(rng, (1, 1, c, co), c)),
                         ("bias", (rng.standard_normal(co) * 0.1).astype(F32))])
            c = co
        else:
            _, k, s, pad, act = st
            x = b.layer("DepthwiseConv2D", [x], {"kernel_size": k, "strides": s, "padding": pad,
                                                 "activation": act},
                        [("kernel", he(rng, (k, k, c), k * k)),
                         ("bias", (rng.standard_normal(c) * 0.1).astype(F32))])
        if post_bn and i % 3 == 1:
            x = b.layer("BatchNorm", [x], None, bn_params(rng, c))
    if gap:
        x = b.layer("GlobalAveragePooling2D", [x])
    return b.build([x])


@pytest.mark.parametrize("n", [1, 3, 37])
@pytest.mark.parametrize("case", [
    (16, 16, 32, [("p", 64, "relu6"), ("d", 3, 1, "same", "relu6"), ("p", 64, "relu"),
                  ("d", 3, 2, "same", "relu6"), ("p", 128, "relu6"), ("d", 3, 1, "same", "linear"),
                  ("p", 128, "relu6")], True, True),
    (8, 8, 64, [("d", 3, 1, "same", "relu"), ("p", 64, "linear"), ("d", 5, 1, "same", "relu6"),
                ("p", 128, "tanh"), ("d", 3, 2, "valid", "relu")], False, False),
    (4, 4, 128, [("p", 256, "relu6"), ("d", 3, 1, "same", "relu6"), ("p", 256, "sigmoid"),
                 ("d", 3, 1, "same", "elu")], True, True)])
def test_chain_kernel_vs_oracle(case, n):
    """planner.fuse_chain + nnb_chain.cuh: a run of small depthwise / pointwise
    layers (strides, 'same' / 'valid', 5x5 taps, post-BN, closing GAP or a
    stored map) in one CTA-per-image kernel, against the oracle."""
    h, w, c, spec, gap, post_bn = case
    rng = np.random.default_rng(len(spec) * 10 + c)
    m, wt = _chain_net(rng, h, w, c, spec, gap, post_bn)
    x = rng.uniform(-1, 2, (n, h, w, c)).astype(F32)
    got, net = gpu(m, wt, x, chain=True)
    assert [u.kind for u in net.plan.units] == ["Chain"], net.plan.describe()
    assert any("chain" in l.kernel for l in net.artifact.launches)
    np.testing.assert_allclose(got, ref(m, wt, x), **TOL)
    got2, net2 = gpu(m, wt, x, ApproximationOptions(), chain=True)
    np.testing.assert_allclose(got2, ref(m, wt, x, ApproximationOptions()), **TOL)
    unf, _ = gpu(m, wt, x)
    np.testing.assert_allclose(got, unf, **TOL)


@pytest.mark.parametrize("h,w,ci,co,up,n,tc", [
    (16, 32, 16, 32, False, 3, True), (24, 16, 32, 64, True, 2, True),
    (30, 40, 16, 32, True, 2, True), (12, 20, 16, 64, False, 2, False),
    (10, 14, 8, 16, True, 3, False)])
def test_dual_pooled_store(h, w, ci, co, up, n, tc):
    """planner.fuse_pool_dual: a conv whose output is both a skip and the
    input of a 2x2 max-pool stores the pooled (optionally x2 upsampled) map
    as a second epilogue store -- tcgen05 KPACK (CO=32) and plain conv tiles
    (CO=64) -- or, for kernels without it, gets the pool as its own launch."""
    rng = np.random.default_rng(h * w + co)
    b = NetBuilder()
    x = b.input((h, w, ci))
    c = b.layer("Conv2D", [x], {"filters": co, "kernel_size": 3, "padding": "same",
                                "activation": "relu"},
                [("kernel", he(rng, (3, 3, ci, co), 9 * ci)),
                 ("bias", (rng.standard_normal(co) * 0.1).astype(F32))])
    p = b.maxpool(c)
    if up:
        p = b.layer("UpSample2D", [p], {"factor": 2})
        cat = b.layer("Concatenate", [c, p])
        y = b.layer("Conv2D", [cat], {"filters": 16, "kernel_size": 1, "activation": "linear"},
                    [("kernel", he(rng, (1, 1, 2 * co, 16), 2 * co)), ("bias", np.zeros(16, F32))])
        outs = [y]
    else:
        d = b.layer("Conv2D", [p], {"filters": 16, "kernel_size": 1}, [("kernel", he(rng, (1, 1, co, 16), co)),
                                                                        ("bias", np.zeros(16, F32))])
        outs = [d, c]
    m, wt = b.build(outs)
    xin = rng.uniform(-2, 2, (n, h, w, ci)).astype(F32)
    kw = dict(tc_min_rows=1, tc_tile_use=0) if tc else dict(use_tc=False)
    net = compile_model(m, wt, EXACT, batch=n, tuning=kw)
    got = [o.cpu().numpy() for o in net.run([xin])]
    conv = [u for u in net.plan.units if u.kind == "Conv2D" and u.dual_pool is not None]
    assert len(conv) == 1 and "Pool" not in [u.kind for u in net.plan.units]
    ls = [l for l in net.artifact.launches if l.n_min <= n <= l.n_max]
    assert any("pooled second store" in l.note for l in ls) == tc
    assert any("maxpool" in l.kernel for l in ls) == (not tc)
    want = oracle.run(m, wt, [xin], "exact")
    for g, wv in zip(got, want):
        np.testing.assert_allclose(g, wv, **TOL)


@pytest.mark.parametrize("n", [1, 3, 40, 77, 330])     # 330: persistent CTAs take a second tile
@pytest.mark.parametrize("case", [
    # cfg3's 8x8 stage: pw -> dw pairs (stride 1, then stride 2 to 4x4), post-BN after some
    (8, 8, 64, [("p", 128, "relu6"), ("d", 3, 1, "same", "relu6"), ("p", 128, "relu6"),
                ("d", 3, 2, "same", "relu6"), ("p", 256, "relu6"), ("d", 3, 1, "same", "relu6"),
                ("p", 256, "linear")], True, True),
    # 4x8 maps (four images per tile), 5x5 and 'valid' windows, 96 channels (BN = 96 -> 128),
    # two N tiles (160 channels), tanh / sigmoid epilogues
    (4, 8, 32, [("p", 96, "tanh"), ("d", 5, 1, "same", "relu"), ("p", 160, "sigmoid"),
                ("d", 3, 1, "valid", "elu"), ("p", 32, "linear")], False, False),
    # 2x2 maps (32 images per tile) and a 16x8 map (one image per tile)
    (16, 8, 16, [("p", 64, "relu"), ("d", 3, 2, "same", "relu6"), ("p", 64, "relu6"),
                 ("d", 3, 2, "valid", "linear"), ("p", 32, "relu"), ("d", 3, 2, "same", "tanh")],
     False, True),
    # one image per tile (16x8 = 128 pixels), then a 1x1 map (128 images per tile: only the centre tap)
    (16, 8, 32, [("p", 64, "relu"), ("d", 3, 1, "same", "relu6"), ("p", 32, "linear"),
                 ("d", 5, 2, "same", "relu")], False, False),
    (1, 1, 32, [("p", 64, "tanh"), ("d", 3, 1, "same", "relu"), ("p", 32, "linear")], False, True),
    # band tiles: cfg3's 16x16 stage (3 bands of 8 rows per image; stride 1, then 2 to 8x8)
    (16, 16, 32, [("p", 64, "relu6"), ("d", 3, 1, "same", "relu6"), ("p", 64, "relu6"),
                  ("d", 3, 2, "same", "relu6"), ("p", 128, "relu6"), ("d", 3, 1, "same", "linear"),
                  ("p", 32, "linear")], False, True),
    # bands of 16 rows of a 32x8 map (5x5 taps), then 8 rows of a 24x16 map with 'valid' windows
    (32, 8, 16, [("p", 32, "tanh"), ("d", 5, 1, "same", "relu"), ("p", 64, "sigmoid"),
                 ("d", 3, 2, "valid", "linear"), ("p", 32, "relu")], False, False),
    (24, 16, 32, [("p", 96, "relu"), ("d", 3, 1, "valid", "relu6"), ("p", 40, "elu"),
                  ("d", 3, 2, "same", "tanh")], False, True)])
@pytest.mark.parametrize("opts", [EXACT, ApproximationOptions()], ids=["exact", "default"])
def test_pointwise_with_depthwise_epilogue(case, n, opts):
    """planner.fuse_pw_dw + nnb_gemm_tc.cuh EDW: a 1x1 conv whose consumer is a
    depthwise conv over a map that fits a 128-row tile computes that conv in
    its tcgen05 epilogue (ragged batches leave part of a tile empty); batch
    sizes below the tcgen05 threshold run the depthwise conv as a second
    launch of the unit.  Against the oracle and the unfused plan."""
    h, w, c, spec, gap, post_bn = case
    rng = np.random.default_rng(len(spec) * 13 + c + n)
    m, wt = _chain_net(rng, h, w, c, spec, gap, post_bn)
    x = rng.uniform(-1, 2, (n, h, w, c)).astype(F32)
    want = ref(m, wt, x, "exact" if opts == EXACT else opts)
    bands = 128 % (h * w) != 0            # maps larger than a tile: the opt-in band tiles
    for forced in (True, False):
        tune = dict(tc_min_rows=1, tc_min_images=1, small_conv=False) if forced else {}
        if bands:
            tune = dict(tune, pw_dw="bands")
        got, net = gpu(m, wt, x, opts, **tune)
        fused = [u for u in net.plan.units if u.dw_after is not None]
        assert fused, net.plan.describe()
        act = [l for l in net.artifact.launches if l.n_min <= n <= l.n_max]
        if forced:
            assert any("depthwise conv in the epilogue" in l.note for l in act), [l.kernel for l in act]
        for u in fused:      # one fused launch, or the pointwise kernel + a depthwise launch
            mine = [l for l in act if net.plan.units[l.unit] is u]
            assert len(mine) == (1 if "in the epilogue" in mine[0].note else 2)
        np.testing.assert_allclose(got, want, **TOL)
    unf, net0 = gpu(m, wt, x, opts, pw_dw=False)
    assert not [u for u in net0.plan.units if u.dw_after is not None]
    np.testing.assert_allclose(got, unf, **TOL)


@pytest.mark.parametrize("n", [1, 2, 5, 64])
@pytest.mark.parametrize("case", [
    # cfg3-like: pw 64->128 reading an 8x8 map from the arena, dw/pw pairs at 8x8,
    # closing stride-2 dw to 4x4 (stored)
    (8, 8, 64, [("p", 128, "relu6"), ("d", 3, 1, "same", "relu6"),
                ("p", 128, "relu6"), ("d", 3, 1, "same", "relu"), ("p", 128, "linear"),
                ("d", 3, 2, "same", "relu6")], False, True),
    # 7x7 maps (49 of 64 rows live), 5x5 taps, 'valid' ahead of the chain, a
    # closing pointwise (stored)
    (9, 9, 32, [("d", 3, 1, "valid", "relu"), ("p", 64, "tanh"), ("d", 5, 1, "same", "relu6"),
                ("p", 32, "relu"), ("d", 3, 1, "same", "linear"), ("p", 96, "sigmoid")], False, False)])
def test_tc_chain_vs_oracle(case, n):
    """planner.fuse_tc_chain + nnb_tcchain.cuh: the 8x8 stage of a MobileNet-
    style net on the tensor cores, two images per CTA (odd batches leave half
    a CTA empty), against the oracle; and against the per-layer launches."""
    h, w, c, spec, gap, post_bn = case
    rng = np.random.default_rng(len(spec) * 7 + c + n)
    m, wt = _chain_net(rng, h, w, c, spec, gap, post_bn)
    x = rng.uniform(-1, 2, (n, h, w, c)).astype(F32)
    got, net = gpu(m, wt, x, tc_chain=True)
    assert "TcChain" in [u.kind for u in net.plan.units], net.plan.describe()
    assert any("tcchain" in l.kernel for l in net.artifact.launches)
    np.testing.assert_allclose(got, ref(m, wt, x), **TOL)
    got2, _ = gpu(m, wt, x, ApproximationOptions(), tc_chain=True)
    np.testing.assert_allclose(got2, ref(m, wt, x, ApproximationOptions()), **TOL)
    unf, net3 = gpu(m, wt, x)
    assert "TcChain" not in [u.kind for u in net3.plan.units]
    np.testing.assert_allclose(got, unf, **TOL)


@pytest.mark.parametrize("n", [1, 3, 64])
@pytest.mark.parametrize("opts", [EXACT, ApproximationOptions()], ids=["exact", "default"])
def test_tinynet_whole_network_launch(n, opts):
    """kernels.Specializer._tiny / nnb_tiny.cuh: cfg0 and a small net with a
    residual, BatchNorm, depthwise, avg-pool, padding-valid stride-2 conv and a
    softmax run as ONE launch at small batches, against the oracle."""
    nets = [zoo.build(0)]
    rng = np.random.default_rng(n)
    b = NetBuilder()
    x = b.input((12, 10, 4))
    c1 = b.layer("Conv2D", [x], {"filters": 8, "kernel_size": 3, "padding": "same", "activation": "relu"},
                 [("kernel", he(rng, (3, 3, 4, 8), 36)), ("bias", (rng.standard_normal(8) * .1).astype(F32))])
    d = b.layer("DepthwiseConv2D", [c1], {"kernel_size": 3, "padding": "same", "activation": "tanh"},
                [("kernel", he(rng, (3, 3, 8), 9)), ("bias", (rng.standard_normal(8) * .1).astype(F32))])
    a = b.layer("Add", [c1, d])
    bn = b.layer("BatchNorm", [a], None, bn_params(rng, 8))
    c2 = b.layer("Conv2D", [bn], {"filters": 8, "kernel_size": 3, "strides": 2, "padding": "valid",
                                  "activation": "sigmoid"},
                 [("kernel", he(rng, (3, 3, 8, 8), 72)), ("bias", np.zeros(8, F32))])
    p = b.layer("AvgPool2D", [c2], {"pool_size": 2, "strides": 1})
    f = b.layer("Flatten", [p])
    y = b.layer("Dense", [f], {"units": 7, "activation": "linear"},
                [("kernel", he(rng, (4 * 3 * 8, 7), 96)), ("bias", np.zeros(7, F32))])
    nets.append(b.build([b.layer("Softmax", [y])]))
    for k, (m, w) in enumerate(nets):
        xin = (zoo.inputs(0, n) if k == 0 else rng.uniform(-2, 2, (n, 12, 10, 4)).astype(F32))
        got, net = gpu(m, w, xin, opts, tiny=True)
        act = [l for l in net.artifact.launches if l.n_min <= n <= l.n_max]
        assert [("tinynet" in l.kernel) for l in act] == [True], [l.kernel for l in act]
        np.testing.assert_allclose(got, ref(m, w, xin, "exact" if opts == EXACT else opts), **TOL)


@pytest.mark.parametrize("h,w,ci,co,n", [(8, 8, 16, 16, 5), (9, 7, 12, 16, 3), (16, 16, 8, 16, 2),
                                         (10, 6, 16, 8, 4)])
def test_direct_conv_pool_window_split_over_lanes(h, w, ci, co, n):
    """ConvDirect with a fused 2x2 max-pool whose window is split over 2
    lanes (PSPLIT 2: one row each) or 4 (one pixel each) so the weights stay
    instruction immediates within the compile budget (odd maps: the last
    row / column has no window)."""
    rng = np.random.default_rng(h * ci + co)
    b = NetBuilder()
    x = b.input((h, w, ci))
    y = b.maxpool(b.layer("Conv2D", [x], {"filters": co, "kernel_size": 3, "padding": "same",
                                          "activation": "relu"},
                          [("kernel", he(rng, (3, 3, ci, co), 9 * ci)),
                           ("bias", (rng.standard_normal(co) * 0.1).astype(F32))]))
    m, wt = b.build([y])
    xin = rng.uniform(-2, 2, (n, h, w, ci)).astype(F32)
    got, net = gpu(m, wt, xin)
    assert any("direct" in l.kernel and "immediates" in l.note for l in net.artifact.launches)
    np.testing.assert_allclose(got, ref(m, wt, xin), **TOL)


@pytest.mark.gpu
@pytest.mark.parametrize("h,w,ci,co,k,pad,n", [
    (19, 35, 32, 32, 3, "same", 2), (12, 21, 16, 32, 5, "same", 2), (13, 18, 32, 64, 3, "valid", 2),
    (20, 33, 128, 32, 3, "same", 1)])
def test_row_shared_kpack_conv(h, w, ci, co, k, pad, n):
    """KPACK conv tiles with one A box of 8 + KH - 1 rows shared by every
    kernel row (RS, 16-row descriptor offsets; 16-channel k-blocks when two
    32-channel stages do not fit), against the oracle and the per-row-box form."""
    rng = np.random.default_rng(ci * k + co)
    b = NetBuilder()
    x = b.input((h, w, ci))
    y = b.layer("Conv2D", [x], {"filters": co, "kernel_size": k, "padding": pad, "activation": "tanh"},
                [("kernel", he(rng, (k, k, ci, co), k * k * ci)),
                 ("bias", (rng.standard_normal(co) * 0.1).astype(F32))])
    m, wt = b.build([y])
    xin = rng.uniform(-2, 2, (n, h, w, ci)).astype(F32)
    got, net = gpu(m, wt, xin, tc_min_rows=1, tc_tile_use=0, direct_imm=False)
    assert any("rows shared" in l.note for l in net.artifact.launches), \
        [l.note for l in net.artifact.launches]
    want = ref(m, wt, xin)
    np.testing.assert_allclose(got, want, **TOL)
    per_row, net1 = gpu(m, wt, xin, tc_min_rows=1, tc_tile_use=0, direct_imm=False, rowshare=False)
    assert not any("rows shared" in l.note for l in net1.artifact.launches)
    np.testing.assert_allclose(per_row, want, **TOL)


def test_weight_prefetch_branch(monkeypatch):
    """nnb_runtime.cpp prefetch_branch: graphs of small batches carry a second
    branch that prefetches the constant pool into L2 (NNB_PREFETCH_MAX_N, default
    16).  It changes no result, and larger batches keep the single chain."""
    m, w = zoo.build(2)
    for n in (1, 16, 17):
        x = zoo.inputs(2, n)
        outs = []
        for env in ("0", None):
            if env is None:
                monkeypatch.delenv("NNB_PREFETCH_MAX_N", raising=False)
            else:
                monkeypatch.setenv("NNB_PREFETCH_MAX_N", env)
            got, net = gpu(m, w, x, ApproximationOptions())
            got2 = net.run([x])[0].cpu().numpy()          # the cached graph replays
            assert np.array_equal(got, got2)
            outs.append(got)
        assert np.array_equal(outs[0], outs[1])
        np.testing.assert_allclose(outs[1], ref(m, w, x, ApproximationOptions()), **TOL)


@pytest.mark.parametrize("h,w,c,co,act,softmax,n", [
    (8, 10, 128, 4, "linear", False, 37), (4, 4, 256, 10, "linear", True, 5), (3, 5, 8, 1, "tanh", False, 1),
    (7, 7, 40, 32, "relu", False, 130), (1, 1, 16, 3, "sigmoid", True, 9)])
@pytest.mark.parametrize("opts", [EXACT, ApproximationOptions()], ids=["exact", "default"])
def test_gap_dense_head(h, w, c, co, act, softmax, n, opts):
    """planner.fuse_gap_dense + nnb_small.cuh GapDense: GlobalAveragePooling2D
    and the narrow Dense consuming it as one launch (one warp per image; more
    than 32 channel quads per lane group, softmax, ragged last block)."""
    rng = np.random.default_rng(h * w + c + co)
    b = NetBuilder()
    x = b.input((h, w, c))
    # (a depthwise conv ahead of the pool: a 1x1 conv over a map that fits a
    # tcgen05 tile would take the pool in its own epilogue, planner.fuse_pw_dw)
    y = b.layer("DepthwiseConv2D", [x], {"kernel_size": 3, "padding": "same", "activation": "relu"},
                [("kernel", he(rng, (3, 3, c), 9)), ("bias", (rng.standard_normal(c) * 0.1).astype(F32))])
    g = b.layer("GlobalAveragePooling2D", [y])
    d = b.layer("Dense", [g], {"units": co, "activation": act},
                [("kernel", he(rng, (c, co), c)), ("bias", (rng.standard_normal(co) * 0.1).astype(F32))])
    if softmax:
        d = b.layer("Softmax", [d])
    m, wt = b.build([d])
    xin = rng.uniform(-2, 2, (n, h, w, c)).astype(F32)
    got, net = gpu(m, wt, xin, opts)
    assert [u.kind for u in net.plan.units][-1] == "Dense" and net.plan.units[-1].gap is not None, \
        net.plan.describe()
    assert [l.kernel.split("_", 2)[2] for l in net.artifact.launches][-1].startswith("gap_dense")
    np.testing.assert_allclose(got, ref(m, wt, xin, "exact" if opts == EXACT else opts), **TOL)
    sep, net2 = gpu(m, wt, xin, opts, gap_dense=False)
    assert "Pool" in [u.kind for u in net2.plan.units]
    np.testing.assert_allclose(got, sep, rtol=1e-5, atol=2e-6)
