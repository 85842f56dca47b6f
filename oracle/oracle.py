"""CPU oracle driver (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module -- as the checker or the
reported CPU baseline, never as the product path.

Executes a layer graph node by node, exactly like the reference interpreter
(pkg/src/nnjit/interpreter.py:125-195): no fusion, fresh storage per tensor,
per-layer arithmetic in ``libnnoracle.so`` (oracle/nnoracle.c).  Every
tensor carries a leading batch axis; images are independent, so the batch
axis changes nothing numerically.

``mode`` selects the transcendental semantics:
  * ``"exact"``    -- the interpreter (float64 tanh/sigmoid/exp, rounded once);
  * an ``ApproximationOptions``-like object with ``activation_mode`` in
    {rational, fast, exact} and ``softmax_exp`` in {fast, precise, exact} --
    the compiled path's approximation models (codegen/approx.py:72-128).
"""

import ctypes
import os
import pathlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB = HERE / "libnnoracle.so"
F32 = np.float32
ACT = {"linear": 0, "relu": 1, "sigmoid": 2, "tanh": 3, "relu6": 4, "elu": 5}
AMODE = {"rational": 0, "fast": 1, "exact": 2}
SMODE = {"fast": 0, "precise": 1, "exact": 2}

_lib = None


def build(force=False):
    """Compile libnnoracle.so with the flags that keep float32 rounding exact."""
    import subprocess
    if LIB.exists() and not force and LIB.stat().st_mtime >= (HERE / "nnoracle.c").stat().st_mtime:
        return LIB
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
                           "-fno-fast-math", "-o", str(LIB), str(HERE / "nnoracle.c"),
                           "-lm", "-lpthread"])
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = ctypes.CDLL(str(LIB))
        for name in ("nno_tanh_rational", "nno_sigmoid_rational", "nno_exp_fast",
                     "nno_sigmoid_fast", "nno_tanh_fast", "nno_exp_precise"):
            fn = getattr(_lib, name)
            fn.restype, fn.argtypes = ctypes.c_float, [ctypes.c_float]
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a):
    return np.ascontiguousarray(a, dtype=F32)


def same_padding(size, kernel, stride):
    out = -(-size // stride)
    total = max((out - 1) * stride + kernel - size, 0)
    return total // 2, total - total // 2


def _modes(mode):
    if mode == "exact" or mode is None:
        return 2, 2
    return AMODE[mode.activation_mode], SMODE[mode.softmax_exp]


def activation(x, tag, amode=2):
    x = _c(x)
    y = np.empty_like(x)
    lib().nno_activation(_p(x), _p(y), ctypes.c_long(x.size), ACT[tag], amode)
    return y


def dense(x, k, b, threads):
    x, k, b = _c(x), _c(k), _c(b)
    n, kin = x.shape[0], x.reshape(x.shape[0], -1).shape[1]
    y = np.empty((n, k.shape[1]), F32)
    lib().nno_dense(_p(x), n, kin, _p(k), _p(b), k.shape[1], _p(y), threads)
    return y


def conv(x, k, b, stride, padding, depthwise, threads):
    x, k, b = _c(x), _c(k), _c(b)
    n, h, w, ci = x.shape
    kh, kw = k.shape[0], k.shape[1]
    co = ci if depthwise else k.shape[3]
    if padding == "same":
        pt, pl = same_padding(h, kh, stride)[0], same_padding(w, kw, stride)[0]
        ho, wo = -(-h // stride), -(-w // stride)
    else:
        pt = pl = 0
        ho, wo = (h - kh) // stride + 1, (w - kw) // stride + 1
    y = np.empty((n, ho, wo, co), F32)
    lib().nno_conv2d(_p(x), n, h, w, ci, _p(k), _p(b), kh, kw, co, stride, pt, pl, ho, wo,
                     _p(y), int(depthwise), threads)
    return y


def pool(x, ph, pw, stride, padding, avg):
    x = _c(x)
    n, h, w, c = x.shape
    if padding == "same":
        pt, pl = same_padding(h, ph, stride)[0], same_padding(w, pw, stride)[0]
        ho, wo = -(-h // stride), -(-w // stride)
    else:
        pt = pl = 0
        ho, wo = (h - ph) // stride + 1, (w - pw) // stride + 1
    y = np.empty((n, ho, wo, c), F32)
    lib().nno_pool(_p(x), n, h, w, c, ph, pw, stride, pt, pl, ho, wo, int(avg), _p(y))
    return y


def softmax(x, smode=2):
    x = _c(x)
    y = np.empty_like(x)
    L = x.shape[-1]
    lib().nno_softmax(_p(x), _p(y), ctypes.c_long(x.size // L), L, smode)
    return y


def _weights(spec, store):
    from paper_1906_05737_b200.model_format import layer_weights
    return layer_weights(spec, store) if spec.weight_refs else {}


def run_graph(graph, inputs, mode="exact", threads=None):
    """Evaluate ``graph`` (paper_1906_05737_b200.graph.ComputationGraph) on
    batched inputs (each ``[n, *input_dims]``); returns batched outputs."""
    threads = threads or os.cpu_count() or 1
    amode, smode = _modes(mode)
    L = lib()
    vals = {}
    for nid, x in zip(graph.input_ids, inputs):
        vals[nid] = _c(x)
    for idx in graph.order:
        node = graph.nodes[idx]
        kind, cfg = node.kind, node.config
        if kind == "Input":
            continue
        ins = [vals[i] for i in node.input_ids]
        x = ins[0]
        n = x.shape[0]
        w = _weights(node.spec, graph.weights)
        if kind == "Dense":
            b = w.get("bias", np.zeros(cfg["units"], F32))
            y = activation(dense(x, w["kernel"], b, threads), cfg["activation"], amode)
        elif kind in ("Conv2D", "DepthwiseConv2D"):
            dw = kind == "DepthwiseConv2D"
            nb = x.shape[-1] if dw else cfg["filters"]
            b = w.get("bias", np.zeros(nb, F32))
            y = conv(x, w["kernel"], b, cfg["strides"], cfg["padding"], dw, threads)
            y = activation(y, cfg["activation"], amode)
        elif kind == "SeparableConv2D":
            t = conv(x, w["depthwise"], np.zeros(x.shape[-1], F32), cfg["strides"],
                     cfg["padding"], True, threads)
            b = w.get("bias", np.zeros(cfg["filters"], F32))
            y = activation(conv(t, w["pointwise"], b, 1, "valid", False, threads),
                           cfg["activation"], amode)
        elif kind in ("MaxPool2D", "AvgPool2D"):
            ph, pw = cfg["pool_size"]
            y = pool(x, ph, pw, cfg["strides"], cfg["padding"], kind == "AvgPool2D")
        elif kind == "GlobalAveragePooling2D":
            y = pool(x, x.shape[1], x.shape[2], 1, "valid", True).reshape(n, -1)
        elif kind == "ZeroPadding2D":
            (t, bt), (l, r) = cfg["padding"]
            _, h, wd, c = x.shape
            y = np.empty((n, h + t + bt, wd + l + r, c), F32)
            L.nno_zeropad(_p(x), n, h, wd, c, t, l, h + t + bt, wd + l + r, _p(y))
        elif kind == "BatchNorm":
            s, o = _c(w["scale"]), _c(w["offset"])
            y = np.empty_like(x)
            L.nno_affine(_p(x), _p(y), ctypes.c_long(x.size), _p(s), _p(o), len(s))
        elif kind == "Activation":
            y = activation(x, cfg["activation"], amode)
        elif kind == "Softmax":
            y = softmax(x, smode)
        elif kind == "Flatten":
            y = x.reshape(n, -1)
        elif kind == "UpSample2D":
            f = cfg["factor"]
            _, h, wd, c = x.shape
            y = np.empty((n, h * f, wd * f, c), F32)
            L.nno_upsample(_p(x), n, h, wd, c, f, _p(y))
        elif kind == "Add":
            y = x.copy()
            for other in ins[1:]:
                L.nno_add(_p(y), _p(_c(other)), ctypes.c_long(y.size))
        elif kind == "Concatenate":
            ct = sum(t.shape[-1] for t in ins)
            y = np.empty(x.shape[:-1] + (ct,), F32)
            p = int(np.prod(x.shape[1:-1])) if x.ndim > 2 else 1
            c0 = 0
            for t in ins:
                t = _c(t)
                L.nno_concat_part(_p(t), n, ctypes.c_long(p), t.shape[-1], _p(y), ct, c0)
                c0 += t.shape[-1]
        else:
            raise AssertionError(f"oracle: unhandled kind {kind}")
        vals[idx] = y
    return [vals[i] for i in graph.output_ids]


def run(manifest, weights, inputs, mode="exact", threads=None):
    from paper_1906_05737_b200.graph import build_graph
    return run_graph(build_graph(manifest, weights), inputs, mode, threads)
