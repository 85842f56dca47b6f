"""``interpret(graph, inputs)`` -- the SimpleNN analogue of the public API
(pkg/src/nnjit/interpreter.py:176-195), in numpy on the host.

This is an API-parity entry point for users and for ``cli verify`` (which,
like the reference's, compares the compiled network against it).  It is NOT
used by ``CompiledNetwork``: compile()/apply() only ever run the sm_100a
kernels through libnnb.so.

Semantics are the reference interpreter's: per-op float32 rounding in the
documented accumulation orders, transcendentals in float64 rounded once.
Every tensor carries a leading batch axis when ``batched=True``.
"""

import numpy as np

from .errors import InputShapeMismatch
from .graph import same_padding
from .model_format import layer_weights

F32 = np.float32


def _pad(x, kh, kw, s, padding, fill=0.0):
    if padding == "valid":
        return x
    _, h, w, c = x.shape
    pt, pb = same_padding(h, kh, s)
    pl, pr = same_padding(w, kw, s)
    out = np.full((x.shape[0], h + pt + pb, w + pl + pr, c), fill, F32)
    out[:, pt:pt + h, pl:pl + w] = x
    return out


def _taps(xp, ky, kx, ho, wo, s):
    return xp[:, ky:ky + ho * s:s, kx:kx + wo * s:s]


def _act(x, tag):
    if tag == "linear":
        return x.copy()
    if tag == "relu":
        return np.maximum(x, F32(0))
    if tag == "relu6":
        return np.minimum(np.maximum(x, F32(0)), F32(6))
    x64 = x.astype(np.float64)
    if tag == "tanh":
        return np.tanh(x64).astype(F32)
    if tag == "sigmoid":
        with np.errstate(over="ignore"):
            return (1.0 / (1.0 + np.exp(-x64))).astype(F32)
    if tag == "elu":
        return np.where(x > 0, x, np.expm1(x64).astype(F32)).astype(F32)
    raise AssertionError(tag)


def _conv(x, k, b, s, padding, ho, wo, depthwise):
    kh, kw = k.shape[:2]
    xp = _pad(x, kh, kw, s, padding)
    co = k.shape[2] if depthwise else k.shape[3]
    acc = np.empty((x.shape[0], ho, wo, co), F32)
    acc[:] = b
    for ky in range(kh):
        for kx in range(kw):
            t = _taps(xp, ky, kx, ho, wo, s)
            if depthwise:
                acc += t * k[ky, kx]
            else:
                for ci in range(k.shape[2]):
                    acc += t[..., ci, None] * k[ky, kx, ci]
    return acc


def _pool(x, ph, pw, s, padding, ho, wo, avg):
    xp = _pad(x, ph, pw, s, padding, 0.0 if avg else -np.inf)
    if avg:
        ones = _pad(np.ones(x.shape[:3] + (1,), F32), ph, pw, s, padding)
        acc = np.zeros((x.shape[0], ho, wo, x.shape[3]), F32)
        cnt = np.zeros((x.shape[0], ho, wo, 1), F32)
        for ky in range(ph):
            for kx in range(pw):
                acc += _taps(xp, ky, kx, ho, wo, s)
                cnt += _taps(ones, ky, kx, ho, wo, s)
        return acc / cnt
    acc = np.full((x.shape[0], ho, wo, x.shape[3]), -np.inf, F32)
    for ky in range(ph):
        for kx in range(pw):
            np.maximum(acc, _taps(xp, ky, kx, ho, wo, s), out=acc)
    return acc


def _softmax(x):
    x64 = x.astype(np.float64)
    e = np.exp(x64 - x.max(axis=-1, keepdims=True).astype(np.float64))
    return (e / e.sum(axis=-1, keepdims=True)).astype(F32)


def _node(node, ins, weights):
    kind, cfg = node.kind, node.config
    x = ins[0]
    n = x.shape[0]
    w = layer_weights(node.spec, weights) if node.spec.weight_refs else {}
    shape = node.output_shape.dims
    if kind == "Dense":
        acc = np.empty((n, cfg["units"]), F32)
        acc[:] = w.get("bias", np.zeros(cfg["units"], F32))
        k = w["kernel"]
        for i in range(k.shape[0]):
            acc += x[:, i, None] * k[i]
        return _act(acc, cfg["activation"])
    if kind in ("Conv2D", "DepthwiseConv2D"):
        dw = kind == "DepthwiseConv2D"
        b = w.get("bias", np.zeros(shape[-1], F32))
        y = _conv(x, w["kernel"], b, cfg["strides"], cfg["padding"], shape[0], shape[1], dw)
        return _act(y, cfg["activation"])
    if kind == "SeparableConv2D":
        kh, kw = cfg["kernel_size"]
        hh = shape[0]
        ww = shape[1]
        t = _conv(x, w["depthwise"], np.zeros(x.shape[-1], F32), cfg["strides"], cfg["padding"],
                  hh, ww, True)
        y = _conv(t, w["pointwise"], w.get("bias", np.zeros(shape[-1], F32)), 1, "valid",
                  hh, ww, False)
        return _act(y, cfg["activation"])
    if kind in ("MaxPool2D", "AvgPool2D"):
        ph, pw = cfg["pool_size"]
        return _pool(x, ph, pw, cfg["strides"], cfg["padding"], shape[0], shape[1],
                     kind == "AvgPool2D")
    if kind == "GlobalAveragePooling2D":
        return _pool(x, x.shape[1], x.shape[2], 1, "valid", 1, 1, True).reshape(n, -1)
    if kind == "ZeroPadding2D":
        (t, b), (l, r) = cfg["padding"]
        return np.pad(x, ((0, 0), (t, b), (l, r), (0, 0)))
    if kind == "BatchNorm":
        return (x * w["scale"] + w["offset"]).astype(F32)
    if kind == "Activation":
        return _act(x, cfg["activation"])
    if kind == "Softmax":
        return _softmax(x)
    if kind == "Flatten":
        return x.reshape(n, -1)
    if kind == "UpSample2D":
        f = cfg["factor"]
        return np.repeat(np.repeat(x, f, axis=1), f, axis=2)
    if kind == "Add":
        acc = x.copy()
        for o in ins[1:]:
            acc += o
        return acc
    if kind == "Concatenate":
        return np.concatenate(ins, axis=-1)
    raise AssertionError(kind)


def interpret(graph, inputs, batched=False):
    """Evaluate ``graph`` on host inputs (one array per graph input).  With
    ``batched=True`` every input carries a leading batch axis."""
    if len(inputs) != len(graph.input_ids):
        raise InputShapeMismatch(f"model takes {len(graph.input_ids)} inputs, got {len(inputs)}")
    vals = {}
    for nid, arr in zip(graph.input_ids, inputs):
        arr = np.asarray(arr, F32)
        want = graph.nodes[nid].output_shape.dims
        got = arr.shape[1:] if batched else arr.shape
        if tuple(got) != tuple(want):
            raise InputShapeMismatch(f"input '{graph.nodes[nid].name}' expects shape {want}, "
                                     f"got {arr.shape}")
        vals[nid] = arr if batched else arr[None]
    for i in graph.order:
        node = graph.nodes[i]
        if node.kind != "Input":
            vals[i] = _node(node, [vals[s] for s in node.input_ids], graph.weights)
    outs = [vals[i] for i in graph.output_ids]
    return outs if batched else [o[0] for o in outs]
