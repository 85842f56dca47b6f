"""Keras -> container exporter.

Counterpart of the reference's exporter (pkg/keras-exporter/src/
nnjit_keras_export/export.py:245-286, cli.py): walk a built Keras 3 model's
tensor graph structurally -- ``tensor._keras_history`` ->
``operation._inbound_nodes[i]`` -- so no backend is imported, and emit the
JSON manifest + little-endian float32 blob that ``model_format.load_model``
reads.  BatchNormalization statistics are folded to (scale, offset) in
float64 at export time, as the reference does (export.py:163-169).

Beyond the reference's layer set this covers the BASELINE vocabulary
(SURVEY.md section 2.3): SeparableConv2D, GlobalAveragePooling2D,
ZeroPadding2D, ReLU(max_value=6) / activation ``relu6``, ELU(alpha=1) /
activation ``elu`` and Softmax over the channel axis of a rank-3 tensor.

keras is not installed in this environment; ``tests/test_keras_export.py``
drives the exporter with stand-in objects that expose the same attributes.
"""

import json
import pathlib

import numpy as np

from .errors import ModelFormatError


class ExportError(ModelFormatError):
    """The Keras model uses something the container cannot express."""


_TAGS = {"linear": "linear", "relu": "relu", "tanh": "tanh", "sigmoid": "sigmoid",
         "relu6": "relu6", "elu": "elu", "softmax": "softmax"}
_DROPPED = frozenset(["Dropout", "SpatialDropout2D", "GaussianDropout", "GaussianNoise",
                      "AlphaDropout"])


def _two(v, what):
    if isinstance(v, (tuple, list)):
        if len(v) != 2:
            raise ExportError(f"{what}: expected an int or a pair, got {v!r}")
        return [int(v[0]), int(v[1])]
    return [int(v), int(v)]


def _act(op):
    fn = getattr(op, "activation", None)
    name = "linear" if fn is None else getattr(fn, "__name__", str(fn))
    if name not in _TAGS:
        raise ExportError(f"{op.name}: activation {name!r} has no container tag")
    return _TAGS[name]


def _channels_last(op):
    if getattr(op, "data_format", None) not in (None, "channels_last"):
        raise ExportError(f"{op.name}: channels_last data format required")


def _conv_checks(op):
    _channels_last(op)
    if _two(getattr(op, "dilation_rate", 1), op.name) != [1, 1]:
        raise ExportError(f"{op.name}: dilated convolution is unsupported")
    if int(getattr(op, "groups", 1)) != 1:
        raise ExportError(f"{op.name}: grouped convolution is unsupported")
    if int(getattr(op, "depth_multiplier", 1)) != 1:
        raise ExportError(f"{op.name}: depth_multiplier must be 1")
    s = _two(op.strides, op.name)
    if s[0] != s[1]:
        raise ExportError(f"{op.name}: non-square strides are unsupported")


class _Writer:
    """Accumulates manifest layers and the weight blob."""

    def __init__(self):
        self.layers, self.blob, self.used = [], bytearray(), set()

    def name(self, base):
        n, i = base, 0
        while n in self.used:
            i += 1
            n = f"{base}_{i}"
        self.used.add(n)
        return n

    def tensor(self, name, arr):
        a = np.ascontiguousarray(np.asarray(arr, dtype=np.float64).astype("<f4"))
        if not np.isfinite(a).all():
            raise ExportError(f"{name}: non-finite values")
        ref = {"name": name, "shape": list(a.shape), "offset": len(self.blob),
               "length": a.nbytes}
        self.blob += a.tobytes()
        return ref

    def layer(self, base, kind, inputs=(), config=None, weights=()):
        n = self.name(base)
        d = {"name": n, "kind": kind}
        if inputs:
            d["inputs"] = list(inputs)
        if config:
            d["config"] = config
        if weights:
            d["weights"] = [self.tensor(f"{n}.{role}", a) for role, a in weights]
        self.layers.append(d)
        return n


# -- converters: (writer, op, node, input names) -> output name -------------------

def _x_input(w, op, node, ins):
    shape = list(node.output_tensors[0].shape)[1:]
    if not shape or any(d is None for d in shape):
        raise ExportError(f"{op.name}: the input shape must be fully defined")
    return w.layer(op.name, "Input", config={"shape": [int(d) for d in shape]})


def _with_softmax(w, op, name, act):
    return w.layer(f"{op.name}_softmax", "Softmax", [name]) if act == "softmax" else name


def _x_dense(w, op, node, ins):
    act = _act(op)
    ws = [np.asarray(a) for a in op.get_weights()]
    weights = [("kernel", ws[0])] + ([("bias", ws[1])] if op.use_bias else [])
    cfg = {"units": int(op.units), "activation": "linear" if act == "softmax" else act,
           "use_bias": bool(op.use_bias)}
    return _with_softmax(w, op, w.layer(op.name, "Dense", ins, cfg, weights), act)


def _conv_cfg(op, act):
    return {"kernel_size": _two(op.kernel_size, op.name), "strides": _two(op.strides, op.name),
            "padding": str(op.padding), "activation": "linear" if act == "softmax" else act,
            "use_bias": bool(op.use_bias)}


def _x_conv(w, op, node, ins):
    _conv_checks(op)
    act = _act(op)
    ws = [np.asarray(a) for a in op.get_weights()]
    kind = type(op).__name__
    cfg = _conv_cfg(op, act)
    if kind == "Conv2D":
        cfg["filters"] = int(op.filters)
        weights = [("kernel", ws[0])]
    elif kind == "DepthwiseConv2D":
        weights = [("kernel", ws[0][:, :, :, 0])]          # (kh, kw, c, 1) -> (kh, kw, c)
    else:                                                    # SeparableConv2D
        cfg["filters"] = int(op.filters)
        weights = [("depthwise", ws[0][:, :, :, 0]), ("pointwise", ws[1])]
    if op.use_bias:
        weights.append(("bias", ws[-1]))
    return _with_softmax(w, op, w.layer(op.name, kind, ins, cfg, weights), act)


def _x_bn(w, op, node, ins):
    rank = len(node.input_tensors[0].shape)
    axis = op.axis if isinstance(op.axis, int) else list(op.axis)[0]
    if int(axis) not in (-1, rank - 1):
        raise ExportError(f"{op.name}: BatchNormalization must normalise the channel axis")
    c = int(node.input_tensors[0].shape[-1])
    f64 = lambda v, d: d if v is None else np.asarray(v, np.float64)
    gamma = f64(getattr(op, "gamma", None), np.ones(c)) if getattr(op, "scale", True) else np.ones(c)
    beta = f64(getattr(op, "beta", None), np.zeros(c)) if getattr(op, "center", True) else np.zeros(c)
    mean = np.asarray(op.moving_mean, np.float64)
    var = np.asarray(op.moving_variance, np.float64)
    scale = gamma / np.sqrt(var + float(op.epsilon))
    return w.layer(op.name, "BatchNorm", ins, None,
                   [("scale", scale), ("offset", beta - mean * scale)])


def _x_pool(w, op, node, ins):
    _channels_last(op)
    kind = "MaxPool2D" if type(op).__name__ == "MaxPooling2D" else "AvgPool2D"
    ps, st = _two(op.pool_size, op.name), _two(op.strides or op.pool_size, op.name)
    if st[0] != st[1]:
        raise ExportError(f"{op.name}: non-square strides are unsupported")
    return w.layer(op.name, kind, ins, {"pool_size": ps, "strides": st,
                                        "padding": str(op.padding)})


def _x_gap(w, op, node, ins):
    _channels_last(op)
    if getattr(op, "keepdims", False):
        raise ExportError(f"{op.name}: keepdims=True is unsupported")
    return w.layer(op.name, "GlobalAveragePooling2D", ins)


def _x_activation(w, op, node, ins):
    act = _act(op)
    if act == "softmax":
        return w.layer(op.name, "Softmax", ins)
    return w.layer(op.name, "Activation", ins, {"activation": act})


def _x_relu(w, op, node, ins):
    mv = getattr(op, "max_value", None)
    if float(getattr(op, "negative_slope", 0) or 0) or float(getattr(op, "threshold", 0) or 0):
        raise ExportError(f"{op.name}: leaky / thresholded relu is unsupported")
    if mv is None:
        tag = "relu"
    elif float(mv) == 6.0:
        tag = "relu6"
    else:
        raise ExportError(f"{op.name}: relu clipped at {mv} is unsupported (only 6)")
    return w.layer(op.name, "Activation", ins, {"activation": tag})


def _x_elu(w, op, node, ins):
    if float(getattr(op, "alpha", 1.0)) != 1.0:
        raise ExportError(f"{op.name}: ELU alpha must be 1")
    return w.layer(op.name, "Activation", ins, {"activation": "elu"})


def _x_softmax(w, op, node, ins):
    rank = len(node.input_tensors[0].shape)
    if int(getattr(op, "axis", -1)) not in (-1, rank - 1):
        raise ExportError(f"{op.name}: softmax must run over the channel axis")
    return w.layer(op.name, "Softmax", ins)


def _x_flatten(w, op, node, ins):
    _channels_last(op)
    return w.layer(op.name, "Flatten", ins)


def _x_upsample(w, op, node, ins):
    f = _two(op.size, op.name)
    if f[0] != f[1] or getattr(op, "interpolation", "nearest") != "nearest":
        raise ExportError(f"{op.name}: only square nearest upsampling is supported")
    return w.layer(op.name, "UpSample2D", ins, {"factor": f[0]})


def _x_zeropad(w, op, node, ins):
    _channels_last(op)
    p = op.padding
    if isinstance(p, int):
        pad = [[p, p], [p, p]]
    elif all(isinstance(v, int) for v in p):
        pad = [[int(p[0])] * 2, [int(p[1])] * 2]
    else:
        pad = [[int(a) for a in p[0]], [int(a) for a in p[1]]]
    return w.layer(op.name, "ZeroPadding2D", ins, {"padding": pad})


def _x_concat(w, op, node, ins):
    rank = len(node.input_tensors[0].shape)
    if int(op.axis) not in (-1, rank - 1):
        raise ExportError(f"{op.name}: concatenation must be over the channel axis")
    return w.layer(op.name, "Concatenate", ins)


_CONVERT = {
    "InputLayer": _x_input, "Dense": _x_dense, "Conv2D": _x_conv,
    "DepthwiseConv2D": _x_conv, "SeparableConv2D": _x_conv, "BatchNormalization": _x_bn,
    "MaxPooling2D": _x_pool, "AveragePooling2D": _x_pool,
    "GlobalAveragePooling2D": _x_gap, "Activation": _x_activation, "ReLU": _x_relu,
    "ELU": _x_elu, "Softmax": _x_softmax, "Flatten": _x_flatten,
    "UpSampling2D": _x_upsample, "ZeroPadding2D": _x_zeropad, "Concatenate": _x_concat,
    "Add": lambda w, op, node, ins: w.layer(op.name, "Add", ins),
}


def _topological(model):
    """(operation, node) pairs, every producer before its consumers
    (iterative depth-first walk from the outputs)."""
    if not getattr(model, "inputs", None) or not getattr(model, "outputs", None):
        raise ExportError("the model must be built with a defined input shape")
    order, node_of = [], {}
    stack = [(t, False) for t in reversed(list(model.outputs))]
    while stack:
        t, leaving = stack.pop()
        h = t._keras_history
        op = h.operation
        if leaving:
            order.append((op, op._inbound_nodes[h.node_index]))
            continue
        if h.tensor_index != 0:
            raise ExportError(f"{op.name}: multi-output layers are unsupported")
        if id(op) in node_of:
            if node_of[id(op)] != h.node_index:
                raise ExportError(f"{op.name}: shared layers (applied twice) are unsupported")
            continue
        node_of[id(op)] = h.node_index
        stack.append((t, True))
        for src in reversed(list(op._inbound_nodes[h.node_index].input_tensors)):
            stack.append((src, False))
    return order


def export_model(model):
    """Built Keras model -> (manifest JSON text, blob bytes)."""
    w = _Writer()
    names = {}                                   # id(tensor) -> container layer name
    for op, node in _topological(model):
        kind = type(op).__name__
        ins = [names[id(t)] for t in node.input_tensors]
        out = node.output_tensors[0]
        if kind in _DROPPED:                     # identity at inference
            names[id(out)] = ins[0]
            continue
        conv = _CONVERT.get(kind)
        if conv is None:
            raise ExportError(f"{op.name}: layer type {kind} is not supported "
                              f"(supported: {', '.join(sorted(_CONVERT))})")
        names[id(out)] = conv(w, op, node, ins)
    doc = {"format_version": 1, "layers": w.layers,
           "inputs": [names[id(t)] for t in model.inputs],
           "outputs": [names[id(t)] for t in model.outputs]}
    return json.dumps(doc, indent=1), bytes(w.blob)


def export_to_files(model, manifest_path, blob_path=None):
    """Write ``manifest_path`` and the blob (default: same stem, ``.bin``)."""
    manifest_path = pathlib.Path(manifest_path)
    blob_path = pathlib.Path(blob_path) if blob_path else manifest_path.with_suffix(".bin")
    text, blob = export_model(model)
    manifest_path.write_text(text)
    blob_path.write_bytes(blob)
    return str(manifest_path), str(blob_path)


def main(argv=None):
    """``python -m paper_1906_05737_b200.keras_export model.keras out.json``
    (cli.py of the reference exporter: exit 0, or 2 on any load/convert error)."""
    import argparse
    import sys
    p = argparse.ArgumentParser(prog="nnb-export", description="Keras model -> container files")
    p.add_argument("model")
    p.add_argument("manifest")
    p.add_argument("--weights", default=None)
    a = p.parse_args(argv)
    try:
        import keras
        model = keras.saving.load_model(a.model, compile=False)
        m, b = export_to_files(model, a.manifest, a.weights)
    except (ImportError, ExportError, OSError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    print(f"wrote {m} and {b}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
