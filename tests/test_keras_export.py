"""Keras exporter (paper_1906_05737_b200/keras_export.py) driven by stand-in
objects: keras is not installed here, and the exporter only reads the
structural attributes a built Keras 3 model exposes (``_keras_history``,
``_inbound_nodes``, layer attributes, ``get_weights()``), so a few classes
with those attributes and the Keras class names stand in for it.  The
exported container is checked against the same network written directly
with the NetBuilder (oracle outputs identical)."""
import json
from collections import namedtuple
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import oracle
from paper_1906_05737_b200 import build_graph, parse_manifest
from paper_1906_05737_b200.keras_export import ExportError, export_model, export_to_files
from paper_1906_05737_b200.model_format import load_model, load_weights
from paper_1906_05737_b200.zoo import NetBuilder

F32 = np.float32
History = namedtuple("History", "operation node_index tensor_index")


class KTensor:
    def __init__(self, shape, op, node_index, tensor_index=0):
        self.shape = tuple(shape)
        self._keras_history = History(op, node_index, tensor_index)


class Node:
    def __init__(self, ins, outs):
        self.input_tensors, self.output_tensors = list(ins), list(outs)


class _Layer:
    def __init__(self, name, weights=(), **attrs):
        self.name, self._w, self._inbound_nodes = name, [np.asarray(w) for w in weights], []
        self.__dict__.update(attrs)

    def get_weights(self):
        return self._w

    def __call__(self, *ins, shape):
        t = KTensor((None,) + tuple(shape), self, len(self._inbound_nodes))
        self._inbound_nodes.append(Node(ins, [t]))
        return t


K = {k: type(k, (_Layer,), {}) for k in (
    "InputLayer", "Dense", "Conv2D", "DepthwiseConv2D", "SeparableConv2D",
    "BatchNormalization", "MaxPooling2D", "AveragePooling2D", "GlobalAveragePooling2D",
    "Activation", "ReLU", "ELU", "Softmax", "Flatten", "UpSampling2D", "ZeroPadding2D",
    "Concatenate", "Add", "Dropout", "LayerNormalization")}


def fn(name):
    return SimpleNamespace(__name__=name)


def keras_input(shape):
    op = K["InputLayer"]("input")
    t = KTensor((None,) + tuple(shape), op, 0)
    op._inbound_nodes.append(Node([], [t]))
    return t


def conv_attrs(k, s=1, pad="same", act="linear", bias=True, **kw):
    return dict(kernel_size=(k, k), strides=(s, s), padding=pad, activation=fn(act),
                use_bias=bias, dilation_rate=(1, 1), data_format="channels_last", **kw)


def he(rng, shape, fan):
    return (rng.standard_normal(shape) * np.sqrt(2.0 / fan)).astype(F32)


def mixed_model(rng):
    """Keras-side graph covering every converter, plus its NetBuilder twin."""
    kw1 = he(rng, (3, 3, 3, 8), 27)
    kb1 = (rng.standard_normal(8) * 0.1).astype(F32)
    gamma, beta = rng.uniform(0.5, 1.5, 8), rng.normal(0, 0.1, 8)
    mean, var = rng.normal(0, 0.1, 8), rng.uniform(0.5, 1.5, 8)
    dk = he(rng, (3, 3, 8, 1), 9)
    pk = he(rng, (1, 1, 8, 16), 8)
    sb = (rng.standard_normal(16) * 0.1).astype(F32)
    dw2 = he(rng, (3, 3, 16, 1), 9)
    c1 = he(rng, (1, 1, 16, 16), 16)
    c1b = np.zeros(16, F32)
    dk2 = he(rng, (16, 10), 16)
    db2 = np.zeros(10, F32)

    x = keras_input((12, 14, 3))
    y = K["ZeroPadding2D"]("zp", padding=((1, 1), (2, 0)), data_format="channels_last")(
        x, shape=(14, 16, 3))
    y = K["Conv2D"]("c1", [kw1, kb1], filters=8, groups=1, **conv_attrs(3, pad="valid", act="relu"))(
        y, shape=(12, 14, 8))
    y = K["BatchNormalization"]("bn", axis=-1, gamma=gamma, beta=beta, moving_mean=mean,
                                moving_variance=var, epsilon=1e-3)(y, shape=(12, 14, 8))
    y = K["ReLU"]("r6", max_value=6.0, negative_slope=0.0, threshold=0.0)(y, shape=(12, 14, 8))
    y = K["SeparableConv2D"]("sep", [dk, pk, sb], filters=16, depth_multiplier=1,
                             **conv_attrs(3, s=2))(y, shape=(6, 7, 16))
    a = K["DepthwiseConv2D"]("dw", [dw2], depth_multiplier=1, **conv_attrs(3, bias=False))(
        y, shape=(6, 7, 16))
    a = K["Activation"]("elu", activation=fn("elu"))(a, shape=(6, 7, 16))
    a = K["Dropout"]("drop")(a, shape=(6, 7, 16))
    b = K["Conv2D"]("c2", [c1, c1b], filters=16, groups=1, **conv_attrs(1))(y, shape=(6, 7, 16))
    z = K["Add"]("add")(a, b, shape=(6, 7, 16))
    z = K["GlobalAveragePooling2D"]("gap", data_format="channels_last", keepdims=False)(
        z, shape=(16,))
    z = K["Dense"]("head", [dk2, db2], units=10, activation=fn("softmax"), use_bias=True)(
        z, shape=(10,))
    model = SimpleNamespace(inputs=[x], outputs=[z])

    nb = NetBuilder()
    t = nb.input((12, 14, 3))
    t = nb.layer("ZeroPadding2D", [t], {"padding": [[1, 1], [2, 0]]})
    t = nb.layer("Conv2D", [t], {"filters": 8, "kernel_size": 3, "padding": "valid",
                                 "activation": "relu"}, [("kernel", kw1), ("bias", kb1)])
    scale = gamma / np.sqrt(var + 1e-3)
    t = nb.layer("BatchNorm", [t], None, [("scale", scale.astype(F32)),
                                          ("offset", (beta - mean * scale).astype(F32))])
    t = nb.layer("Activation", [t], {"activation": "relu6"})
    t = nb.layer("SeparableConv2D", [t], {"filters": 16, "kernel_size": 3, "strides": 2,
                                          "padding": "same"},
                 [("depthwise", dk[:, :, :, 0]), ("pointwise", pk), ("bias", sb)])
    u = nb.layer("DepthwiseConv2D", [t], {"kernel_size": 3, "padding": "same",
                                          "use_bias": False}, [("kernel", dw2[:, :, :, 0])])
    u = nb.layer("Activation", [u], {"activation": "elu"})
    v = nb.layer("Conv2D", [t], {"filters": 16, "kernel_size": 1, "padding": "same"},
                 [("kernel", c1), ("bias", c1b)])
    s = nb.layer("Add", [u, v])
    s = nb.layer("GlobalAveragePooling2D", [s])
    s = nb.layer("Dense", [s], {"units": 10}, [("kernel", dk2), ("bias", db2)])
    s = nb.layer("Softmax", [s])
    return model, nb.build([s])


def test_export_matches_the_directly_written_container(tmp_path):
    model, (m_ref, w_ref) = mixed_model(np.random.default_rng(3))
    text, blob = export_model(model)
    doc = json.loads(text)
    kinds = [l["kind"] for l in doc["layers"]]
    assert kinds == ["Input", "ZeroPadding2D", "Conv2D", "BatchNorm", "Activation",
                     "SeparableConv2D", "DepthwiseConv2D", "Activation", "Conv2D", "Add",
                     "GlobalAveragePooling2D", "Dense", "Softmax"]
    assert "Dropout" not in text
    m = parse_manifest(text)
    w = load_weights(m, blob)
    x = np.random.default_rng(4).random((3, 12, 14, 3), dtype=np.float32)
    got = oracle.run_graph(build_graph(m, w), [x])[0]
    want = oracle.run_graph(build_graph(m_ref, w_ref), [x])[0]
    np.testing.assert_array_equal(got, want)
    mp, bp = export_to_files(model, tmp_path / "net.json")
    m2, w2 = load_model(mp, bp)
    np.testing.assert_array_equal(oracle.run_graph(build_graph(m2, w2), [x])[0], want)


def test_export_rejects_what_the_format_cannot_express():
    x = keras_input((8, 8, 4))
    y = K["LayerNormalization"]("ln")(x, shape=(8, 8, 4))
    with pytest.raises(ExportError, match="not supported"):
        export_model(SimpleNamespace(inputs=[x], outputs=[y]))
    x = keras_input((8, 8, 4))
    y = K["ReLU"]("r", max_value=4.0)(x, shape=(8, 8, 4))
    with pytest.raises(ExportError, match="clipped"):
        export_model(SimpleNamespace(inputs=[x], outputs=[y]))
    x = keras_input((8, 8, 4))
    y = K["Conv2D"]("c", [np.zeros((3, 3, 4, 2)), np.zeros(2)], filters=2, groups=1,
                    **dict(conv_attrs(3), dilation_rate=(2, 2)))(x, shape=(8, 8, 2))
    with pytest.raises(ExportError, match="dilated"):
        export_model(SimpleNamespace(inputs=[x], outputs=[y]))
    x = keras_input((8, 8, 4))
    shared = K["Activation"]("a", activation=fn("relu"))
    y = shared(x, shape=(8, 8, 4))
    z = shared(y, shape=(8, 8, 4))
    with pytest.raises(ExportError, match="shared"):
        export_model(SimpleNamespace(inputs=[x], outputs=[z]))
    x = keras_input((8, 8, 4))
    y = K["Activation"]("a", activation=fn("gelu"))(x, shape=(8, 8, 4))
    with pytest.raises(ExportError, match="gelu"):
        export_model(SimpleNamespace(inputs=[x], outputs=[y]))
    with pytest.raises(ExportError, match="input shape"):
        export_model(SimpleNamespace(inputs=[], outputs=[]))


def test_cli_without_keras_reports_and_exits_2(tmp_path, capsys):
    from paper_1906_05737_b200.keras_export import main
    assert main([str(tmp_path / "m.keras"), str(tmp_path / "o.json")]) == 2
    assert "error" in capsys.readouterr().err
