"""Graph building and shape inference (pkg/src/nnjit/graph.py semantics)."""
import json

import numpy as np
import pytest

from builders import conv_net, he
from paper_1906_05737_b200 import build_graph, parse_manifest, zoo
from paper_1906_05737_b200.errors import (CycleDetected, ShapeMismatch, UnknownInput,
                                          WeightShapeMismatch)
from paper_1906_05737_b200.graph import same_padding
from paper_1906_05737_b200.zoo import NetBuilder

F32 = np.float32


@pytest.mark.parametrize("size,kernel,stride,expect", [
    (5, 3, 1, (1, 1)), (5, 3, 2, (1, 1)), (6, 3, 2, (0, 1)), (7, 5, 3, (2, 2)),
    (4, 1, 1, (0, 0)), (3, 7, 1, (3, 3)), (10, 2, 2, (0, 0)), (2, 4, 2, (1, 1)),
    (1, 3, 1, (1, 1))])
def test_same_padding_tf_split(size, kernel, stride, expect):
    assert same_padding(size, kernel, stride) == expect


def shapes(m, w):
    g = build_graph(m, w)
    return {n.name: n.output_shape.dims for n in g.nodes}


@pytest.mark.parametrize("cfg,out", [(0, (2,)), (1, (10,)), (2, (4,)), (3, (1000,)),
                                     (4, (120, 160, 3))])
def test_zoo_output_shapes(cfg, out):
    m, w = zoo.build(cfg)
    g = build_graph(m, w)
    assert g.nodes[g.output_ids[0]].output_shape.dims == out


def test_shape_rules_chain():
    rng = np.random.default_rng(0)
    b = NetBuilder()
    x = b.input((11, 9, 3))
    c = b.layer("Conv2D", [x], {"filters": 8, "kernel_size": 3, "strides": 2, "padding": "same"},
                [("kernel", he(rng, (3, 3, 3, 8), 27)), ("bias", np.zeros(8, F32))])
    v = b.layer("Conv2D", [c], {"filters": 4, "kernel_size": [3, 2], "padding": "valid"},
                [("kernel", he(rng, (3, 2, 8, 4), 48)), ("bias", np.zeros(4, F32))])
    p = b.layer("MaxPool2D", [v], {"pool_size": 2, "strides": 2, "padding": "same"})
    u = b.layer("UpSample2D", [p], {"factor": 3})
    z = b.layer("ZeroPadding2D", [u], {"padding": [[1, 0], [2, 3]]})
    cat = b.layer("Concatenate", [z, z])
    g = b.layer("GlobalAveragePooling2D", [cat])
    s = b.layer("Softmax", [g])
    f = b.layer("Flatten", [cat])
    m, w = b.build([s, f])
    sh = shapes(m, w)
    assert sh[c] == (6, 5, 8) and sh[v] == (4, 4, 4) and sh[p] == (2, 2, 4)
    assert sh[u] == (6, 6, 4) and sh[z] == (7, 11, 4) and sh[cat] == (7, 11, 8)
    assert sh[g] == (8,) and sh[s] == (8,) and sh[f] == (7 * 11 * 8,)


def _graph_error(build, exc):
    b = NetBuilder()
    out = build(b)
    m, w = b.build([out])
    with pytest.raises(exc):
        build_graph(m, w)


def test_shape_errors():
    rng = np.random.default_rng(1)
    _graph_error(lambda b: b.layer("Conv2D", [b.input((2, 2, 1))],
                                   {"filters": 1, "kernel_size": 3, "padding": "valid"},
                                   [("kernel", he(rng, (3, 3, 1, 1), 9)),
                                    ("bias", np.zeros(1, F32))]), ShapeMismatch)
    _graph_error(lambda b: b.layer("Dense", [b.input((2, 2, 1))], {"units": 2},
                                   [("kernel", np.zeros((4, 2), F32)),
                                    ("bias", np.zeros(2, F32))]), ShapeMismatch)
    _graph_error(lambda b: b.layer("Conv2D", [b.input((4,))],
                                   {"filters": 1, "kernel_size": 1},
                                   [("kernel", np.zeros((1, 1, 4, 1), F32)),
                                    ("bias", np.zeros(1, F32))]), ShapeMismatch)
    _graph_error(lambda b: b.layer("Conv2D", [b.input((4, 4, 2))],
                                   {"filters": 1, "kernel_size": 1},
                                   [("kernel", np.zeros((1, 1, 3, 1), F32)),
                                    ("bias", np.zeros(1, F32))]), WeightShapeMismatch)
    _graph_error(lambda b: b.layer("BatchNorm", [b.input((4, 4, 2))], None,
                                   [("scale", np.ones(3, F32)), ("offset", np.ones(3, F32))]),
                 WeightShapeMismatch)
    _graph_error(lambda b: b.layer("UpSample2D", [b.input((4,))], {"factor": 2}), ShapeMismatch)
    _graph_error(lambda b: b.layer("GlobalAveragePooling2D", [b.input((4,))]), ShapeMismatch)


def test_add_and_concat_shape_checks():
    def add(b):
        x = b.input((4, 4, 2))
        p = b.layer("MaxPool2D", [x], {"pool_size": 2})
        return b.layer("Add", [x, p])
    _graph_error(add, ShapeMismatch)

    def cat(b):
        x = b.input((4, 4, 2))
        p = b.layer("MaxPool2D", [x], {"pool_size": 2})
        return b.layer("Concatenate", [x, p])
    _graph_error(cat, ShapeMismatch)


def test_unknown_input_and_cycle():
    d = {"format_version": 1, "layers": [
        {"name": "in", "kind": "Input", "config": {"shape": [3]}},
        {"name": "a", "kind": "Activation", "inputs": ["ghost"], "config": {"activation": "relu"}}],
         "inputs": ["in"], "outputs": ["a"]}
    with pytest.raises(UnknownInput):
        build_graph(parse_manifest(json.dumps(d)), None)
    d["layers"] = [d["layers"][0],
                   {"name": "a", "kind": "Add", "inputs": ["in", "b"]},
                   {"name": "b", "kind": "Activation", "inputs": ["a"],
                    "config": {"activation": "relu"}}]
    with pytest.raises(CycleDetected):
        build_graph(parse_manifest(json.dumps(d)), None)


def test_order_topological_with_manifest_tiebreak():
    d = {"format_version": 1, "layers": [
        {"name": "z", "kind": "Add", "inputs": ["y", "x"]},
        {"name": "in", "kind": "Input", "config": {"shape": [3]}},
        {"name": "y", "kind": "Activation", "inputs": ["in"], "config": {"activation": "relu"}},
        {"name": "x", "kind": "Activation", "inputs": ["in"], "config": {"activation": "tanh"}}],
         "inputs": ["in"], "outputs": ["z"]}
    g = build_graph(parse_manifest(json.dumps(d)), None)
    assert [g.nodes[i].name for i in g.order] == ["in", "y", "x", "z"]
    assert g.consumers[1] == [2, 3]
    assert build_graph(parse_manifest(json.dumps(d)), None).order == g.order


def test_conv_weight_layout_cross_check():
    rng = np.random.default_rng(2)
    m, w = conv_net(rng, 5, 5, 3, 4, k=(3, 2))
    g = build_graph(m, w)
    assert g.nodes[1].output_shape.dims == (5, 5, 4)
