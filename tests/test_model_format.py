"""Container format: the reference's validation behaviour
(pkg/src/nnjit/model_format.py, pinned by pkg/tests/test_model_format.py)
plus the extended vocabulary."""
import json

import numpy as np
import pytest

from paper_1906_05737_b200 import (load_model, load_weights, manifest_to_json, parse_manifest,
                                   save_model)
from paper_1906_05737_b200.errors import (BlobTooShort, DuplicateName, ManifestSyntaxError,
                                          MissingWeight, ModelFormatError, NonFiniteWeight,
                                          SchemaError, UnknownLayerKind)
from paper_1906_05737_b200 import zoo


def doc(**over):
    d = {"format_version": 1,
         "layers": [{"name": "in", "kind": "Input", "config": {"shape": [4]}},
                    {"name": "sm", "kind": "Softmax", "inputs": ["in"]}],
         "inputs": ["in"], "outputs": ["sm"]}
    d.update(over)
    return d


def parse(d):
    return parse_manifest(json.dumps(d))


def dense_doc(use_bias, n_weights):
    ws = [{"name": f"w{i}", "shape": [4, 2] if i == 0 else [2], "offset": 32 * i,
           "length": 32 if i == 0 else 8} for i in range(n_weights)]
    return {"format_version": 1,
            "layers": [{"name": "in", "kind": "Input", "config": {"shape": [4]}},
                       {"name": "fc", "kind": "Dense", "inputs": ["in"],
                        "config": {"units": 2, "use_bias": use_bias}, "weights": ws}],
            "inputs": ["in"], "outputs": ["fc"]}


def test_minimal_parses_and_defaults():
    m = parse(doc())
    assert [l.name for l in m.layers] == ["in", "sm"]
    assert m.inputs == ("in",) and m.outputs == ("sm",)
    d = parse(dense_doc(True, 2)).layers[1].config
    assert d == {"units": 2, "activation": "linear", "use_bias": True}


@pytest.mark.parametrize("text,exc", [(b"\xff\xfe junk", ManifestSyntaxError),
                                      ("{nope", ManifestSyntaxError), ("[1]", SchemaError),
                                      ("{}", SchemaError), ("null", SchemaError)])
def test_syntax_errors(text, exc):
    with pytest.raises(exc):
        parse_manifest(text)


def test_every_failure_is_a_model_format_error():
    for bad in ("", "1", '{"format_version": 1}', json.dumps(doc(layers=[]))):
        with pytest.raises(ModelFormatError):
            parse_manifest(bad)


@pytest.mark.parametrize("mutate,exc,match", [
    (lambda d: d.update(extra=1), SchemaError, "unknown key"),
    (lambda d: d.update(format_version=2), SchemaError, "format_version"),
    (lambda d: d["layers"][1].update(kind="LSTM"), UnknownLayerKind, "LSTM"),
    (lambda d: d["layers"].append({"name": "sm", "kind": "Softmax", "inputs": ["in"]}),
     DuplicateName, "sm"),
    (lambda d: d["layers"][0]["config"].update(stride=2), SchemaError, "unknown config"),
    (lambda d: d["layers"][1].update(inputs=["in", "in"]), SchemaError, "exactly one input"),
    (lambda d: d["layers"].__setitem__(1, {"name": "sm", "kind": "Add", "inputs": ["in"]}),
     SchemaError, "at least two"),
    (lambda d: d["layers"][0].update(inputs=["sm"]), SchemaError, "no inputs"),
    (lambda d: d.update(outputs=["ghost"]), SchemaError, "not a layer"),
    (lambda d: d.update(outputs=["sm", "sm"]), SchemaError, "repeated"),
    (lambda d: d.update(inputs=["sm"]), SchemaError, "not an Input"),
    (lambda d: d["layers"].insert(0, {"name": "i2", "kind": "Input", "config": {"shape": [2]}}),
     SchemaError, "not listed"),
    (lambda d: d["layers"][0]["config"].update(shape=[2, 2]), SchemaError, "1 or 3"),
    (lambda d: d["layers"][0]["config"].update(shape=[0]), SchemaError, "positive"),
    (lambda d: d["layers"][0]["config"].update(shape=[True]), SchemaError, "positive"),
    (lambda d: d["layers"][1].update(weights=[{"name": "w", "shape": [1], "offset": 0,
                                               "length": 4}]), SchemaError, "carry no weights"),
])
def test_schema_violations(mutate, exc, match):
    d = doc()
    mutate(d)
    with pytest.raises(exc, match=match):
        parse(d)


@pytest.mark.parametrize("layer,match", [
    ({"kind": "Activation", "config": {"activation": "gelu"}}, "gelu"),
    ({"kind": "Conv2D", "config": {"filters": 2}}, "kernel_size"),
    ({"kind": "Conv2D", "config": {"filters": 2, "kernel_size": 3, "strides": [1, 2]}},
     "non-square"),
    ({"kind": "Conv2D", "config": {"filters": 2, "kernel_size": 3, "padding": "full"}},
     "padding"),
    ({"kind": "MaxPool2D", "config": {"pool_size": [2, 3]}}, "explicit strides"),
    ({"kind": "Dense", "config": {"units": 2, "use_bias": 1}}, "boolean"),
    ({"kind": "UpSample2D", "config": {}}, "factor"),
    ({"kind": "ZeroPadding2D", "config": {"padding": [[1, 2, 3]]}}, "padding"),
])
def test_config_validation(layer, match):
    d = doc()
    d["layers"][1] = dict(layer, name="x", inputs=["in"])
    d["outputs"] = ["x"]
    with pytest.raises(SchemaError, match=match):
        parse(d)


def test_pool_default_stride_and_rectangular_with_strides():
    d = doc()
    d["layers"] = [{"name": "in", "kind": "Input", "config": {"shape": [6, 6, 1]}},
                   {"name": "p", "kind": "MaxPool2D", "inputs": ["in"],
                    "config": {"pool_size": 3}},
                   {"name": "q", "kind": "AvgPool2D", "inputs": ["p"],
                    "config": {"pool_size": [2, 1], "strides": 1}}]
    d["outputs"] = ["q"]
    m = parse(d)
    assert m.layers[1].config["strides"] == 3
    assert m.layers[2].config["pool_size"] == (2, 1)


def test_extended_vocabulary_parses():
    d = doc()
    d["layers"] = [{"name": "in", "kind": "Input", "config": {"shape": [6, 6, 2]}},
                   {"name": "a", "kind": "Activation", "inputs": ["in"],
                    "config": {"activation": "relu6"}},
                   {"name": "e", "kind": "Activation", "inputs": ["a"],
                    "config": {"activation": "elu"}},
                   {"name": "z", "kind": "ZeroPadding2D", "inputs": ["e"], "config": {"padding": 1}},
                   {"name": "g", "kind": "GlobalAveragePooling2D", "inputs": ["z"]}]
    d["outputs"] = ["g"]
    m = parse(d)
    assert m.layers[3].config["padding"] == ((1, 1), (1, 1))


def test_weight_ref_checks():
    for ref, match in (({"name": "w", "shape": [4, 2], "offset": 0, "length": 16}, "length"),
                       ({"name": "w", "shape": [4, 2], "offset": 2, "length": 32}, "align"),
                       ({"name": "w", "shape": [], "offset": 0, "length": 4}, "non-empty"),
                       ({"name": "w", "shape": [4, 2], "offset": -4, "length": 32}, "offset"),
                       ({"name": "w", "shape": [4, 2], "offset": 0}, "length")):
        d = dense_doc(False, 1)
        d["layers"][1]["weights"] = [ref]
        with pytest.raises(SchemaError, match=match):
            parse(d)
    d = dense_doc(True, 2)
    d["layers"][1]["weights"][1]["name"] = "w0"
    with pytest.raises(DuplicateName):
        parse(d)


def test_weight_arity_blob_and_finiteness():
    blob = bytes(64)
    load_weights(parse(dense_doc(True, 2)), blob)
    load_weights(parse(dense_doc(False, 1)), blob)
    with pytest.raises(MissingWeight):
        load_weights(parse(dense_doc(True, 1)), blob)
    with pytest.raises(MissingWeight):
        load_weights(parse(dense_doc(False, 2)), blob)
    with pytest.raises(BlobTooShort):
        load_weights(parse(dense_doc(False, 1)), bytes(16))
    with pytest.raises(NonFiniteWeight):
        load_weights(parse(dense_doc(False, 1)), np.full(10, np.inf, "<f4").tobytes())
    with pytest.raises(TypeError):
        load_weights(parse(dense_doc(False, 1)), "not bytes")


def test_weights_are_readonly_float32_in_declared_shape():
    m, w = zoo.build(0)
    for name in w.names():
        arr = w[name]
        assert arr.dtype == np.float32 and not arr.flags.writeable


@pytest.mark.parametrize("cfg", range(5))
def test_round_trip_json_and_files(cfg, tmp_path):
    m, w, arrays = zoo.build(cfg, with_arrays=True)
    assert parse_manifest(manifest_to_json(m)) == m
    save_model(m, arrays, tmp_path / "net.json")
    m2, w2 = load_model(tmp_path / "net.json")
    assert m2 == m
    for n in w.names():
        np.testing.assert_array_equal(w[n], w2[n])


def test_save_model_rejects_wrong_shape(tmp_path):
    m, w, arrays = zoo.build(1, with_arrays=True)
    k = next(iter(arrays))
    arrays[k] = arrays[k].reshape(-1)
    with pytest.raises(ValueError):
        save_model(m, arrays, tmp_path / "x.json")
