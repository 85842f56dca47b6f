"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference package ``nnjit`` and records, for seeded inputs:

* ``net_<net>.npz`` ``interp`` -- reference interpreter outputs (oracle A) for a set
  of reference-expressible networks (single-layer sweeps, a small classifier,
  and the reference-compatible encodings of BASELINE configs 0-4);
* ``compiled_*``         -- the reference's compiled x86 path under its default
  options, ``softmax_exp="precise"`` and ``activation_mode="fast"`` (oracle B);
* ``approx.npz``         -- the reference's bit-faithful approximation models
  (pkg/src/nnjit/codegen/approx.py:72-128) on a fixed grid;
* ``plan:*`` entries     -- SHA-256 of the folded weights/biases/post-affines
  of the reference fusion planner (pkg/src/nnjit/optimizer.py) per unit.

Every network is written as manifest JSON + weight arrays so the fixtures are
self-contained on machines without the reference (the GPU box).
"""

import hashlib
import json
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

import nnjit  # noqa: E402  (the reference; needs PYTHONPATH)
from nnjit.codegen import approx as ref_approx  # noqa: E402

from paper_1906_05737_b200 import zoo  # noqa: E402
from paper_1906_05737_b200.model_format import manifest_to_json  # noqa: E402

F32 = np.float32


def nets():
    """name -> (manifest, arrays, input shape, inputs U(-2,2) or zoo inputs)."""
    out = {}
    rng = np.random.default_rng(1234)

    def add(name, b, shape, n=3, inputs=None):
        doc = {"format_version": 1, "layers": b.layers, "inputs": ["input"],
               "outputs": [b.layers[-1]["name"]]}
        x = inputs if inputs is not None else rng.uniform(-2, 2, (n,) + shape).astype(F32)
        arrays = dict(b.arrays)
        for k in arrays:                      # non-trivial biases
            if k.endswith(".bias"):
                arrays[k] = (rng.standard_normal(arrays[k].shape) * 0.1).astype(F32)
        out[name] = (doc, arrays, x)

    # single-layer sweeps over irregular sizes
    for i, (h, w, ci, co, k, s, pad, act) in enumerate([
            (7, 9, 3, 5, 3, 1, "same", "relu"), (8, 6, 4, 8, 3, 2, "same", "tanh"),
            (5, 5, 2, 3, 2, 1, "valid", "sigmoid"), (9, 7, 1, 4, 3, 2, "valid", "linear"),
            (6, 6, 5, 7, 1, 1, "valid", "relu"), (10, 12, 8, 16, 3, 1, "same", "relu")]):
        b = zoo.NetBuilder(seed=100 + i)
        x = b.input((h, w, ci))
        b.conv(x, ci, co, k=k, stride=s, padding=pad, act=act, bias=i % 2 == 0)
        add(f"conv{i}", b, (h, w, ci))
    for i, (h, w, c, k, s, pad) in enumerate([(7, 9, 3, 3, 1, "same"), (8, 8, 8, 3, 2, "same"),
                                              (6, 5, 5, 2, 1, "valid")]):
        b = zoo.NetBuilder(seed=200 + i)
        x = b.input((h, w, c))
        b.dwconv(x, c, k=k, stride=s, padding=pad, bias=True)
        add(f"dw{i}", b, (h, w, c))
    for i, (kin, units, act) in enumerate([(5, 3, "relu"), (64, 33, "tanh"), (130, 7, "sigmoid"),
                                           (17, 1, "linear")]):
        b = zoo.NetBuilder(seed=300 + i)
        x = b.input((kin,))
        b.dense(x, kin, units, act)
        add(f"dense{i}", b, (kin,))
    for i, (op, h, w, c, p, s, pad) in enumerate([("MaxPool2D", 7, 9, 3, 2, 2, "same"),
                                                  ("AvgPool2D", 7, 9, 3, 3, 2, "same"),
                                                  ("AvgPool2D", 6, 6, 4, 2, 1, "valid"),
                                                  ("MaxPool2D", 5, 7, 2, 3, 1, "same")]):
        b = zoo.NetBuilder(seed=400 + i)
        x = b.input((h, w, c))
        b.layer(op, [x], {"pool_size": p, "strides": s, "padding": pad})
        add(f"pool{i}", b, (h, w, c))
    for i, tag in enumerate(["relu", "tanh", "sigmoid"]):
        b = zoo.NetBuilder(seed=500 + i)
        x = b.input((37,))
        b.layer("Activation", [x], {"activation": tag})
        add(f"act_{tag}", b, (37,), n=4)
    b = zoo.NetBuilder(seed=600)
    x = b.input((33,))
    b.layer("Softmax", [x])
    add("softmax", b, (33,), n=4)
    b = zoo.NetBuilder(seed=601)
    x = b.input((4, 5, 6))
    b.bn(x, 6)
    add("batchnorm", b, (4, 5, 6))
    b = zoo.NetBuilder(seed=602)
    x = b.input((3, 4, 5))
    b.layer("UpSample2D", [x], {"factor": 2})
    add("upsample", b, (3, 4, 5))
    # a small classifier with fan-out, concat and add (graph-level golden)
    b = zoo.NetBuilder(seed=700)
    x = b.input((16, 16, 2))
    c1 = b.conv(x, 2, 6, act="relu")
    c2 = b.conv(c1, 6, 6)
    c3 = b.conv(c1, 6, 6, act="tanh")
    a = b.layer("Add", [c2, c3])
    bn = b.bn(a, 6)
    p = b.maxpool(bn)
    cat = b.layer("Concatenate", [p, b.conv(p, 6, 4, act="sigmoid")])
    f = b.layer("Flatten", [cat])
    d = b.dense(f, 8 * 8 * 10, 12, "relu")
    b.softmax(b.dense(d, 12, 5))
    add("mixed_net", b, (16, 16, 2), n=3)
    # the BASELINE configs in reference vocabulary (cost stand-ins: ELU -> tanh,
    # ReLU6 -> ReLU, cfg4's per-pixel softmax omitted); cfg4 on one image
    # (its interpreter run takes ~1 s per image)
    for cfg in range(5):
        m, store, arrs = zoo.build(cfg, reference_compatible=True, with_arrays=True)
        doc = json.loads(manifest_to_json(m))
        out[f"cfg{cfg}_ref"] = (doc, arrs, zoo.inputs(cfg, 1 if cfg == 4 else 2))
    return out


def to_reference(doc, arrays):
    m = nnjit.parse_manifest(json.dumps(doc))
    refs = [r for l in m.layers for r in l.weight_refs]
    blob = bytearray(max((r.offset + r.length for r in refs), default=0))
    for r in refs:
        blob[r.offset:r.offset + r.length] = np.asarray(arrays[r.name], "<f4").tobytes()
    return m, nnjit.load_weights(m, bytes(blob))


def main(only=None):
    results = {}
    for name, (doc, arrays, x) in nets().items():
        if only and name not in only:
            continue
        m, w = to_reference(doc, arrays)
        g = nnjit.build_graph(m, w)
        interp = np.stack([nnjit.interpret(g, [xi])[0] for xi in x])
        rec = {"manifest": np.frombuffer(json.dumps(doc).encode(), np.uint8), "interp": interp}
        if x.nbytes > 256 * 1024:
            # large zoo inputs are regenerated by tests/golden_util.py from
            # zoo.inputs(cfg, n) and pinned by hash instead of stored
            rec["xsha"] = np.frombuffer(hashlib.sha256(x.tobytes()).digest(), np.uint8)
            rec["xn"] = np.array([len(x)])
        else:
            rec["x"] = x
        if name.startswith("cfg"):
            # regenerated from paper_1906_05737_b200.zoo; pin the bytes by hash
            for k, v in arrays.items():
                rec["wsha:" + k] = np.frombuffer(
                    hashlib.sha256(np.asarray(v, "<f4").tobytes()).digest(), np.uint8)
        else:
            for k, v in arrays.items():
                rec["w:" + k] = v
        for tag, opts in (("compiled_default", nnjit.ApproximationOptions()),
                          ("compiled_precise", nnjit.ApproximationOptions(softmax_exp="precise")),
                          ("compiled_fast", nnjit.ApproximationOptions(activation_mode="fast"))):
            net = nnjit.CompiledNetwork(m, w, opts)
            ys = []
            for xi in x:
                ys.append(np.array(net.run([xi])[0]))
            rec[tag] = np.stack(ys)
        plan = nnjit.build_plan(g)
        for i, u in enumerate(plan.units):
            for fld in ("kernel", "bias", "post_scale", "post_offset", "scale", "offset"):
                v = getattr(u, fld)
                if v is not None:   # folded arrays pinned bit-for-bit by hash
                    rec[f"plan:{i}:{u.kind}:{fld}"] = np.frombuffer(
                        hashlib.sha256(np.ascontiguousarray(v, "<f4").tobytes()).digest(),
                        np.uint8)
            rec[f"plan:{i}:{u.kind}:act"] = np.frombuffer(u.activation.encode(), np.uint8)
        np.savez_compressed(HERE / f"net_{name}.npz", **rec)
        results[name] = interp.shape
    if only:
        print(json.dumps({k: list(v) for k, v in results.items()}))
        return
    # approximation models on a fixed grid, incl. saturation and clamp edges
    grid = np.concatenate([np.linspace(-12, 12, 4001), [0.0, -0.0, 1.0, 5.7, -5.7, 80, -80, 90,
                                                        -90, 1e-8, -1e-8]]).astype(F32)
    np.savez_compressed(
        HERE / "approx.npz", x=grid,
        tanh_rational=ref_approx.tanh_model(grid), sigmoid_rational=ref_approx.sigmoid_model(grid),
        tanh_fast=ref_approx.fast_tanh_model(grid), sigmoid_fast=ref_approx.fast_sigmoid_model(grid),
        exp_fast=ref_approx.fast_exp_model(grid), exp_precise=ref_approx.exp_precise_model(grid),
        pade_at_clamp=np.array([ref_approx.PADE_AT_CLAMP], F32),
        sat_delta=np.array([ref_approx.SAT_DELTA], F32))
    print(json.dumps({k: list(v) for k, v in results.items()}))


if __name__ == "__main__":
    main(sys.argv[1:] or None)      # optional: names of the nets to (re)generate
