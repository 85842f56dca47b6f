"""Loading of the fixtures written by tests/golden/make_golden.py."""

import hashlib
import json
import pathlib

import numpy as np

from paper_1906_05737_b200 import load_weights, parse_manifest, zoo
from paper_1906_05737_b200.model_format import WeightStore

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


def names():
    return sorted(p.stem[4:] for p in GOLDEN.glob("net_*.npz"))


def load(name):
    """(manifest, WeightStore, x, record) for golden net ``name``."""
    rec = dict(np.load(GOLDEN / f"net_{name}.npz"))
    doc = json.loads(bytes(rec["manifest"]).decode())
    manifest = parse_manifest(json.dumps(doc))
    if name.startswith("cfg"):
        cfg = int(name[3])
        _, _, arrays = zoo.build(cfg, reference_compatible=True, with_arrays=True)
        for k, v in arrays.items():
            digest = hashlib.sha256(np.asarray(v, "<f4").tobytes()).digest()
            assert digest == bytes(rec["wsha:" + k]), f"zoo drifted from golden for {k}"
    else:
        arrays = {k[2:]: v for k, v in rec.items() if k.startswith("w:")}
    refs = [r for l in manifest.layers for r in l.weight_refs]
    blob = bytearray(max((r.offset + r.length for r in refs), default=0))
    for r in refs:
        blob[r.offset:r.offset + r.length] = np.asarray(arrays[r.name], "<f4").tobytes()
    if "x" in rec:
        x = rec["x"]
    else:       # a large zoo input, regenerated and checked against its hash
        x = zoo.inputs(int(name[3]), int(rec["xn"][0]))
        assert hashlib.sha256(x.tobytes()).digest() == bytes(rec["xsha"]), "zoo inputs drifted"
    return manifest, load_weights(manifest, bytes(blob)), x, rec


def sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr, "<f4").tobytes()).digest()
