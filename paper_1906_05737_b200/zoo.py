"""The five BASELINE.json configurations, generated directly in container form.

Keras and the paper's evaluation networks are not available (SURVEY.md
section 8(c)), so every net is synthesised here with seeded weights, exactly
as BASELINE.md section 2 specifies:

* weights ``numpy.random.default_rng(0)``, inputs ``default_rng(1)``;
* He-normal ``N(0, 2/fan_in)`` (fan_in = kh*kw*cin for Conv2D, kh*kw for
  DepthwiseConv2D, in for Dense), Glorot-uniform + zero bias for cfg1,
  zero conv/dense biases elsewhere (Keras defaults);
* BatchNorm gamma U[0.5,1.5], beta N(0,0.1), moving mean N(0,0.1), moving
  variance U[0.5,1.5], eps 1e-3, folded to scale/offset in float64 the way the
  reference exporter does (pkg/keras-exporter/src/nnjit_keras_export/
  export.py:163-169).

Frozen interpretations of the ambiguous spec text:

* cfg2 -- blocks are ``DepthwiseConv2D(3x3, no bias) -> Conv2D 1x1 -> BN ->
  ReLU``; strides 2 on the 2nd and 4th blocks; the residual Add is on the 3rd
  block (15x20x64 -> 15x20x64, the only block whose shapes match); the head is
  GlobalAveragePooling -> Dense 4.
* cfg4 -- the decoder concatenates the *pre-pool* encoder activations
  (60x80x64, then 120x160x32); ZeroPadding2D is an identity at 240x320 (every
  pooled size is even) and is not emitted.

``reference_compatible=True`` re-encodes a config in the reference's own
vocabulary (GAP -> AvgPool2D + Flatten) and, where the reference has no
equivalent, substitutes the cost stand-ins of BASELINE.md section 2
(ELU -> tanh, ReLU6 -> ReLU, per-pixel softmax dropped).
"""

import json

import numpy as np

from .model_format import load_weights, parse_manifest

F32 = np.float32

CONFIGS = {
    0: dict(name="cfg0_patch_cnn", batches=(1, 4096)),
    1: dict(name="cfg1_mlp", batches=(1, 65536)),
    2: dict(name="cfg2_dwsep_encoder", batches=(1, 1024)),
    3: dict(name="cfg3_mobilenetv1_025", batches=(1, 256)),
    4: dict(name="cfg4_seg_encdec", batches=(1, 64)),
}


class NetBuilder:
    """Accumulates layers + a weight blob; ``build()`` goes through the public
    parser so a zoo net is exactly what a user-supplied file would be."""

    def __init__(self, seed=0, reference_compatible=False):
        self.rng = np.random.default_rng(seed)
        self.ref = reference_compatible
        self.layers = []
        self.blob = bytearray()
        self.arrays = {}
        self._n = 0

    def _name(self, stem):
        self._n += 1
        return f"{stem}{self._n}"

    def _weight(self, lname, role, arr):
        arr = np.ascontiguousarray(arr, dtype="<f4")
        ref = {"name": f"{lname}.{role}", "shape": list(arr.shape),
               "offset": len(self.blob), "length": arr.nbytes}
        self.blob += arr.tobytes()
        self.arrays[ref["name"]] = arr
        return ref

    def layer(self, kind, inputs=(), config=None, weights=(), name=None):
        name = name or self._name(kind.lower())
        obj = {"name": name, "kind": kind}
        if inputs:
            obj["inputs"] = list(inputs)
        if config:
            obj["config"] = config
        if weights:
            obj["weights"] = [self._weight(name, r, a) for r, a in weights]
        self.layers.append(obj)
        return name

    # -- initialisers --------------------------------------------------------
    def he(self, shape, fan_in):
        return (self.rng.standard_normal(shape) * np.sqrt(2.0 / fan_in)).astype(F32)

    def glorot(self, fan_in, fan_out):
        lim = np.sqrt(6.0 / (fan_in + fan_out))
        return self.rng.uniform(-lim, lim, size=(fan_in, fan_out)).astype(F32)

    # -- layer helpers -------------------------------------------------------
    def input(self, shape):
        return self.layer("Input", config={"shape": list(shape)}, name="input")

    def conv(self, x, cin, cout, k=3, stride=1, padding="same", act="linear", bias=True):
        w = [("kernel", self.he((k, k, cin, cout), k * k * cin))]
        if bias:
            w.append(("bias", np.zeros(cout, F32)))
        return self.layer("Conv2D", [x], {"filters": cout, "kernel_size": k, "strides": stride,
                                          "padding": padding, "activation": self.act(act),
                                          "use_bias": bias}, w)

    def dwconv(self, x, c, k=3, stride=1, padding="same", bias=False):
        w = [("kernel", self.he((k, k, c), k * k))]
        if bias:
            w.append(("bias", np.zeros(c, F32)))
        return self.layer("DepthwiseConv2D", [x], {"kernel_size": k, "strides": stride,
                                                   "padding": padding, "use_bias": bias}, w)

    def dense(self, x, nin, nout, act="linear", init="he"):
        k = self.glorot(nin, nout) if init == "glorot" else self.he((nin, nout), nin)
        return self.layer("Dense", [x], {"units": nout, "activation": self.act(act)},
                          [("kernel", k), ("bias", np.zeros(nout, F32))])

    def bn(self, x, c, eps=1e-3):
        gamma = self.rng.uniform(0.5, 1.5, c)
        beta = self.rng.normal(0.0, 0.1, c)
        mean = self.rng.normal(0.0, 0.1, c)
        var = self.rng.uniform(0.5, 1.5, c)
        scale = gamma / np.sqrt(var + eps)
        offset = beta - mean * scale
        return self.layer("BatchNorm", [x], None,
                          [("scale", scale.astype(F32)), ("offset", offset.astype(F32))])

    def act(self, tag):
        if self.ref and tag == "elu":
            return "tanh"
        if self.ref and tag == "relu6":
            return "relu"
        return tag

    def activation(self, x, tag):
        return self.layer("Activation", [x], {"activation": self.act(tag)})

    def maxpool(self, x):
        return self.layer("MaxPool2D", [x], {"pool_size": 2, "strides": 2})

    def gap(self, x, h, w):
        if self.ref:
            p = self.layer("AvgPool2D", [x], {"pool_size": [h, w], "strides": 1,
                                              "padding": "valid"})
            return self.layer("Flatten", [p])
        return self.layer("GlobalAveragePooling2D", [x])

    def softmax(self, x, per_pixel=False):
        if per_pixel and self.ref:
            return x
        return self.layer("Softmax", [x])

    def build(self, outputs):
        doc = {"format_version": 1, "layers": self.layers, "inputs": ["input"],
               "outputs": list(outputs)}
        manifest = parse_manifest(json.dumps(doc))
        return manifest, load_weights(manifest, bytes(self.blob))


def cfg0(b):
    x = b.input((32, 32, 1))
    c = 1
    for f in (8, 16, 16):
        x = b.conv(x, c, f)
        x = b.bn(x, f)
        x = b.activation(x, "relu")
        x = b.maxpool(x)
        c = f
    x = b.layer("Flatten", [x])
    x = b.dense(x, 256, 32, "relu")
    x = b.dense(x, 32, 2)
    return b.softmax(x)


def cfg1(b):
    x = b.input((1024,))
    x = b.dense(x, 1024, 512, "tanh", init="glorot")
    x = b.dense(x, 512, 256, "sigmoid", init="glorot")
    x = b.dense(x, 256, 128, "elu", init="glorot")
    x = b.dense(x, 128, 10, init="glorot")
    return b.softmax(x)


def cfg2(b):
    x = b.input((60, 80, 3))
    x = b.conv(x, 3, 16, stride=2)
    x = b.activation(b.bn(x, 16), "relu")
    c = 16
    for i, (f, s) in enumerate(((32, 1), (64, 2), (64, 1), (128, 2))):
        block_in = x
        y = b.dwconv(x, c, stride=s)
        y = b.conv(y, c, f, k=1, padding="valid", bias=False)
        y = b.activation(b.bn(y, f), "relu")
        if i == 2:
            y = b.layer("Add", [block_in, y])
        x, c = y, f
    x = b.gap(x, 8, 10)
    return b.dense(x, 128, 4)


MOBILENET_BLOCKS = ((16, 1), (32, 2), (32, 1), (64, 2), (64, 1), (128, 2), (128, 1),
                    (128, 1), (128, 1), (128, 1), (128, 1), (256, 2), (256, 1))


def cfg3(b):
    x = b.input((128, 128, 3))
    x = b.conv(x, 3, 8, stride=2, bias=False)
    x = b.activation(b.bn(x, 8), "relu6")
    c = 8
    for f, s in MOBILENET_BLOCKS:
        x = b.dwconv(x, c, stride=s)
        x = b.activation(b.bn(x, c), "relu6")
        x = b.conv(x, c, f, k=1, padding="valid", bias=False)
        x = b.activation(b.bn(x, f), "relu6")
        c = f
    x = b.gap(x, 4, 4)
    x = b.dense(x, 256, 1000)
    return b.softmax(x)


def cfg4(b):
    x = b.input((240, 320, 3))
    skips = []
    c = 3
    for f in (16, 32, 64):
        x = b.conv(x, c, f)
        x = b.activation(b.bn(x, f), "relu")
        skips.append(x)
        x = b.maxpool(x)
        c = f
    # decoder: up x2, concat the matching pre-pool skip, conv 3x3
    for f, skip, cs in ((32, skips[2], 64), (16, skips[1], 32)):
        up = b.layer("UpSample2D", [x], {"factor": 2})
        x = b.layer("Concatenate", [up, skip])
        x = b.conv(x, c + cs, f, act="relu")
        c = f
    x = b.conv(x, c, 3, k=1, padding="valid")
    return b.softmax(x, per_pixel=True)


_GEN = {0: cfg0, 1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4}
INPUT_SHAPES = {0: (32, 32, 1), 1: (1024,), 2: (60, 80, 3), 3: (128, 128, 3),
                4: (240, 320, 3)}


def build(cfg, seed=0, reference_compatible=False, with_arrays=False):
    """(manifest, WeightStore) for BASELINE config ``cfg`` (0..4)."""
    b = NetBuilder(seed, reference_compatible)
    out = _GEN[cfg](b)
    manifest, store = b.build([out])
    if with_arrays:
        return manifest, store, b.arrays
    return manifest, store


def inputs(cfg, n, seed=1):
    """``n`` seeded input images: U[0,1) (cfg1: N(0,1)), float32."""
    rng = np.random.default_rng(seed)
    shape = (n,) + INPUT_SHAPES[cfg]
    if cfg == 1:
        return rng.standard_normal(shape).astype(F32)
    return rng.random(shape, dtype=np.float32)
