"""Seeded model generators for the test-suite (all go through the public
container parser via zoo.NetBuilder)."""

import numpy as np

from paper_1906_05737_b200.zoo import NetBuilder

F32 = np.float32
ACTS = ("linear", "relu", "tanh", "sigmoid", "relu6", "elu")


def he(rng, shape, fan_in):
    return (rng.standard_normal(shape) * np.sqrt(2.0 / fan_in)).astype(F32)


def single(kind, in_shape, config=None, weights=(), seed=0):
    b = NetBuilder(seed=seed)
    x = b.input(in_shape)
    y = b.layer(kind, [x], config, weights)
    return b.build([y])


def dense_net(rng, k, units, act="relu", bias=True):
    b = NetBuilder()
    x = b.input((k,))
    w = [("kernel", he(rng, (k, units), k))]
    if bias:
        w.append(("bias", (rng.standard_normal(units) * 0.1).astype(F32)))
    y = b.layer("Dense", [x], {"units": units, "activation": act, "use_bias": bias}, w)
    return b.build([y])


def conv_net(rng, h, w, ci, co, k=3, stride=1, padding="same", act="relu", bias=True,
             depthwise=False):
    b = NetBuilder()
    x = b.input((h, w, ci))
    kh, kw = (k, k) if isinstance(k, int) else k
    if depthwise:
        wt = [("kernel", he(rng, (kh, kw, ci), kh * kw))]
        if bias:
            wt.append(("bias", (rng.standard_normal(ci) * 0.1).astype(F32)))
        y = b.layer("DepthwiseConv2D", [x], {"kernel_size": [kh, kw], "strides": stride,
                                             "padding": padding, "activation": act,
                                             "use_bias": bias}, wt)
    else:
        wt = [("kernel", he(rng, (kh, kw, ci, co), kh * kw * ci))]
        if bias:
            wt.append(("bias", (rng.standard_normal(co) * 0.1).astype(F32)))
        y = b.layer("Conv2D", [x], {"filters": co, "kernel_size": [kh, kw], "strides": stride,
                                    "padding": padding, "activation": act, "use_bias": bias}, wt)
    return b.build([y])


def bn_params(rng, c):
    return [("scale", (rng.standard_normal(c) * 0.3 + 1.0).astype(F32)),
            ("offset", (rng.standard_normal(c) * 0.2).astype(F32))]


def random_network(rng, max_layers=8, extended=True):
    """A random DAG: conv / depthwise / BN / activation / pool chains with
    branch-and-merge (Add, Concatenate), ending in Flatten -> Dense
    (-> Softmax).  ``extended`` also draws relu6/elu/GAP/zero-padding."""
    b = NetBuilder(seed=int(rng.integers(1 << 30)))
    h, w, c = int(rng.integers(6, 14)), int(rng.integers(6, 14)), int(rng.integers(1, 6))
    cur = b.input((h, w, c))
    acts = ACTS if extended else ACTS[:4]

    def conv(src, shape, cout, act, pad=None, k=None):
        kh = k or int(rng.integers(1, min(4, shape[0] + 1)))
        kw = k or int(rng.integers(1, min(4, shape[1] + 1)))
        pad = pad or str(rng.choice(["same", "valid"]))
        wt = [("kernel", he(rng, (kh, kw, shape[2], cout), kh * kw * shape[2]))]
        bias = bool(rng.integers(0, 2))
        if bias:
            wt.append(("bias", (rng.standard_normal(cout) * 0.1).astype(F32)))
        name = b.layer("Conv2D", [src], {"filters": cout, "kernel_size": [kh, kw],
                                         "padding": pad, "activation": act, "use_bias": bias}, wt)
        hh = shape[0] if pad == "same" else shape[0] - kh + 1
        ww = shape[1] if pad == "same" else shape[1] - kw + 1
        return name, (hh, ww, cout)

    shape = (h, w, c)
    for _ in range(max_layers):
        if shape[0] < 2 or shape[1] < 2:
            break
        roll = int(rng.integers(0, 12))
        if roll < 4:
            cur, shape = conv(cur, shape, int(rng.integers(1, 9)), str(rng.choice(acts)))
        elif roll < 5:
            cur = b.layer("BatchNorm", [cur], None, bn_params(rng, shape[2]))
        elif roll < 6:
            cur = b.layer("Activation", [cur], {"activation": str(rng.choice(acts[1:]))})
        elif roll < 7:
            cur = b.layer("MaxPool2D" if rng.integers(0, 2) else "AvgPool2D", [cur],
                          {"pool_size": 2, "strides": 2,
                           "padding": str(rng.choice(["same", "valid"]))})
            shape = (-(-shape[0] // 2), -(-shape[1] // 2), shape[2]) \
                if b.layers[-1]["config"]["padding"] == "same" else \
                (shape[0] // 2, shape[1] // 2, shape[2])
            if not shape[0] or not shape[1]:
                return random_network(rng, max_layers, extended)
        elif roll < 8 and shape[0] >= 3 and shape[1] >= 3:
            cout = int(rng.integers(1, 7))
            a, sa = conv(cur, shape, cout, "linear", pad="same")
            bb, _ = conv(cur, shape, cout, str(rng.choice(acts)), pad="same")
            cur, shape = b.layer("Add", [a, bb]), sa
        elif roll < 9:
            a, sa = conv(cur, shape, int(rng.integers(1, 5)), "linear", pad="same")
            bb, sb = conv(cur, shape, int(rng.integers(1, 5)), "relu", pad="same")
            cur = b.layer("Concatenate", [a, bb])
            shape = (sa[0], sa[1], sa[2] + sb[2])
        elif roll < 10:
            cur = b.layer("DepthwiseConv2D", [cur],
                          {"kernel_size": 3, "padding": "same", "activation": "linear",
                           "use_bias": False},
                          [("kernel", he(rng, (3, 3, shape[2]), 9))])
        elif roll < 11 and extended:
            t, bt, l, r = (int(v) for v in rng.integers(0, 2, 4))
            cur = b.layer("ZeroPadding2D", [cur], {"padding": [[t, bt], [l, r]]})
            shape = (shape[0] + t + bt, shape[1] + l + r, shape[2])
        else:
            cur = b.layer("UpSample2D", [cur], {"factor": 2}) if shape[0] < 8 else cur
            if shape[0] < 8:
                shape = (shape[0] * 2, shape[1] * 2, shape[2])
    if extended and rng.integers(0, 3) == 0:
        cur = b.layer("GlobalAveragePooling2D", [cur])
        flat = shape[2]
    else:
        cur = b.layer("Flatten", [cur])
        flat = shape[0] * shape[1] * shape[2]
    units = int(rng.integers(2, 17))
    cur = b.layer("Dense", [cur], {"units": units, "activation": str(rng.choice(acts[:3]))},
                  [("kernel", he(rng, (flat, units), flat)),
                   ("bias", (rng.standard_normal(units) * 0.1).astype(F32))])
    if rng.integers(0, 2):
        cur = b.layer("Softmax", [cur])
    m, wts = b.build([cur])
    return m, wts, (h, w, c)
