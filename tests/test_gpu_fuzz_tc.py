"""Randomised parity of the tensor-core paths: networks with tcgen05-friendly
shapes (channels multiples of 16, 1x1 / 3x3 convs, residual Adds, depthwise
+ pointwise blocks, pools, upsample + concat, Dense heads), compiled with the
tensor-core thresholds forced down so every eligible unit takes the tcgen05
kernel (CTA pairs, KPACK, TMA-store epilogue, residual prefetch, depthwise
fusion), checked against the oracle at the FP32 tolerance."""
import numpy as np
import pytest

from builders import bn_params, he
from oracle import oracle
from paper_1906_05737_b200 import EXACT, compile_model
from paper_1906_05737_b200.zoo import NetBuilder

pytestmark = pytest.mark.gpu
F32 = np.float32
TOL = dict(rtol=1e-4, atol=1e-5)
CH = (16, 32, 48, 64, 96, 128)


def tc_network(rng):
    b = NetBuilder(seed=int(rng.integers(1 << 30)))
    h, w = int(rng.integers(6, 40)), int(rng.integers(6, 40))
    c = int(rng.choice(CH))
    cur = b.input((h, w, c))
    shape = (h, w, c)

    def conv(src, shape, cout, k, act="relu", stride=1):
        wt = [("kernel", he(rng, (k, k, shape[2], cout), k * k * shape[2])),
              ("bias", (rng.standard_normal(cout) * 0.1).astype(F32))]
        name = b.layer("Conv2D", [src], {"filters": cout, "kernel_size": k, "strides": stride,
                                         "padding": "same", "activation": act}, wt)
        return name, (-(-shape[0] // stride), -(-shape[1] // stride), cout)

    for _ in range(int(rng.integers(2, 6))):
        roll = int(rng.integers(0, 7))
        if roll < 2:
            cur, shape = conv(cur, shape, int(rng.choice(CH)), int(rng.choice([1, 3])),
                              str(rng.choice(["relu", "linear", "relu6", "tanh"])))
        elif roll == 2:                                   # residual block
            a, sa = conv(cur, shape, shape[2], 1, "relu")
            cur = b.layer("Add", [cur, a])
        elif roll == 3:                                   # separable block
            s = int(rng.choice([1, 2]))
            d = b.layer("DepthwiseConv2D", [cur], {"kernel_size": 3, "strides": s,
                                                   "padding": "same", "use_bias": False},
                        [("kernel", he(rng, (3, 3, shape[2]), 9))])
            d = b.layer("BatchNorm", [d], None, bn_params(rng, shape[2]))
            d = b.layer("Activation", [d], {"activation": "relu6"})
            shape = (-(-shape[0] // s), -(-shape[1] // s), shape[2])
            cur, shape = conv(d, shape, int(rng.choice(CH)), 1, "relu")
        elif roll == 4 and shape[0] >= 4 and shape[1] >= 4:
            cur = b.layer("MaxPool2D", [cur], {"pool_size": 2, "strides": 2})
            shape = (shape[0] // 2, shape[1] // 2, shape[2])
        elif roll == 5 and shape[0] >= 4 and shape[1] >= 4:   # decoder step
            lo = b.layer("MaxPool2D", [cur], {"pool_size": 2, "strides": 2})
            lo, sl = conv(lo, (shape[0] // 2, shape[1] // 2, shape[2]), 32, 3)
            up = b.layer("UpSample2D", [lo], {"factor": 2})
            if shape[0] % 2 == 0 and shape[1] % 2 == 0:
                cat = b.layer("Concatenate", [up, cur])
                cur, shape = conv(cat, (shape[0], shape[1], 32 + shape[2]), int(rng.choice(CH)), 3)
        else:
            cur = b.layer("BatchNorm", [cur], None, bn_params(rng, shape[2]))
    cur = b.layer("GlobalAveragePooling2D", [cur]) if rng.integers(0, 2) else b.layer("Flatten", [cur])
    k = shape[2] if "global" in cur else shape[0] * shape[1] * shape[2]
    units = int(rng.choice([32, 64, 128, 256]))
    cur = b.layer("Dense", [cur], {"units": units, "activation": "tanh"},
                  [("kernel", he(rng, (k, units), k)), ("bias", np.zeros(units, F32))])
    m, wt = b.build([cur])
    return m, wt, (h, w, c)


@pytest.mark.parametrize("seed", range(48))
def test_random_tensor_core_networks(seed):
    rng = np.random.default_rng(1000 + seed)
    m, w, shape = tc_network(rng)
    n = int(rng.choice([1, 2, 5, 17]))
    x = rng.uniform(-1, 1, (n,) + shape).astype(F32)
    want = oracle.run(m, w, [x], "exact")[0]
    net = compile_model(m, w, EXACT, batch=n,
                        tuning=dict(tc_min_rows=1, tc_tile_use=0, dw_fusion=bool(seed % 2)))
    got = net.run([x])[0].cpu().numpy()
    np.testing.assert_allclose(got, want, err_msg=net.describe(), **TOL)
