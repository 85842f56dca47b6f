"""Debug the tcgen05 depthwise-fused pointwise path on one small layer."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
from builders import he
from oracle import oracle
from paper_1906_05737_b200 import EXACT, compile_model
from paper_1906_05737_b200.zoo import NetBuilder
F32 = np.float32
h, w, c, co, s = [int(a) for a in sys.argv[1:6]]
kw = dict(a.split("=") for a in sys.argv[6:])
kw = {k: eval(v) for k, v in kw.items()}
rng = np.random.default_rng(0)
b = NetBuilder()
x = b.input((h, w, c))
d = b.layer("DepthwiseConv2D", [x], {"kernel_size": 3, "strides": s, "padding": "same", "use_bias": False},
            [("kernel", he(rng, (3, 3, c), 9))])
y = b.layer("Conv2D", [d], {"filters": co, "kernel_size": 1}, [("kernel", he(rng, (1, 1, c, co), c)),
                                                             ("bias", np.zeros(co, F32))])
m, wt = b.build([y])
n = 2
xin = rng.uniform(-2, 2, (n, h, w, c)).astype(F32)
net = compile_model(m, wt, EXACT, batch=n, tuning=dict(dw_fusion=True, tc_min_rows=1, tc_tile_use=0, **kw))
print([l.note for l in net.artifact.launches])
got = net.run([xin])[0].cpu().numpy()
want = oracle.run_graph(net.graph, [xin])[0]
bad = np.abs(got - want) > 1e-5 + 1e-4 * np.abs(want)
print("bad", bad.sum(), "of", bad.size)
if bad.any():
    idx = np.argwhere(bad)
    print("bad pixels (img, y, x):", sorted({tuple(i[:3]) for i in idx})[:40])
    print("bad channels:", sorted({int(i[3]) for i in idx}))
    i = tuple(idx[0]); print("example", i, got[i], want[i])
