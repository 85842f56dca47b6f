"""Error statistics of the tcgen05 3xTF32 Dense path vs the oracle, for
accumulator layouts (csplit: separate correction chain; chunk: k-blocks of
32 per TMEM chunk).  usage: tc_error.py ['csplit=False chunk=4' ...]"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
from builders import dense_net
from oracle import oracle
from paper_1906_05737_b200 import EXACT, compile_model
variants = sys.argv[1:] or ["csplit=True"]
for k, units, act in ((1024, 512, "tanh"), (1024, 512, "linear"), (256, 96, "relu6"), (4096, 256, "linear")):
    rng = np.random.default_rng(k + units)
    m, w = dense_net(rng, k, units, act)
    x = rng.uniform(-2, 2, (2049, k)).astype(np.float32)
    want = oracle.run(m, w, [x])[0]
    for v in variants:
        kw = {a.split("=")[0]: eval(a.split("=")[1]) for a in v.split()}
        net = compile_model(m, w, EXACT, batch=2049, tuning=kw)
        got = net.run([x])[0].cpu().numpy()
        d = np.abs(got.astype(np.float64) - want)
        lim = 1e-5 + 1e-4 * np.abs(want)
        print(f"K={k} N={units} {act:6s} [{v}]: max|d|={d.max():.3e} max d/lim={np.max(d / lim):.3f} "
              f"mean={d.mean():.3e} viol={(d > lim).sum()}")
