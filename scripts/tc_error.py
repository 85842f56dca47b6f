"""Error statistics of the tcgen05 3xTF32 Dense path vs the oracle."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
from builders import dense_net
from oracle import oracle
from paper_1906_05737_b200 import EXACT, compile_model
for k, units, act in ((1024, 512, "tanh"), (1024, 512, "linear"), (256, 96, "relu6"), (4096, 256, "linear")):
    rng = np.random.default_rng(k + units)
    m, w = dense_net(rng, k, units, act)
    x = rng.uniform(-2, 2, (2049, k)).astype(np.float32)
    want = oracle.run(m, w, [x])[0]
    for tc in (True, False):
        net = compile_model(m, w, EXACT, batch=2049, use_tc=tc)
        got = net.run([x])[0].cpu().numpy()
        d = np.abs(got.astype(np.float64) - want)
        viol = d > 1e-5 + 1e-4 * np.abs(want)
        print(f"K={k} N={units} {act:6s} tc={tc}: max|d|={d.max():.3e} p99.99={np.quantile(d, 0.9999):.3e} mean={d.mean():.3e} viol={viol.sum()}")
