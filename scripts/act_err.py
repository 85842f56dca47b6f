"""ulp error of the FP32 exact-mode activations (MODE_EXACT_F32) vs float64."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
from builders import dense_net
from paper_1906_05737_b200 import EXACT, compile_model
from paper_1906_05737_b200.model_format import WeightStore
# identity weights: a K=N=32 Dense whose outputs are the inputs -> activation of x
for act, f in (("tanh", np.tanh), ("sigmoid", lambda v: 1 / (1 + np.exp(-v))), ("elu", lambda v: np.where(v > 0, v, np.expm1(v)))):
    m, w0 = dense_net(np.random.default_rng(0), 32, 32, act)
    w = WeightStore({n: np.eye(32, dtype=np.float32) if w0[n].ndim == 2 else np.zeros_like(w0[n])
                     for n in w0.names()})
    x = np.random.default_rng(1).uniform(-12, 12, (65536, 32)).astype(np.float32)
    x[:8192] *= 0.05
    net = compile_model(m, w, EXACT, batch=65536, tuning={"tc_min_rows": 1})
    assert any("tcgen05" in l.note for l in net.artifact.launches), "not on the TC path"
    got = net.run([x])[0].cpu().numpy().astype(np.float64)
    ref = f(x.astype(np.float64))
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    e = np.abs(got - ref) / ulp
    print(f"{act}: max {e.max():.2f} ulp, mean {e.mean():.3f}, rel max {np.max(np.abs(got-ref)/np.maximum(np.abs(ref),1e-30)):.2e}")
