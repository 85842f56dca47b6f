"""Error statistics of the tcgen05 implicit-GEMM conv tiles (TF32 split in
shared memory) vs the oracle, per split mode / tuning variant.
usage: tc_error_conv.py 'rn_ss=True' 'rn_ss=2' ..."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
from builders import conv_net
from oracle import oracle
from paper_1906_05737_b200 import EXACT, compile_model
variants = sys.argv[1:] or ["rn_ss=True"]
for (h, w, ci, co, act) in ((60, 80, 128, 32, "relu"), (120, 160, 64, 16, "linear"), (60, 80, 96, 64, "linear"),
                            (30, 40, 256, 32, "linear"), (120, 160, 16, 32, "relu")):
    rng = np.random.default_rng(ci * co)
    m, wt = conv_net(rng, h, w, ci, co, k=3, act=act)
    n = 16
    x = rng.uniform(-2, 2, (n, h, w, ci)).astype(np.float32)
    want = oracle.run(m, wt, [x])[0]
    for v in variants:
        kw = {a.split("=")[0]: eval(a.split("=")[1]) for a in v.split()}
        net = compile_model(m, wt, EXACT, batch=n, tuning=kw)
        notes = [net.artifact.launches[i].note for i in net.launches_for()]
        got = net.run([x])[0].cpu().numpy()
        d = np.abs(got.astype(np.float64) - want)
        lim = 1e-5 + 1e-4 * np.abs(want)
        print(f"{h}x{w}x{ci}->{co} {act:6s} [{v}]: max|d|={d.max():.3e} max d/lim={np.max(d / lim):.3f} "
              f"mean={d.mean():.3e} bias={np.mean(got.astype(np.float64) - want):.2e} viol={(d > lim).sum()} "
              f"{'tc' if any('tcgen05' in t for t in notes) else 'NOT tc'}")
