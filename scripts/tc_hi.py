"""Does the tensor core truncate FP32 operands to TF32?  Compare accuracy with
A_hi written explicitly vs the raw A left in place."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
from builders import dense_net
from oracle import oracle
from paper_1906_05737_b200 import EXACT, compile_model
from paper_1906_05737_b200 import kernels as K
orig = K.Specializer.run
for inplace in (1, 0):
    def run(self, v=inplace):
        spec = orig(self)
        spec.sources = [f"#define NNB_HI_INPLACE {v}\n" + s for s in spec.sources]
        return spec
    K.Specializer.run = run
    for k, units in ((1024, 512), (256, 96)):
        rng = np.random.default_rng(k + units)
        m, w = dense_net(rng, k, units, "linear")
        x = rng.uniform(-2, 2, (4096, k)).astype(np.float32)
        want = oracle.run(m, w, [x])[0]
        net = compile_model(m, w, EXACT, batch=4096, tuning={"aldg": False}, cache_dir="")
        got = net.run([x])[0].cpu().numpy()
        d = np.abs(got.astype(np.float64) - want)
        i = [j for j in net.launches_for() if "_tc_" in net.artifact.launches[j].kernel][0]
        print(f"inplace={inplace} K={k} N={units} max|d|={d.max():.3e} mean={d.mean():.3e} "
              f"t={net.time_launch(i, iters=5):.4f} ms")
