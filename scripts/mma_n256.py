"""Per-instruction cost of tcgen05.mma kind::tf32 at N=128 vs N=256 (MMA-only
diagnostic, NNB_TC_DBG=30; the N=256 variant overrides the instruction width
on BN=128 tiles, so its results are meaningless -- timing only)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
from builders import dense_net
from paper_1906_05737_b200 import EXACT, compile_model, kernels as K

orig = K.Specializer.run
rows, k, n = 1 << 19, 256, 128
for defs in ("#define NNB_TC_DBG 30\n", "#define NNB_TC_DBG 30\n#define NNB_TC_NDBG 256\n",
             "#define NNB_TC_DBG 30\n#define NNB_TC_NDBG 64\n"):
    def run(self, defs=defs):
        sp = orig(self)
        sp.sources = [defs + s for s in sp.sources]
        return sp
    K.Specializer.run = run
    for kw in ({"pair": False, "tmem_a": False}, {"pair": False, "nacc": 1}):
        m, w = dense_net(np.random.default_rng(0), k, n, "linear")
        net = compile_model(m, w, EXACT, batch=rows, tuning=dict(tc_min_rows=1, **kw))
        i = [i for i in net.launches_for() if "_tc_" in net.artifact.launches[i].kernel][0]
        ms = net.time_launch(i, rows, iters=5)
        instr = (rows // 128) * (k // 32) * 12
        print(defs.replace("\n", " "), kw, f"{ms*1e3:.1f} us, {ms*1e6/instr*148:.1f} ns/instr/SM")
