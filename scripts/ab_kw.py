"""A/B CompiledNetwork keyword options: replay + per-launch times of one zoo config.
usage: ab_kw.py CONFIG BATCH 'epi_tma=True' 'epi_tma=False D:NNB_TC_DBG=1' ...
(D:NAME=VAL entries are prepended to every kernel source as #defines;
 M:mode / S:mode select the activation / softmax-exp approximation modes,
 default exact)"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1906_05737_b200 import EXACT, ApproximationOptions, compile_model, zoo, kernels as K  # noqa: E402

cfg, batch = int(sys.argv[1]), int(sys.argv[2])
m, w = zoo.build(cfg)
x = torch.from_numpy(zoo.inputs(cfg, batch))
ref = None
orig = K.Specializer.run
for variant in sys.argv[3:]:
    kw = {k: eval(v) for k, v in (a.split("=") for a in variant.split() if not a[:2] in ("D:", "M:", "S:"))}
    modes = [a[2:] for a in variant.split() if a.startswith("M:")]
    smx = [a[2:] for a in variant.split() if a.startswith("S:")]
    opts = EXACT
    if modes or smx:
        opts = ApproximationOptions(activation_mode=modes[0] if modes else EXACT.activation_mode,
                                    softmax_exp=smx[0] if smx else EXACT.softmax_exp)
    defs = "".join(f"#define {a[2:].split('=')[0]} {a.split('=')[1]}\n"
                   for a in variant.split() if a.startswith("D:"))

    def run(self, defs=defs):
        sp = orig(self)
        sp.sources = [defs + src for src in sp.sources]
        return sp
    K.Specializer.run = run
    net = compile_model(m, w, opts, batch=batch, cache_dir="", tuning=kw)
    net.input_views[0].copy_(x)
    net.apply(); torch.cuda.synchronize()
    y = net.output_views[0].cpu().numpy().copy()
    same = "" if ref is None else f" max|d| vs first {float(np.max(np.abs(y - ref))):.3g}"
    ref = y if ref is None else ref
    print(f"[{variant}] replay {net.time_apply(iters=20):.4f} ms{same}")
    for i in net.launches_for():
        l = net.artifact.launches[i]
        print(f"   {l.kernel:32s} {net.time_launch(i, iters=10):8.4f} ms  {l.note[-70:]}")
