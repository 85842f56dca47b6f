"""A/B the fused depthwise + pointwise kernel (nnb_sep.cuh) at wider
pointwise layers: planner.SEP_CI_MAX / SEP_CO_MAX raised per variant.
usage: ab_sep.py CONFIG BATCH CI,CO [CI,CO ...]   (32,32 = the default)"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1906_05737_b200 import EXACT, compile_model, zoo, planner  # noqa: E402

cfg, batch = int(sys.argv[1]), int(sys.argv[2])
m, w = zoo.build(cfg)
x = torch.from_numpy(zoo.inputs(cfg, batch))
ref = None
for v in sys.argv[3:]:
    planner.SEP_CI_MAX, planner.SEP_CO_MAX = (int(t) for t in v.split(","))
    net = compile_model(m, w, EXACT, batch=batch, cache_dir="")
    net.input_views[0].copy_(x)
    net.apply(); torch.cuda.synchronize()
    y = net.output_views[0].cpu().numpy().copy()
    if ref is None:
        ref, same = y, ""
    else:
        rel = float(np.max(np.abs(y - ref) / (1e-5 + 1e-4 * np.abs(ref))))
        same = f" max|d|/(atol+rtol|ref|) vs first {rel:.3g}"
    print(f"[{v}] replay {net.time_apply(iters=20):.4f} ms{same}")
    for i in net.launches_for():
        l = net.artifact.launches[i]
        print(f"   {l.kernel:32s} {net.time_launch(i, iters=10):8.4f} ms  {l.note[-90:]}")
