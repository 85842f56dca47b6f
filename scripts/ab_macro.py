"""A/B a kernel compile-time macro: per-launch times of one zoo config with
each '-D' set prepended to every generated kernel source.
usage: ab_macro.py CONFIG BATCH 'A=1 B=2' 'A=0' ..."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_1906_05737_b200 import EXACT, compile_model, zoo, kernels as K  # noqa: E402

cfg, batch = int(sys.argv[1]), int(sys.argv[2])
orig = K.Specializer.run
m, w = zoo.build(cfg)
x = torch.from_numpy(zoo.inputs(cfg, batch))
for variant in sys.argv[3:]:
    defs = "".join(f"#define {d.split('=')[0]} {d.split('=')[1]}\n" for d in variant.split())

    def run(self, defs=defs):
        s = orig(self)
        s.sources = [defs + src for src in s.sources]
        return s
    K.Specializer.run = run
    net = compile_model(m, w, EXACT, batch=batch, cache_dir="")
    net.input_views[0].copy_(x)
    net.apply(); torch.cuda.synchronize()
    print(f"[{variant}] replay {net.time_apply(iters=20):.4f} ms")
    for i in net.launches_for():
        print(f"   {net.artifact.launches[i].kernel:32s} {net.time_launch(i, iters=10):8.4f} ms")
