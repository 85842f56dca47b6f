"""Diagnostic: time one tcgen05 launch with MMAs skipped / loads skipped."""
import sys, pathlib, re
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_1906_05737_b200 import EXACT, compile_model, zoo
from paper_1906_05737_b200 import kernels as K

cfg, batch, unit = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
m, w = zoo.build(cfg)
orig = K.Specializer.run
for dbg in (0, 1, 2):
    def run(self, dbg=dbg):
        spec = orig(self)
        spec.sources = [f"#define NNB_TC_DBG {dbg}\n" + s for s in spec.sources]
        return spec
    K.Specializer.run = run
    for aldg in (False, True):
        net = compile_model(m, w, EXACT, batch=batch, aldg=aldg, cache_dir="")
        for i in net.launches_for():
            l = net.artifact.launches[i]
            if unit in l.kernel:
                print(f"dbg={dbg} aldg={aldg} {l.kernel} {net.time_launch(i, iters=5):.4f} ms  {l.note}")
K.Specializer.run = orig
