"""Compile one zoo config at a batch and replay it a few times (profiling
target for ncu; prints per-launch CUDA-event times)."""
import argparse
import sys
import pathlib

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1906_05737_b200 import ApproximationOptions, EXACT, compile_model, zoo  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=1)
p.add_argument("--batch", type=int, default=65536)
p.add_argument("--mode", default="exact")
p.add_argument("--reps", type=int, default=3)
p.add_argument("--no-tc", action="store_true")
p.add_argument("--no-tmem-a", action="store_true")
p.add_argument("--nacc", type=int, default=None)
p.add_argument("--aldg", action="store_true")
p.add_argument("--no-kpack", action="store_true")
a = p.parse_args()
opts = EXACT if a.mode == "exact" else ApproximationOptions()
m, w = zoo.build(a.config)
net = compile_model(m, w, opts, batch=a.batch, tuning=dict(use_tc=not a.no_tc, tmem_a=not a.no_tmem_a,
                                                         nacc=a.nacc, aldg=a.aldg,
                                                         kpack=not a.no_kpack))
net.input_views[0].copy_(torch.from_numpy(zoo.inputs(a.config, a.batch)))
for _ in range(a.reps):
    net.apply()
torch.cuda.synchronize()
print("replay ms", net.time_apply(iters=10))
for i in net.launches_for():
    l = net.artifact.launches[i]
    print(f"{l.kernel:32s} {net.time_launch(i, iters=5):8.4f} ms  {l.note}")
