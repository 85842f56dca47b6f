import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_1906_05737_b200 import EXACT, compile_model, zoo
m, w = zoo.build(2)
net = compile_model(m, w, EXACT, batch=6)
print(net.describe())
x = zoo.inputs(2, 6)
net.run([x]); torch.cuda.synchronize()
net.output_views[0].zero_(); torch.cuda.synchronize()
print("after zero", net.output_views[0].cpu().numpy())
net.run([x[:2]]); torch.cuda.synchronize()
print("after run2", net.output_views[0].cpu().numpy())
for i in net.launches_for(2):
    l = net.artifact.launches[i]
    net.output_views[0].zero_(); torch.cuda.synchronize()
    net.time_launch(i, n=2, iters=1); torch.cuda.synchronize()
    o = net.output_views[0].cpu().numpy()
    print(l.kernel, "rows>=2 nonzero:", bool(np.any(o[2:] != 0)))
