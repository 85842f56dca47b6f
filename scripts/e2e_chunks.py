"""e2e host-buffer throughput of cfg1 @65536 through run_host: one network vs
PipelinedNetwork(host_chunks=k); plus the raw pinned H2D / D2H bandwidth."""
import sys
import pathlib
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1906_05737_b200 import EXACT, compile_model, pinned_empty, zoo  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
B = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
m, w = zoo.build(cfg)
x = zoo.inputs(cfg, B)
hx = pinned_empty(x.shape)
hx[...] = x
d = torch.empty(x.shape, dtype=torch.float32, device="cuda")
for _ in range(3):
    d.copy_(torch.from_numpy(hx), non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    d.copy_(torch.from_numpy(hx), non_blocking=True)
torch.cuda.synchronize()
print(f"raw H2D {hx.nbytes * 10 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
for k in (None, 2, 4, 8, 16):
    net = compile_model(m, w, EXACT, batch=B, host_chunks=k)
    shapes = [tuple(v.shape[1:]) for v in (net.nets[0] if k else net).output_views]
    hy = [pinned_empty((B,) + s) for s in shapes]
    for _ in range(3):
        net.run_host([hx], hy)
    t0 = time.perf_counter()
    for _ in range(10):
        net.run_host([hx], hy)
    dt = (time.perf_counter() - t0) / 10
    print(f"chunks {k}: {dt * 1e3:.3f} ms/step  {B / dt / 1e6:.2f} M img/s")
