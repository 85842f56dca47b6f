"""Replay time per batch size for every zoo config (one compile at the
largest batch, partial-batch replays): finds batch ranges where the kernel
selection is off (time per image should not rise with the batch)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_1906_05737_b200 import EXACT, compile_model, zoo  # noqa: E402

MAXB = {0: 8192, 1: 65536, 2: 2048, 3: 512, 4: 64}
for cfg in (int(a) for a in (sys.argv[1:] or "01234")):
    m, w = zoo.build(cfg)
    B = MAXB[cfg]
    net = compile_model(m, w, EXACT, batch=B)
    net.input_views[0].copy_(torch.from_numpy(zoo.inputs(cfg, B)))
    n = 1
    while n <= B:
        for k in sorted({n, n + n // 2}):
            if k <= B:
                ms = net.time_apply(k, iters=20)
                print(f"cfg{cfg} n={k:6d}  {ms * 1e3:9.1f} us  {ms * 1e3 / k:8.3f} us/img  "
                      f"launches {len(net.launches_for(k))}", flush=True)
        n *= 2
