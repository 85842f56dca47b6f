"""Target for compute-sanitizer (one tool per gpurun call): compile BASELINE
configs at their bench batch (default options), replay each network's CUDA
graph twice and check sampled images against the oracle, so memcheck /
racecheck / synccheck see every hand-written kernel (tcgen05 / TMA / mbarrier
included) inside a real graph replay.

    compute-sanitizer --tool memcheck python scripts/sanitize.py 3 4
"""
import sys
import pathlib

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_1906_05737_b200 import ApproximationOptions, compile_model, zoo  # noqa: E402

BIG = {0: 4096, 1: 65536, 2: 1024, 3: 256, 4: 64}
opts = ApproximationOptions()
for cfg in map(int, sys.argv[1:] or ["3", "4"]):
    n = BIG[cfg]
    m, w = zoo.build(cfg)
    net = compile_model(m, w, opts, batch=n)
    x = zoo.inputs(cfg, n)
    net.input_views[0].copy_(torch.from_numpy(x))
    for _ in range(2):
        net.apply()
    torch.cuda.synchronize()
    idx = np.array([0, n // 2, n - 1])
    got = net.output_views[0][torch.as_tensor(idx, device="cuda")].cpu().numpy()
    want = oracle.run(m, w, [x[idx]], opts)[0]
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-5)
    print(f"cfg{cfg} @{n}: {len(net.launches_for(n))} launches replayed twice, sampled outputs ok",
          flush=True)
