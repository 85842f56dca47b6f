"""Tail of the tcgen05 error for the N=256 (wide) Dense tiles over seeds and
input distributions: max |d| / (atol + rtol |ref|) per trial."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
from builders import dense_net, he
from oracle import oracle
from paper_1906_05737_b200 import EXACT, compile_model, zoo
variants = sys.argv[1:] or ["wide_chunk=32", "wide_chunk=16"]
ROWS = 18944 + 128          # N = 256 tiles from 74 x 256 rows at 512 columns (kernels.WIDE_MIN_TILES)
trials = []
for seed in range(3):
    for dist in ("normal", "uniform2", "scaled"):
        trials.append((seed, dist))
for v in variants:
    kw = {a.split("=")[0]: eval(a.split("=")[1]) for a in v.split()}
    worst = 0.0
    for seed, dist in trials:
        rng = np.random.default_rng(seed)
        m, w = dense_net(rng, 1024, 512, "linear")
        if dist == "normal":
            x = rng.standard_normal((ROWS, 1024)).astype(np.float32)
        elif dist == "uniform2":
            x = rng.uniform(-2, 2, (ROWS, 1024)).astype(np.float32)
        else:
            x = (rng.standard_normal((ROWS, 1024)) * rng.uniform(0.1, 10, (ROWS, 1))).astype(np.float32)
        want = oracle.run(m, w, [x])[0]
        net = compile_model(m, w, EXACT, batch=ROWS, tuning=kw)
        got = net.run([x])[0].cpu().numpy()
        d = np.abs(got.astype(np.float64) - want)
        r = np.max(d / (1e-5 + 1e-4 * np.abs(want)))
        # the stated bound of the tensor-core paths:
        # FP32 gate + 2^-19 (tf32 split) / 2^-16 (bf16 correction) sum |a b|
        wk = he(np.random.default_rng(seed), (1024, 512), 1024).astype(np.float64)
        mag = np.abs(x.astype(np.float64)) @ np.abs(wk)
        sb = max(np.max(d / (1e-5 + 1e-4 * np.abs(want) + 2.0 ** e * mag)) for e in (-19,))
        sb16 = np.max(d / (1e-5 + 1e-4 * np.abs(want) + 2.0 ** -16 * mag))
        worst = max(worst, r)
        print(f"[{v}] seed {seed} {dist:8s}: max d/lim {r:.3f}  vs 2^-19 bound {sb:.3f}  vs 2^-16 bound {sb16:.3f}")
    m, w = zoo.build(1)
    x = zoo.inputs(1, ROWS)
    want = oracle.run(m, w, [x])[0]
    got = compile_model(m, w, EXACT, batch=ROWS, tuning=kw).run([x])[0].cpu().numpy()
    r = np.max(np.abs(got.astype(np.float64) - want) / (1e-5 + 1e-4 * np.abs(want)))
    print(f"[{v}] cfg1 end to end: max d/lim {r:.3f}; worst dense trial {worst:.3f}")
