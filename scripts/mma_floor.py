"""tcgen05 kind::tf32 issue floor vs N: a Dense K=1024 layer over 65536 rows
compiled with the MMA-only diagnostic (NNB_TC_DBG=30: no TMA, no A split,
no epilogue work), so the kernel time is the MMA stream alone.  Prints ns
per MMA instruction and MACs per SM-cycle at 1.965 GHz (upper bound)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
import torch
from builders import dense_net
from paper_1906_05737_b200 import EXACT, compile_model, kernels as K

orig = K.Specializer.run


def run(self):
    sp = orig(self)
    sp.sources = ["#define NNB_TC_DBG 30\n" + s for s in sp.sources]
    return sp


K.Specializer.run = run
rows, k = 1 << 19, 256
for n in (16, 32, 48, 64, 96, 128, 256):
    for kw in ({"pair": False, "nacc": 1}, {"pair": False, "tmem_a": False}, {"pair": True}):
        m, w = dense_net(np.random.default_rng(0), k, n, "linear")
        net = compile_model(m, w, EXACT, batch=rows, tuning=dict(tc_min_rows=1, **kw))
        idx = [i for i in net.launches_for() if "_tc_" in net.artifact.launches[i].kernel]
        if not idx:
            continue
        l = net.artifact.launches[idx[0]]
        ms = net.time_launch(idx[0], rows, iters=5)
        bn = int(l.note.split(" tile ")[1].split("x")[1])
        pair = "CTA pair" in l.note
        tiles = (rows // (256 if pair else 128)) * -(-n // bn)
        instr = tiles * (k // 32) * 12
        per_sm_mac = rows * n * k * 3 / 148
        print(f"N={n:3d} BN={bn:3d} {'pair' if pair else 'single'} {'TA' if 'TMEM' in l.note else 'SS'} "
              f"{ms * 1e3:8.1f} us  {ms * 1e6 / instr:6.2f} ns/instr  "
              f"{per_sm_mac / (ms * 1e-3 * 1.965e9):7.0f} MAC/SM-cycle")
