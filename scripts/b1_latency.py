"""Batch-1 (and small-batch) replay latency of every BASELINE config, L2 flushed
before each replay (bench.time_config) and warm (nnb_time_apply).
usage: [NNB_PREFETCH_MAX_N=0] python scripts/b1_latency.py [batch ...]"""
import sys
import pathlib

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1906_05737_b200 import ApproximationOptions, zoo  # noqa: E402

batches = [int(a) for a in sys.argv[1:]] or [1]
for c in range(5):
    for b in batches:
        ms, net = bench.time_config(c, b, 0, torch, ApproximationOptions(), iters=50)
        warm = net.time_apply(b, iters=50)
        print(f"cfg{c} {zoo.CONFIGS[c]['name']:24s} batch {b}: flushed {ms * 1e3:7.1f} us  warm {warm * 1e3:7.1f} us"
              f"  launches {len(net.launches_for(b))}", flush=True)
