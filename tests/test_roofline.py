"""Per-launch roofline (roofline.py) on the specialiser's real launch lists,
and the reference CPU baseline (oracle/refbench.py) -- no GPU needed."""
import types

import numpy as np
import pytest

from golden_util import load
from paper_1906_05737_b200 import ApproximationOptions, build_graph, build_plan, plan_buffers, zoo
from paper_1906_05737_b200 import roofline
from paper_1906_05737_b200.kernels import specialize

PEAKS = {"hbm_gbs": 6456.8, "bf16_tflops": 1690.1}
FFMA = 71.8


def fake_net(cfg, batch):
    g = build_graph(*zoo.build(cfg))
    plan = build_plan(g)
    spec = specialize(plan, plan_buffers(plan, reserve_heads=True), ApproximationOptions(),
                      batch, (batch + 15) // 16 * 16)
    net = types.SimpleNamespace(plan=plan, artifact=types.SimpleNamespace(launches=spec.launches))
    net.launches_for = lambda n: [i for i, l in enumerate(spec.launches)
                                  if l.n_min <= n <= l.n_max]
    return net


def test_cfg1_dense_on_tensor_pipe_with_split_multiplier():
    net = fake_net(1, 65536)
    rows, total = roofline.net_roofline(net, 65536, PEAKS, FFMA)
    d0 = rows[0]
    assert d0["pipe"] == "tensor" and d0["flops"] == 2 * 65536 * 1024 * 512
    L0 = net.artifact.launches[net.launches_for(65536)[0]]
    assert d0["products_per_mac"] == (2 if "bf16 corr" in L0.note else 3) == 2
    assert d0["peak_tflops"] == pytest.approx(1690.1 / 2)
    # compute-bound: 2 x 68.7 GFLOP at 845 TF/s = 163 us > 405 MB at 6.46 TB/s = 63 us
    assert d0["bound"] == "compute" and d0["roof_us"] == pytest.approx(
        d0["products_per_mac"] * d0["flops"] / 845.05e12 * 1e6)
    assert total == pytest.approx(sum(r["roof_us"] for r in rows))
    assert all(r["pipe"] == "ffma" for r in rows if "_tc_" not in r["kernel"])


@pytest.mark.parametrize("cfg", range(5))
def test_every_launch_has_work_and_a_pipe(cfg):
    B = {0: 4096, 1: 65536, 2: 1024, 3: 256, 4: 64}[cfg]
    net = fake_net(cfg, B)
    rows, total = roofline.net_roofline(net, B, PEAKS, FFMA, {i: 1.0 for i in range(200)})
    assert rows and total > 0
    for r in rows:
        assert r["bytes"] > 0 and r["roof_us"] > 0 and r["pipe"] in ("tensor", "ffma")
        assert r["frac"] == pytest.approx(r["roof_us"] / 1e3)


@pytest.mark.parametrize("cfg", range(5))
def test_layer_roofline_keeps_the_traffic_fusion_removes(cfg):
    """roofline.layer_roofline: the per-LAYER bound over the reference-style
    plan (north_star's wording) with the compiled network's pipes.  It is at
    least the per-launch bound wherever launches fuse layers (cfg2-cfg4), and
    every Dense / conv layer a tcgen05 launch covers is on the tensor pipe."""
    from paper_1906_05737_b200.planner import build_reference_plan
    B = {0: 4096, 1: 65536, 2: 1024, 3: 256, 4: 64}[cfg]
    net = fake_net(cfg, B)
    rp = build_reference_plan(build_graph(*zoo.build(cfg)))
    us, rows = roofline.layer_roofline(net, rp, B, PEAKS, FFMA)
    _, launch_us = roofline.net_roofline(net, B, PEAKS, FFMA)
    assert len(rows) == len(rp.units) and us == pytest.approx(sum(r["roof_us"] for r in rows))
    assert us >= 0.99 * launch_us, (us, launch_us)
    if cfg in (2, 3, 4):
        assert us > 1.05 * launch_us
    n_tc = sum("_tc_" in net.artifact.launches[i].kernel for i in net.launches_for(B))
    assert sum(r["pipe"] == "tensor" for r in rows) >= n_tc - (1 if cfg == 1 else 0)   # cfg1: fused head
    assert all(r["pipe"] == "ffma" for r in rows if r["kind"] not in ("Dense", "Conv2D"))


def test_ffma_peak_source_order(tmp_path):
    assert roofline.ffma_peak_tflops(70.0) == (70.0, "nnb_ffma_peak measured in this run")
    tf, src = roofline.ffma_peak_tflops(None)
    assert tf > 60 and ("profiles/" in src or "derived" in src)


def test_reference_cpu_path_is_the_real_reference():
    """oracle/_ref runs the unmodified nnjit compiled x86 path: its output on
    BASELINE cfg0 equals the reference's own recorded compiled_default
    output (tests/golden/net_cfg0_ref.npz, make_golden.py) bit for bit."""
    from oracle import refbench
    try:
        refbench.nnjit()
    except ImportError:
        pytest.skip("oracle/_ref is absent")
    net, _ = refbench.compile_reference(0)
    _, _, x, rec = load("cfg0_ref")
    got = np.stack([np.array(net.run([xi])[0]) for xi in x])
    np.testing.assert_array_equal(got, rec["compiled_default"])
    us, calls = refbench.batch1_latency_us(0, seconds=0.2, net=net)
    assert us > 0 and calls >= 5


@pytest.mark.parametrize("cfg,batch", [(1, 65536), (3, 256), (0, 4096)])
def test_bench_dominant_roofline_any_pipe(cfg, batch):
    """bench.dominant_roofline on the real launch lists: tensor-, FFMA- and
    HBM-bound dominant launches all yield a fraction of their own peak."""
    import pathlib
    import sys
    sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
    import bench
    net = fake_net(cfg, batch)
    idx = net.launches_for(batch)
    lt = {i: 0.01 * (k + 1) for k, i in enumerate(idx)}          # the last launch dominates
    roof = bench.dominant_roofline(net, batch, lt, PEAKS, (FFMA, "test"))
    assert roof["bound"] in ("tensor", "fp32_ffma", "hbm") and 0 < roof["frac"]
    assert roof["kernel"] == net.artifact.launches[idx[-1]].kernel
    rows, roof_us, meas = bench.launch_table(net, batch, lt, PEAKS, (FFMA, "test"))
    assert len(rows) == len(idx) and roof_us > 0 and meas > 0
