"""GPU parity: the five BASELINE configs through the C ABI vs the C oracle."""
import numpy as np
import pytest

from oracle import oracle
from paper_1906_05737_b200 import EXACT, ApproximationOptions, compile_model, zoo

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-5          # BASELINE.json north_star FP32 tolerance


@pytest.mark.parametrize("cfg,n", [(0, 1), (0, 37), (1, 1), (1, 20), (2, 1), (2, 9),
                                   (3, 1), (3, 5), (4, 1), (4, 2)])
def test_config_exact_vs_oracle(cfg, n):
    m, w = zoo.build(cfg)
    net = compile_model(m, w, EXACT, batch=n)
    x = zoo.inputs(cfg, n)
    got = net.run([x])[0].cpu().numpy()
    want = oracle.run(m, w, [x], "exact")[0]
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("cfg", [0, 1, 3])
def test_config_default_modes_vs_oracle_models(cfg):
    opts = ApproximationOptions()
    m, w = zoo.build(cfg)
    net = compile_model(m, w, opts, batch=6)
    x = zoo.inputs(cfg, 6)
    got = net.run([x])[0].cpu().numpy()
    want = oracle.run(m, w, [x], opts)[0]
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("cfg,n", [(1, 2048), (1, 3001), (2, 40), (3, 33)])
def test_tensor_core_path_vs_oracle(cfg, n):
    """Batches large enough for the tcgen05 3xTF32 GEMM (Dense, 1x1 conv)."""
    m, w = zoo.build(cfg)
    net = compile_model(m, w, EXACT, batch=n)
    assert any("_tc_" in l.kernel for l in net.artifact.launches
               if l.n_min <= n <= l.n_max), "tensor-core kernel not selected"
    x = zoo.inputs(cfg, n)
    got = net.run([x])[0].cpu().numpy()
    want = oracle.run(m, w, [x], "exact")[0]
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("opts", [EXACT, ApproximationOptions()], ids=["exact", "default"])
@pytest.mark.parametrize("cfg,n", [(0, 4096), (1, 65536), (2, 1024), (3, 256), (4, 64)])
def test_baseline_batch_sampled_images_vs_oracle(cfg, n, opts):
    """At the BASELINE batch sizes (the bench workloads), under interpreter-
    grade and the reference's default options: images are independent, so
    16 images of the batch -- the first, the last and 14 seeded others -- are
    checked against the oracle run on just those images (>= 16
    sampled images per config), plus finiteness of the whole output."""
    m, w = zoo.build(cfg)
    net = compile_model(m, w, opts, batch=n)
    x = zoo.inputs(cfg, n)
    got = net.run([x])[0].cpu().numpy()
    assert np.isfinite(got).all()
    rest = np.random.default_rng(cfg).choice(np.arange(1, n - 1), size=14, replace=False)
    idx = np.sort(np.concatenate([[0, n - 1], rest]))
    want = oracle.run(m, w, [x[idx]], "exact" if opts == EXACT else opts)[0]
    np.testing.assert_allclose(got[idx], want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("cfg,n,k", [(1, 5000, 4), (0, 999, 3), (3, 20, 8)])
def test_pipelined_host_call(cfg, n, k):
    """compile_model(host_chunks=k) -> PipelinedNetwork: nnb_run_host_chunked
    splits the host buffers into k chunks (ragged last chunk) over k
    networks and streams; same results as the oracle, and as one network."""
    from paper_1906_05737_b200 import PipelinedNetwork, pinned_empty
    m, w = zoo.build(cfg)
    net = compile_model(m, w, EXACT, batch=n, host_chunks=k)
    assert isinstance(net, PipelinedNetwork) and len(net.nets) == k
    x = zoo.inputs(cfg, n)
    hx = pinned_empty(x.shape)
    hx[...] = x
    got = net.run_host([hx])[0]
    idx = np.sort(np.random.default_rng(cfg).choice(n, size=min(n, 8), replace=False))
    idx[-1] = n - 1                                         # the ragged last chunk
    want = oracle.run(m, w, [x[idx]], "exact")[0]
    np.testing.assert_allclose(got[idx], want, rtol=RTOL, atol=ATOL)
    one = compile_model(m, w, EXACT, batch=n).run_host([hx])[0]
    np.testing.assert_allclose(got, one, rtol=RTOL, atol=ATOL)
    part = net.run_host([hx], n=n // 2 + 1)[0]               # fewer images than the batch
    np.testing.assert_allclose(part, one[:n // 2 + 1], rtol=RTOL, atol=ATOL)
