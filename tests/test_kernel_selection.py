"""Kernel selection per batch size (kernels.py TC_MIN_ROWS, SMALL_DENSE_ROWS,
TC_MIN_IMAGES), checked on the specialised launch lists without a GPU: the
thresholds come from scripts/batch_sweep.py on a B200 (profiles/README.md)."""
import numpy as np

from builders import dense_net
from paper_1906_05737_b200 import EXACT, zoo
from paper_1906_05737_b200.buffers import plan_buffers
from paper_1906_05737_b200.graph import build_graph
from paper_1906_05737_b200.kernels import (SMALL_DENSE_ROWS, TC_MIN_IMAGES, WIDE_MIN_TILES,
                                           specialize)
from paper_1906_05737_b200.planner import build_plan


def launches(m, w, max_batch, chain=False, **kw):
    plan = build_plan(build_graph(m, w), chain=chain)
    return specialize(plan, plan_buffers(plan), EXACT, max_batch, max_batch, **kw).launches


def serving(ls, unit, n):
    return [l for l in ls if l.unit == unit and l.n_min <= n <= l.n_max]


def test_dense_row_kernel_then_tensor_cores():
    m, w = dense_net(np.random.default_rng(0), 1024, 512, "tanh")
    ls = launches(m, w, 65536)
    for n, want in ((1, "gemv"), (SMALL_DENSE_ROWS, "gemv"), (SMALL_DENSE_ROWS + 1, "dense_tc"),
                    (1024, "dense_tc"), (65536, "dense_tc")):
        (l,) = serving(ls, 0, n)
        assert want in l.kernel, (n, l.kernel)
    # N = 256 tiles with the BF16 correction split once a launch has enough tiles
    big = serving(ls, 0, 65536)[0]
    assert "256x256" in big.note and "bf16 corr" in big.note
    small = serving(ls, 0, 1024)[0]
    assert "bf16 corr" not in small.note and "A in TMEM" in small.note
    edge = -(-WIDE_MIN_TILES // 2) * 256
    assert "256x256" in serving(ls, 0, edge)[0].note
    assert "256x256" not in serving(ls, 0, edge - 1)[0].note


def test_narrow_dense_hands_over_earlier():
    m, w = dense_net(np.random.default_rng(1), 256, 32, "relu")
    ls = launches(m, w, 4096)
    assert "gemv" in serving(ls, 0, 128)[0].kernel
    assert "dense_tc" in serving(ls, 0, 129)[0].kernel


def test_pointwise_convs_stay_off_tensor_cores_for_a_few_images():
    m, w = zoo.build(3)                       # MobileNetV1 0.25: 1x1 convs of 16..4096 rows/image
    ls = launches(m, w, 256)
    tc_units = {l.unit for l in ls if "_tc_" in l.kernel}
    assert tc_units
    for u in tc_units:
        for n in (1, TC_MIN_IMAGES - 1):
            rows_ok = [l for l in serving(ls, u, n) if "_tc_" in l.kernel]
            # below TC_MIN_IMAGES only launches of >= 2048 rows use tcgen05
            for l in rows_ok:
                assert n * l.items_per_image >= 2048 or "conv" not in l.kernel, (u, n, l.note)
        assert any("_tc_" in l.kernel for l in serving(ls, u, 256)), u


def test_concat_fed_pointwise_conv_never_takes_the_row_gemm():
    """a 1x1 conv whose input is a fused Concatenate must
    not be served by the tcgen05 row GEMM (one A map over input 0 only)."""
    from builders import he
    from paper_1906_05737_b200.zoo import NetBuilder
    rng = np.random.default_rng(3)
    b = NetBuilder()
    x = b.input((16, 16, 4))
    a = b.layer("Conv2D", [x], {"filters": 32, "kernel_size": 3, "padding": "same", "use_bias": False},
                [("kernel", he(rng, (3, 3, 4, 32), 36))])
    c = b.layer("Conv2D", [x], {"filters": 32, "kernel_size": 3, "padding": "same", "use_bias": False},
                [("kernel", he(rng, (3, 3, 4, 32), 36))])
    cat = b.layer("Concatenate", [a, c])
    y = b.layer("Conv2D", [cat], {"filters": 64, "kernel_size": 1, "use_bias": False},
                [("kernel", he(rng, (1, 1, 64, 64), 64))])
    m, w = b.build([y])
    plan = build_plan(build_graph(m, w))
    assert "Concat" not in [u.kind for u in plan.units]
    pos = next(i for i, u in enumerate(plan.units) if u.concat_in)
    ls = specialize(plan, plan_buffers(plan), EXACT, 64, 64).launches
    for n in (1, 8, 64):
        (l,) = serving(ls, pos, n)
        if "_tc_" in l.kernel:         # only the conv-mode tiles: 4-D boxes, two A maps
            assert len(l.tmaps[0]["dims"]) == 4, (n, l.kernel, l.note)
            assert l.tmaps[3]["offset"] != l.tmaps[0]["offset"], l.note
    assert "_tc_" in serving(ls, pos, 64)[0].kernel


def test_small_net_small_batch_is_one_tinynet_launch():
    """kernels.Specializer._tiny (opt-in): cfg0 (16 KB arena, 24 KB of weights) runs
    as ONE launch up to TINY_MAX_N images and as per-layer launches above;
    cfg1 (2.8 MB of weights) and the big-arena configs never take it."""
    from paper_1906_05737_b200.kernels import TINY_MAX_N
    ls = launches(*zoo.build(0), 4096, tiny=True)
    tiny = [l for l in ls if "tinynet" in l.kernel]
    assert len(tiny) == 1 and (tiny[0].n_min, tiny[0].n_max) == (1, TINY_MAX_N)
    for n in (1, TINY_MAX_N):
        assert [l.kernel for l in ls if l.n_min <= n <= l.n_max] == [tiny[0].kernel]
    assert all("tinynet" not in l.kernel for l in ls if l.n_min <= TINY_MAX_N + 1 <= l.n_max)
    assert not any("tinynet" in l.kernel for l in ls if l.n_min <= 4096 <= l.n_max)
    for cfg in (1, 2, 3, 4):
        assert not any("tinynet" in l.kernel for l in launches(*zoo.build(cfg), 64, tiny=True))
    ls = launches(*zoo.build(0), 8)                      # opt-in
    assert not any("tinynet" in l.kernel for l in ls)


def test_tc_tiles_fit_shared_memory_and_share_rows():
    """Every tcgen05 launch of the BASELINE configs fits the 227 KB opt-in
    shared memory at its bench batch (row-shared KPACK stages fall back to
    per-row boxes when two do not fit), and cfg4's narrow KPACK convs use the
    row-shared A boxes (one box of 8 + KH - 1 rows)."""
    from paper_1906_05737_b200.kernels import SMEM_MAX
    shared = 0
    for cfg, batch in ((0, 4096), (1, 65536), (2, 1024), (3, 256), (4, 64)):
        m, w = zoo.build(cfg)
        for l in launches(m, w, batch):
            if "_tc_" not in l.kernel:
                continue
            assert l.smem <= SMEM_MAX, (cfg, l.kernel, l.smem)
            if "rows shared" in l.note:
                shared += 1
                assert l.tmaps[0]["box"][2] == 10, l.tmaps[0]
    assert shared >= 2


def _cfg_fields(src, kernel):
    """The specialised Cfg constants of one kernel's translation unit."""
    import re
    return {k: int(v) for k, v in re.findall(r"static constexpr long long (\w+) = (-?\d+)LL;", src)}


def test_wide_kpack_tiles_drain_one_chunk():
    """The N > 128 KPACK epilogue drains one accumulator chunk (nnb_gemm_tc.cuh
    static_assert): on every tcgen05 conv tile of the randomised tensor-core
    networks (tests/test_gpu_fuzz_tc.py) a wide KPACK tile's K fits one chunk,
    with and without row-shared boxes."""
    from test_gpu_fuzz_tc import tc_network
    from paper_1906_05737_b200.tuning import make_tuning
    seen = 0
    for seed in range(48):
        rng = np.random.default_rng(1000 + seed)
        m, w, _ = tc_network(rng)
        n = int(rng.choice([1, 2, 5, 17]))
        for rowshare in (True, False):
            tn = make_tuning(dict(tc_min_rows=1, tc_tile_use=0, dw_fusion=bool(seed % 2), rowshare=rowshare))
            plan = build_plan(build_graph(m, w), dw_fusion=tn.dw_fusion)
            sp = specialize(plan, plan_buffers(plan), EXACT, n, n, **tn.specializer_kwargs())
            for l in sp.launches:
                if "_tc_" not in l.kernel or not l.n_min <= n <= l.n_max:
                    continue
                f = _cfg_fields(sp.sources[sp.kernel_source[sp.kernel_names.index(l.kernel)]], l.kernel)
                if f.get("KPACK") and f["N"] > 128:
                    seen += 1
                    kb = -(-f["K"] // (f["BK"] * f["RS"]))
                    assert kb <= f["CHUNK"], (seed, l.kernel, f["K"], f["BK"], f["RS"], f["CHUNK"])
    assert seen > 0
