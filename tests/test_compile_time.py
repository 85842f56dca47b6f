"""compile() time bound (reference: pkg/tests/test_acceptance.py:486-489, A8:
compile < 250 ms; PAPER.md:109-115 reports 6.5-335 ms for the small nets).

NVRTC needs no GPU, so the cold compile of every BASELINE config is measured
here on the runtime's own parallel job pool (``nnb_compile_parallel``, what
``nnb_create`` runs) over exactly the translation units ``nnb_create``
compiles for ``batch`` (the kernels of a replay over ``batch`` images; other
batch sizes compile on first use).  No cubin cache.  Typical on this 8-core
VM: cfg0 0.5 s, cfg1 1.5 s, cfg3 1.8 s; the gate is
twice that (cfg0 < 1 s, every config < 4 s) because wall times on a shared
VM vary by ~2x, and it exists to catch the 40-s class of regression: before
round 2, cfg0 took 43 s (one direct conv with 1152 weights as function-local
immediates, fully unrolled).  The budget scales with 8 / cpu_count on
smaller machines."""
import os

import pytest

from paper_1906_05737_b200 import EXACT, _native, zoo
from paper_1906_05737_b200.buffers import plan_buffers
from paper_1906_05737_b200.graph import build_graph
from paper_1906_05737_b200.kernels import specialize
from paper_1906_05737_b200.planner import build_plan

BIG = {0: 4096, 1: 65536, 2: 1024, 3: 256, 4: 64}
BUDGET_S = {0: 1.0, 1: 4.0, 2: 4.0, 3: 4.0, 4: 4.0}
SCALE = max(1.0, 8 / (os.cpu_count() or 8))


def create_sources(cfg, batch):
    """The translation units nnb_create compiles for a network of `batch`."""
    m, w = zoo.build(cfg)
    plan = build_plan(build_graph(m, w))
    spec = specialize(plan, plan_buffers(plan, reserve_heads=True), EXACT, batch,
                      (batch + 15) // 16 * 16)
    need = sorted({spec.kernel_source[spec.kernel_names.index(l.kernel)]
                   for l in spec.launches if l.n_min <= batch <= l.n_max})
    return [spec.sources[i] for i in need]


@pytest.mark.parametrize("cfg", sorted(BIG))
@pytest.mark.parametrize("big", [False, True])
def test_cold_compile_within_budget(cfg, big):
    batch = BIG[cfg] if big else 1
    srcs = create_sources(cfg, batch)
    # best of two (the container may be busy); each run is cold (no cache)
    wall = min(_native.compile_parallel(srcs)[0] for _ in range(2)) / 1e3
    print(f"cfg{cfg} batch {batch}: {len(srcs)} kernels, cold NVRTC {wall:.2f} s "
          f"on {os.cpu_count()} threads")
    assert wall < BUDGET_S[cfg] * SCALE, (cfg, batch, wall)


def test_direct_conv_is_not_fully_unrolled_beyond_the_budget():
    """cfg0's second conv (16x16x8 -> 16, 2x2 pool) would unroll 4608 FFMAs
    per thread with one pool window per thread; split over two lanes
    (PSPLIT) it unrolls 2304 and keeps its weights as immediates.  A direct
    conv beyond both bounds keeps its taps loop rolled over shared-memory
    weights."""
    from paper_1906_05737_b200 import kernels
    m, w = zoo.build(0)
    plan = build_plan(build_graph(m, w))
    spec = specialize(plan, plan_buffers(plan, reserve_heads=True), EXACT, 1, 16, tiny=False)
    src = spec.sources[spec.kernel_source[spec.kernel_names.index("nnb_u01_conv3x3_direct_1")]]
    assert "PSPLIT = 2LL" in src and "WIMM = 1LL" in src and "ROLL_KY = 0LL" in src
    stem = spec.sources[spec.kernel_source[0]]
    assert "WIMM = 1LL" in stem and "__device__ const float nnb_Cfg_0_wt" in stem
    assert kernels.DIRECT_UNROLL_MAX >= 3 * 3 * 1 * 8 * 4
    # a larger direct conv (5x5, CI 4 -> CO 32: 3200 FFMAs, no pool to split)
    # keeps its taps loop rolled
    from paper_1906_05737_b200.zoo import NetBuilder
    b = NetBuilder()
    x = b.input((16, 16, 4))
    y = b.conv(x, 4, 32, k=5)
    plan = build_plan(build_graph(*b.build([y])))
    spec = specialize(plan, plan_buffers(plan), EXACT, 1, 16)
    src = spec.sources[spec.kernel_source[0]]
    assert "WIMM = 0LL" in src and "ROLL_KY = 0LL" not in src
