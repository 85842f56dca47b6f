"""Fusion planner: reference fusions (bit-identical folded weights) and the
B200 epilogue fusions (numerically sound, checked with a CPU plan executor)."""
import numpy as np
import pytest

from builders import bn_params, conv_net, he, random_network
from golden_util import load, names, sha
from oracle import oracle
from plan_exec import run_plan
from paper_1906_05737_b200 import build_graph, build_plan, build_reference_plan, zoo
from paper_1906_05737_b200.planner import lower_to_units
from paper_1906_05737_b200.zoo import NetBuilder

F32 = np.float32
TOL = dict(rtol=1e-4, atol=1e-5)


def kinds(plan):
    return [u.kind for u in plan.units]


def test_lowering_kinds_and_flatten_alias():
    m, w = zoo.build(0)
    g = build_graph(m, w)
    p = lower_to_units(g)
    assert kinds(p).count("Conv2D") == 3 and kinds(p).count("Pool") == 3
    assert "Flatten" not in kinds(p)
    dense = [u for u in p.units if u.kind == "Dense"][0]
    pool = [u for u in p.units if u.kind == "Pool"][-1]
    assert dense.input_ids == (pool.output_id,)      # Flatten relabelled


@pytest.mark.parametrize("name", names())
def test_reference_plan_bit_identical_to_reference_optimizer(name):
    """Unit kinds, activations and every folded array match the reference
    planner's (hashes recorded by tests/golden/make_golden.py)."""
    m, w, x, rec = load(name)
    plan = build_reference_plan(build_graph(m, w))
    want = sorted({int(k.split(":")[1]) for k in rec if k.startswith("plan:")})
    assert len(plan.units) == len(want)
    for i, u in enumerate(plan.units):
        assert bytes(rec[f"plan:{i}:{u.kind}:act"]).decode() == u.activation
        for fld in ("kernel", "bias", "post_scale", "post_offset", "scale", "offset"):
            v = getattr(u, fld)
            key = f"plan:{i}:{u.kind}:{fld}"
            assert (v is None) == (key not in rec), key
            if v is not None:
                assert sha(v) == bytes(rec[key]), key


def _net(build):
    b = NetBuilder(seed=0)
    out = build(b, np.random.default_rng(0))
    return build_graph(*b.build([out]))


def test_conv_bn_act_single_unit_and_bn_before_dense():
    def f(b, rng):
        x = b.input((6, 6, 2))
        c = b.layer("Conv2D", [x], {"filters": 3, "kernel_size": 3, "padding": "same"},
                    [("kernel", he(rng, (3, 3, 2, 3), 18)), ("bias", np.zeros(3, F32))])
        bn = b.layer("BatchNorm", [c], None, bn_params(rng, 3))
        a = b.layer("Activation", [bn], {"activation": "relu6"})
        fl = b.layer("Flatten", [a])
        bn2 = b.layer("BatchNorm", [fl], None, bn_params(rng, 108))
        return b.layer("Dense", [bn2], {"units": 4},
                       [("kernel", he(rng, (108, 4), 108)), ("bias", np.zeros(4, F32))])
    p = build_reference_plan(_net(f))
    assert kinds(p) == ["Conv2D", "Dense"]
    assert p.units[0].activation == "relu6" and p.units[0].post_scale is None


def test_case_c_post_affine_and_double_bn_composes():
    def f(b, rng):
        x = b.input((5, 5, 2))
        c = b.layer("Conv2D", [x], {"filters": 2, "kernel_size": 1, "activation": "elu"},
                    [("kernel", he(rng, (1, 1, 2, 2), 2)), ("bias", np.zeros(2, F32))])
        b1 = b.layer("BatchNorm", [c], None, bn_params(rng, 2))
        return b.layer("BatchNorm", [b1], None, bn_params(rng, 2))
    g = _net(f)
    p = build_reference_plan(g)
    assert kinds(p) == ["Conv2D"] and p.units[0].post_scale is not None
    x = np.random.default_rng(1).normal(size=(3, 5, 5, 2)).astype(F32)
    np.testing.assert_allclose(run_plan(p, [x])[0], oracle.run_graph(g, [x])[0], **TOL)


@pytest.mark.parametrize("pad,folds", [("same", False), ("valid", True)])
def test_bn_before_conv_folds_only_when_valid(pad, folds):
    def f(b, rng):
        x = b.input((6, 6, 3))
        bn = b.layer("BatchNorm", [x], None, bn_params(rng, 3))
        return b.layer("Conv2D", [bn], {"filters": 2, "kernel_size": 3, "padding": pad},
                       [("kernel", he(rng, (3, 3, 3, 2), 27)), ("bias", np.zeros(2, F32))])
    # case (b): BN folds forward into the conv only under 'valid' padding
    # (the folded bias would otherwise also apply to the zero padding)
    g = _net(f)
    p = build_reference_plan(g)
    assert sum(1 for u in p.units if u.scale is not None) == (0 if folds else 1)
    x = np.random.default_rng(5).normal(size=(2, 6, 6, 3)).astype(F32)
    np.testing.assert_allclose(run_plan(p, [x])[0], oracle.run_graph(g, [x])[0], **TOL)


def test_fanout_and_output_block_fusion():
    def f(b, rng):
        x = b.input((4, 4, 2))
        c = b.layer("Conv2D", [x], {"filters": 2, "kernel_size": 1},
                    [("kernel", he(rng, (1, 1, 2, 2), 2)), ("bias", np.zeros(2, F32))])
        a = b.layer("Activation", [c], {"activation": "relu"})
        t = b.layer("Activation", [c], {"activation": "tanh"})
        return b.layer("Add", [a, t])
    p = build_plan(_net(f))
    assert kinds(p).count("ElementwiseActivation") == 2     # c has two consumers
    m, w = conv_net(np.random.default_rng(0), 4, 4, 2, 2, act="linear")
    p = build_plan(build_graph(m, w))
    assert kinds(p) == ["Conv2D"]


def test_gpu_fusions_on_zoo():
    p0 = build_plan(build_graph(*zoo.build(0)))
    assert [u.pool_after for u in p0.units if u.kind == "Conv2D"] == [True, True, True]
    assert p0.units[-1].softmax_after and kinds(p0) == ["Conv2D"] * 3 + ["Dense"] * 2
    p2 = build_plan(build_graph(*zoo.build(2)))
    assert sum(u.residual_id is not None for u in p2.units) == 1 and "Add" not in kinds(p2)
    p4 = build_plan(build_graph(*zoo.build(4)))
    convs = [u for u in p4.units if u.kind == "Conv2D"]
    # encoder convs 2 and 3 feed a skip connection: they store their full output
    # and, as a second store, the pooled map (fuse_pool_dual; conv 3's pooled map
    # upsampled for the decoder)
    assert [c.pool_after for c in convs[:3]] == [True, False, False]
    assert [c.dual_pool is not None for c in convs[:3]] == [False, True, True]
    assert convs[2].dual_pool.upsample_after == 2 and "Pool" not in kinds(p4)
    assert convs[-1].softmax_after
    # decoder: conv->upsample epilogue, concat as operand loader
    assert "Upsample" not in kinds(p4) and "Concat" not in kinds(p4)
    assert sum(u.upsample_after == 2 for u in p4.units) == 1
    assert sum(u.concat_in for u in p4.units) == 2
    assert kinds(build_plan(build_graph(*zoo.build(4)), gpu_fusion=False)).count("Pool") == 3


@pytest.mark.parametrize("cfg", range(5))
@pytest.mark.parametrize("dw_fusion", [False, True])
def test_gpu_plan_numerically_sound_on_zoo(cfg, dw_fusion):
    m, w = zoo.build(cfg)
    g = build_graph(m, w)
    x = zoo.inputs(cfg, 2)
    plan = build_plan(g, dw_fusion=dw_fusion)
    if dw_fusion and cfg in (2, 3):
        assert "DepthwiseConv2D" not in kinds(plan)
    np.testing.assert_allclose(run_plan(plan, [x])[0], oracle.run_graph(g, [x])[0], **TOL)


def test_chain_fusion_sound_and_shaped_on_cfg3():
    """planner.fuse_chain (opt-in): cfg3's 16x16 .. 4x4 tail (20 units ending
    in the GAP) becomes one Chain unit whose shared-memory footprint fits a
    CTA, and the chained plan computes the unfused graph."""
    from paper_1906_05737_b200.planner import CHAIN_SMEM_MAX, chain_smem
    m, w = zoo.build(3)
    g = build_graph(m, w)
    plan = build_plan(g, chain=True, tc_chain=False)
    chains = [u for u in plan.units if u.kind == "Chain"]
    assert len(chains) == 1 and len(chains[0].steps) == 20
    assert chains[0].steps[-1].kind == "Pool" and chain_smem(chains[0].steps) <= CHAIN_SMEM_MAX
    for st in chains[0].steps[:-1]:
        assert st.output_id not in plan.tensors          # intermediates never materialise
    x = zoo.inputs(3, 2)
    np.testing.assert_allclose(run_plan(plan, [x])[0], oracle.run_graph(g, [x])[0], **TOL)
    assert "Chain" not in kinds(build_plan(g))          # off by default


def test_tc_chain_fusion_sound_and_shaped_on_cfg3():
    """planner.fuse_tc_chain (opt-in): cfg3's 8x8 stage -- six pointwise
    layers (the first reading 8x8x64 from the arena), five 8x8 depthwise
    layers and the closing stride-2 depthwise to 4x4 -- is one TcChain unit,
    and the plan computes the unfused graph."""
    m, w = zoo.build(3)
    g = build_graph(m, w)
    plan = build_plan(g, tc_chain=True)
    assert "TcChain" not in kinds(build_plan(g))        # opt-in
    (tc,) = [u for u in plan.units if u.kind == "TcChain"]
    assert [st.kind[0] for st in tc.steps] == list("CDCDCDCDCDCD")
    assert tc.input_shapes[0].dims == (8, 8, 64) and tc.output_shape.dims == (4, 4, 128)
    x = zoo.inputs(3, 2)
    np.testing.assert_allclose(run_plan(plan, [x])[0], oracle.run_graph(g, [x])[0], **TOL)


def test_build_plan_idempotent_and_deterministic():
    m, w = zoo.build(3)
    a, b = build_plan(build_graph(m, w)), build_plan(build_graph(m, w))
    assert [u.describe() for u in a.units] == [u.describe() for u in b.units]
    for u, v in zip(a.units, b.units):
        if u.kernel is not None:
            assert sha(u.kernel) == sha(v.kernel) and sha(u.bias) == sha(v.bias)


def test_random_networks_fusion_soundness():
    """A4-style sweep: fused plan == unfused graph on random DAGs."""
    rng = np.random.default_rng(2024)
    for trial in range(120):
        m, w, shape = random_network(rng)
        g = build_graph(m, w)
        x = rng.uniform(-2, 2, (2,) + shape).astype(F32)
        want = oracle.run_graph(g, [x])[0]
        got = run_plan(build_plan(g), [x])[0]
        np.testing.assert_allclose(got, want, rtol=2e-4, atol=2e-5, err_msg=f"trial {trial}")


@pytest.mark.parametrize("mega", [True, False])
@pytest.mark.parametrize("cfg", range(5))
@pytest.mark.parametrize("batch", [1, 3, 64, 300])
def test_specialised_launches_cover_every_unit_once_per_batch(cfg, batch, mega):
    """For every n in [1, batch] each plan unit is covered by exactly one
    launch (n-range variants must tile the batch axis without overlap)."""
    from paper_1906_05737_b200 import plan_buffers
    from paper_1906_05737_b200.kernels import specialize
    from paper_1906_05737_b200.options import EXACT
    plan = build_plan(build_graph(*zoo.build(cfg)))
    spec = specialize(plan, plan_buffers(plan), EXACT, batch, -(-batch // 16) * 16, mega=mega)
    for n in sorted({1, min(2, batch), batch // 2 or 1, batch}):
        act = [l for l in spec.launches if l.n_min <= n <= l.n_max]
        if any(l.cooperative for l in act):        # the batch-1 persistent kernel runs alone
            assert len(act) == 1 and n <= 8, (n, [l.kernel for l in act])
            continue
        # a 1x1 conv whose consumer depthwise conv is computed in its tcgen05
        # epilogue (planner.fuse_pw_dw) runs that depthwise conv as a second
        # launch of the unit at batch sizes served by other kernels
        second = [l for l in act if plan.units[l.unit].dw_after is not None and "_tc_" not in l.kernel
                  and ("_dw" in l.kernel or "_gap_" in l.kernel)]
        for l in second:
            assert not any("in the epilogue" in o.note for o in act if o.unit == l.unit)
        for u_pos in {l.unit for l in act if plan.units[l.unit].dw_after is not None}:
            mine = [l for l in act if l.unit == u_pos]
            assert (len(mine) == 1 and "in the epilogue" in mine[0].note) or \
                (len(mine) == 2 and mine[1] in second), (n, [l.kernel for l in mine])
        units = [l.unit for l in act if l not in second]
        assert sorted(units) == sorted(set(units)), (n, units)
        # a tcgen05 launch with a fused head (kernels.py HEAD) also covers the next unit
        heads = [l.unit + 1 for l in act if "fused Dense head" in l.note]
        assert not set(heads) & set(units), (n, units, heads)
        assert set(units) | set(heads) == set(range(len(plan.units))), (n, units)


def _reference_nnjit():
    from oracle import refbench
    try:
        return refbench.nnjit()
    except ImportError:
        pytest.skip("oracle/_ref (the installed reference) is absent")


@pytest.mark.parametrize("name", ["cfg0_ref", "cfg1_ref", "cfg2_ref", "cfg3_ref", "mixed_net",
                                  "conv1", "dw2", "pool1", "batchnorm"])
def test_reference_planner_output_drives_the_specialiser(name):
    """a maintainer keeps the REFERENCE's planner
    (nnjit.build_plan, pkg/src/nnjit/optimizer.py:328-341, run here from the
    unmodified package in oracle/_ref) and hands its FusionPlan to this
    package via planner.adopt_plan.  The specialised sm_100a sources, launch
    list and weight pool are byte-identical to those of this package's own
    planner."""
    import json
    from paper_1906_05737_b200 import ApproximationOptions, plan_buffers
    from paper_1906_05737_b200.kernels import specialize
    from paper_1906_05737_b200.planner import adopt_plan
    nnjit = _reference_nnjit()
    m, w, x, rec = load(name)
    doc = json.loads(bytes(rec["manifest"]).decode())
    rm = nnjit.parse_manifest(json.dumps(doc))
    refs = [r for l in rm.layers for r in l.weight_refs]
    blob = bytearray(max((r.offset + r.length for r in refs), default=0))
    for r in refs:
        blob[r.offset:r.offset + r.length] = np.asarray(w[r.name], "<f4").tobytes()
    ref_plan = nnjit.build_plan(nnjit.build_graph(rm, nnjit.load_weights(rm, bytes(blob))))
    adopted = adopt_plan(ref_plan)
    ours = build_plan(build_graph(m, w))
    assert adopted.describe() == ours.describe()
    for batch in (1, 300):
        cap = (batch + 15) // 16 * 16
        a = specialize(adopted, plan_buffers(adopted, reserve_heads=True),
                       ApproximationOptions(), batch, cap)
        b = specialize(ours, plan_buffers(ours, reserve_heads=True), ApproximationOptions(),
                       batch, cap)
        assert a.sources == b.sources and a.pool == b.pool
        assert [(l.kernel, l.n_min, l.n_max) for l in a.launches] == \
            [(l.kernel, l.n_min, l.n_max) for l in b.launches]
