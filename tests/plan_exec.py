"""CPU executor of a FusionPlan, built on the oracle's per-layer primitives.

Test infrastructure in the spirit of the reference's ``run_plan``
(pkg/tests/test_optimizer.py:26-72): it evaluates the *fused* units with the
epilogue semantics the sm_100a kernels implement (activation, post-affine,
residual Add, 2x2 max-pool, row softmax), so planner rewrites can be checked
against the unfused graph without a GPU.
"""
import numpy as np

from oracle import oracle

F32 = np.float32
ACT_MODE = 2


def _post(y, u):
    y = oracle.activation(y, u.activation, ACT_MODE)
    if u.post_scale is not None:
        y = (y * u.post_scale).astype(F32) + u.post_offset
    return y.astype(F32)


def run_plan(plan, inputs):
    vals = {t: np.asarray(x, F32) for t, x in zip(plan.input_ids, inputs)}
    for u in plan.units:
        if u.kind in ("Chain", "TcChain"):     # a run of fused units, executed in order
            for st in u.steps:
                _run_unit(st, vals)
        else:
            _run_unit(u, vals)
    return [vals[t] for t in plan.output_ids]


def _run_unit(u, vals):
    if True:
        x = vals[u.input_ids[0]]
        n = x.shape[0]
        if u.kind == "Dense":
            g = getattr(u, "gap", None)
            if g is not None:               # global average pool computed by the same launch
                x = oracle.pool(x.reshape((n,) + g.input_shapes[0].dims), g.kernel_hw[0], g.kernel_hw[1],
                                g.stride, g.padding, True)
            y = _post(oracle.dense(x.reshape(n, -1), u.kernel, u.bias, 1), u)
        elif u.kind in ("Conv2D", "DepthwiseConv2D"):
            dw = u.kind == "DepthwiseConv2D"
            if getattr(u, "dw", None) is not None:
                d = u.dw
                x = oracle.conv(x.reshape((n,) + d.input_shapes[0].dims), d.kernel, d.bias,
                                d.stride, d.padding, True, 1)
                x = _post(x, d)
            if getattr(u, "concat_in", False):
                x = np.concatenate([vals[t].reshape((n,) + sh.dims)
                                    for t, sh in zip(u.input_ids, u.input_shapes)], axis=-1)
            in_hw = (tuple(u.dw.output_shape.dims[:2]) if getattr(u, "dw", None) is not None
                     else tuple(u.input_shapes[0].dims[:2]))
            y = oracle.conv(x.reshape((n,) + in_hw + (-1,)), u.kernel, u.bias, u.stride,
                            u.padding, dw, 1)
            y = _post(y, u)
        elif u.kind == "Pool":
            ph, pw = u.kernel_hw
            y = oracle.pool(x.reshape((n,) + u.input_shapes[0].dims), ph, pw, u.stride,
                            u.padding, u.pool_op == "avg")
        elif u.kind in ("ElementwiseActivation", "Add"):
            y = x.copy()
            for t in u.input_ids[1:]:
                y = (y + vals[t]).astype(F32)
            if u.scale is not None:
                y = ((y.reshape(n, -1, len(u.scale)) * u.scale).astype(F32) + u.offset)
                y = y.astype(F32).reshape(x.shape)
            y = oracle.activation(y, u.activation, ACT_MODE)
        elif u.kind == "Softmax":
            y = oracle.softmax(x.reshape((n,) + u.output_shape.dims))
        elif u.kind == "Upsample":
            f = u.factor
            y = np.repeat(np.repeat(x.reshape((n,) + u.input_shapes[0].dims), f, 1), f, 2)
        elif u.kind == "Concat":
            parts = [vals[t].reshape((n,) + s.dims) for t, s in zip(u.input_ids, u.input_shapes)]
            y = np.concatenate(parts, axis=-1)
        elif u.kind == "Pad":
            (t, b), (l, r) = u.pad
            y = np.pad(x.reshape((n,) + u.input_shapes[0].dims), ((0, 0), (t, b), (l, r), (0, 0)))
        else:
            raise AssertionError(u.kind)
        if getattr(u, "residual_id", None) is not None:
            y = (y.reshape(vals[u.residual_id].shape) + vals[u.residual_id]).astype(F32)
        if getattr(u, "pool_after", False):
            y = oracle.pool(y, 2, 2, 2, "valid", False)
        if getattr(u, "softmax_after", False):
            y = oracle.softmax(y)
        f = getattr(u, "upsample_after", 1)
        if f > 1:
            y = np.repeat(np.repeat(y.reshape((n,) + u.pre_up_shape.dims), f, 1), f, 2)
        vals[u.output_id] = y.reshape((n,) + u.output_shape.dims)
        dp = getattr(u, "dual_pool", None)
        if dp is not None:                # the conv's second, pooled store
            _run_unit(dp, vals)
        da = getattr(u, "dw_after", None)
        if da is not None:                # the depthwise conv computed in the epilogue
            _run_unit(da, vals)
