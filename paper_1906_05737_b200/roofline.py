"""Algorithmic work per launch unit and the per-layer roofline of SURVEY.md 8(d).

    T_roof(N) = sum_u max(N * F_u / P_pipe(u), (N * (In_u + Out_u) + W_u) / BW)

* ``F_u``: 2 x MACs for Dense / Conv2D / DepthwiseConv2D, one op per element
  per tap for pooling, one per element per input for Add, one per element for
  BatchNorm / activation / softmax; data movement (upsample, concat, pad) is
  free.
* ``In_u`` / ``Out_u``: float32 activation bytes per image; ``W_u``: weight,
  bias and affine bytes, read once per batch.
* ``P_pipe``: FP32 FFMA peak of the B200 = 148 SM x 128 lanes x 2 x f_clk
  (74.4 TFLOP/s at the 1965 MHz max clock; derived, not measured), the TF32
  tensor peak for tensor-core units.
* ``BW``: the measured HBM copy bandwidth (MEASURED_PEAKS.json ``hbm_gbs``).

The canonical units are those of the reference-style plan (BN folded,
activations fused, nothing else fused: ``planner.build_reference_plan``);
``fused_ideal`` is the stricter bound ``max(N*sum F / P, (N*IO + sum W)/BW)``.
"""

import json
import pathlib

SM_COUNT = 148
FFMA_LANES = 128
MAX_SM_MHZ = 1965.0


def fp32_peak_tflops(mhz=MAX_SM_MHZ):
    return SM_COUNT * FFMA_LANES * 2 * mhz * 1e6 / 1e12


def measured_peaks():
    p = pathlib.Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback"}


def unit_work(u, plan=None):
    """(flops per image, activation bytes per image (in+out), weight bytes)."""
    ins = sum(4 * s.elements for s in u.input_shapes)
    if getattr(u, "residual_id", None) is not None:
        ins += 4 * u.output_shape.elements
    out = 4 * u.output_shape.elements
    wb = 0
    for arr in (u.kernel, u.bias, u.post_scale, u.post_offset, u.scale, u.offset):
        if arr is not None:
            wb += 4 * arr.size
    k = u.kind
    if k == "Dense":
        kin, units = u.kernel.shape
        f = 2 * kin * units
    elif k == "Conv2D":
        kh, kw, ci, co = u.kernel.shape
        conv_out = (u.pre_pool_shape if getattr(u, "pool_after", False) else
                    u.pre_up_shape if getattr(u, "upsample_after", 1) > 1 else u.output_shape)
        f = 2 * conv_out.h * conv_out.w * kh * kw * ci * co
    elif k == "DepthwiseConv2D":
        kh, kw, c = u.kernel.shape
        f = 2 * u.output_shape.h * u.output_shape.w * kh * kw * c
    elif k == "Pool":
        ph, pw = u.kernel_hw
        f = u.output_shape.elements * ph * pw
    elif k in ("ElementwiseActivation", "Add", "Softmax"):
        f = u.output_shape.elements * max(1, len(u.input_ids))
    else:
        f = 0
    d = getattr(u, "dw", None)
    if d is not None:              # fused depthwise producer
        df, _, dwb = unit_work(d)
        f += df
        wb += dwb
    return f, ins + out, wb


def layerwise_roof_s(plan, n, hbm_gbs, peak_tflops):
    t = 0.0
    for u in plan.units:
        f, io, w = unit_work(u)
        t += max(n * f / (peak_tflops * 1e12), (n * io + w) / (hbm_gbs * 1e9))
    return t


def fused_ideal_s(plan, n, hbm_gbs, peak_tflops):
    F = sum(unit_work(u)[0] for u in plan.units)
    W = sum(unit_work(u)[2] for u in plan.units)
    io = 4 * (sum(plan.tensors[t].elements for t in plan.input_ids)
              + sum(plan.tensors[t].elements for t in plan.output_ids))
    return max(n * F / (peak_tflops * 1e12), (n * io + W) / (hbm_gbs * 1e9))


def total_flops(plan):
    return sum(unit_work(u)[0] for u in plan.units)
