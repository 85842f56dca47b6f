"""Algorithmic work per launch and the per-launch roofline.

    T_roof(N) = sum_launch max(N * F_u * m(k) / P_pipe(k), (N * (In_u + Out_u) + W_u) / BW)

summed over the launches a replay over N images runs, each launch ``k``
serving one fused unit ``u`` of the plan actually compiled:

* ``F_u``: 2 x MACs for Dense / Conv2D / DepthwiseConv2D (a fused depthwise
  producer adds its own), one op per element per tap for pooling, one per
  element per input for Add, one per element for BatchNorm / activation /
  softmax; data movement (upsample, concat, pad) is free.
* ``In_u`` / ``Out_u``: float32 activation bytes per image of the FUSED unit
  (a fused pool / softmax / residual / concat changes what is read and
  written); ``W_u``: weight, bias and affine bytes, read once per launch.
* ``P_pipe(k)`` by the kernel the specialiser selected for the launch:
  - tcgen05 kernels (``*_tc_*``): the dense TF32 tensor rate, taken as half
    the MEASURED bf16 rate (MEASURED_PEAKS.json ``bf16_tflops``: tcgen05
    issues K=8 TF32 in the time of K=16 BF16), with ``m(k)`` = 3 executed
    products per FP32 MAC for the 3xTF32 split, 2 TF32-equivalents with the
    BF16 correction split (one TF32 product + one BF16 K=16 MMA);
  - every other kernel: the FP32 FFMA peak MEASURED by ``nnb_ffma_peak``
    (16 independent FFMA chains per thread, 8 x 148 blocks; 71.8 TFLOP/s on
    the pool's B200, profiles/r02_ffma_peak.json), ``m`` = 1.
* ``BW``: the measured HBM copy bandwidth (MEASURED_PEAKS.json ``hbm_gbs``).

``survey_*`` keep SURVEY.md 8(d)'s original formula over the reference-style
plan (BN folded, activations fused, nothing else fused) for comparison; with
one FFMA peak for every unit it over-credits tensor-core layers and is not a
fraction of anything the hardware can do.
"""

import json
import pathlib

SM_COUNT = 148
FFMA_LANES = 128
MAX_SM_MHZ = 1965.0
ROOT = pathlib.Path(__file__).resolve().parent.parent


def fp32_peak_tflops(mhz=MAX_SM_MHZ):
    """Derived FFMA peak: 148 SM x 128 lanes x 2 x f_clk (74.4 TF at 1965 MHz)."""
    return SM_COUNT * FFMA_LANES * 2 * mhz * 1e6 / 1e12


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback"}


def ffma_peak_tflops(live=None):
    """(TFLOP/s, source): ``live`` (a fresh nnb_ffma_peak reading) if given,
    else the committed measurement, else the derived figure."""
    if live:
        return float(live), "nnb_ffma_peak measured in this run"
    p = ROOT / "profiles" / "r02_ffma_peak.json"
    if p.exists():
        return float(json.loads(p.read_text())["ffma_tflops"]), f"profiles/{p.name}"
    return fp32_peak_tflops(), "derived 148 SM x 128 x 2 x 1965 MHz"


def tf32_peak_tflops(peaks):
    """Dense TF32 tensor rate: half the measured dense bf16 rate."""
    return peaks["bf16_tflops"] / 2.0


def launch_pipe(launch):
    """(pipe, products per FP32 MAC) of the kernel a launch runs."""
    if "_tc_" in launch.kernel or "tcchain" in launch.kernel:
        return ("tensor", 2 if "bf16 corr" in launch.note else 3)
    return ("ffma", 1)


def launch_roofline(unit, launch, n, peaks, ffma_tflops):
    """Roofline of one launch over ``n`` images (a dict; times in µs)."""
    f, io, w = unit_work(unit)
    pipe, mult = launch_pipe(launch)
    p = tf32_peak_tflops(peaks) if pipe == "tensor" else ffma_tflops
    t_c = n * f * mult / (p * 1e12)
    t_m = (n * io + w) / (peaks["hbm_gbs"] * 1e9)
    return {"kernel": launch.kernel, "pipe": pipe, "products_per_mac": mult,
            "flops": n * f, "bytes": n * io + w, "peak_tflops": p,
            "t_compute_us": t_c * 1e6, "t_hbm_us": t_m * 1e6,
            "bound": "compute" if t_c >= t_m else "hbm", "roof_us": max(t_c, t_m) * 1e6}


def net_roofline(net, n, peaks, ffma_tflops, launch_ms=None):
    """Per-launch rooflines of a compiled network's replay over ``n`` images
    and, when ``launch_ms`` ({launch index: measured ms}) is given, each
    launch's achieved fraction.  Returns (rows, total roof µs)."""
    rows, total = [], 0.0
    for i in net.launches_for(n):
        L = net.artifact.launches[i]
        r = launch_roofline(net.plan.units[L.unit], L, n, peaks, ffma_tflops)
        if launch_ms is not None and i in launch_ms:
            r["measured_us"] = launch_ms[i] * 1e3
            r["frac"] = r["roof_us"] / r["measured_us"]
        total += r["roof_us"]
        rows.append(r)
    return rows, total


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
    if k in ("Chain", "TcChain"):  # fused run: its steps' work, chain input + output bytes
        f = wb = 0
        for st in u.steps:
            sf, _, sw = unit_work(st)
            f, wb = f + sf, wb + sw
        return f, ins + out, wb
    if k == "Dense":
        kin, units = u.kernel.shape
        f = 2 * kin * units
        if getattr(u, "gap", None) is not None:      # pooled by the same launch
            f += u.input_shapes[0].elements
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
    dp = getattr(u, "dual_pool", None)
    if dp is not None:             # second, pooled store of the output
        pf, _, _ = unit_work(dp)
        f += pf
        out += 4 * dp.output_shape.elements
    da = getattr(u, "dw_after", None)
    if da is not None:             # depthwise conv in the epilogue: only its output is stored
        df, _, dwb = unit_work(da)
        f += df
        wb += dwb
        out += 4 * (da.output_shape.elements - u.output_shape.elements)
    d = getattr(u, "dw", None)
    if d is not None:              # fused depthwise producer
        df, _, dwb = unit_work(d)
        f += df
        wb += dwb
    return f, ins + out, wb


def layer_roofline(net, ref_plan, n, peaks, ffma_tflops):
    """north_star's "per-layer memory or compute roofline" with the per-pipe
    peaks of ``launch_roofline``: the sum over the LAYERS of the reference-
    style plan (BatchNorm folded, activations fused, nothing else -- one unit
    per Dense / conv / depthwise / pool / ... layer, ``planner.build_reference_plan``)
    of max(compute at the pipe that runs the layer, its own bytes / HBM
    bandwidth).  Compute pipe of a layer: Dense / Conv2D take the pipe of the
    launch that covers them in the compiled network at batch ``n`` (tcgen05
    with its 3 or 2 products per MAC, else FFMA); every other layer --
    depthwise taps, pooling, elementwise, also when a tcgen05 launch carries
    them in its epilogue -- is FFMA work.  Unlike ``net_roofline`` (per fused
    LAUNCH) this bound keeps the activation traffic between layers that the
    compiled network's fusions remove, so a fused launch can beat its layers'
    sum.  Returns (µs, rows)."""
    by_uid = {u.uid: pos for pos, u in enumerate(net.plan.units)}
    for pos, u in enumerate(net.plan.units):          # units carried inside another one
        for inner in (getattr(u, "dw", None), getattr(u, "dw_after", None),
                      getattr(u, "dual_pool", None), getattr(u, "gap", None)):
            if inner is not None:
                by_uid.setdefault(inner.uid, pos)
        for st in getattr(u, "steps", None) or ():
            by_uid.setdefault(st.uid, pos)
    node_of = {}
    for node, uid in ref_plan.node_units.items():
        if uid is not None:
            node_of.setdefault(uid, node)
    active = [net.artifact.launches[i] for i in net.launches_for(n)]
    total, rows = 0.0, []
    for ru in ref_plan.units:
        pipe, mult = "ffma", 1
        if ru.kind in ("Dense", "Conv2D"):
            ours = net.plan.node_units.get(node_of.get(ru.uid))
            pos = by_uid.get(ours)
            main = [L for L in active if L.unit == pos]
            if main:
                pipe, mult = launch_pipe(main[0])
        f, io, w = unit_work(ru)
        p = tf32_peak_tflops(peaks) if pipe == "tensor" else ffma_tflops
        t_c = n * f * mult / (p * 1e12)
        t_m = (n * io + w) / (peaks["hbm_gbs"] * 1e9)
        t = max(t_c, t_m)
        total += t
        rows.append({"layer": ru.name, "kind": ru.kind, "pipe": pipe, "products_per_mac": mult,
                     "roof_us": t * 1e6, "bound": "compute" if t_c >= t_m else "hbm"})
    return total * 1e6, rows


def survey_layerwise_roof_s(plan, n, hbm_gbs, peak_tflops):
    t = 0.0
    for u in plan.units:
        f, io, w = unit_work(u)
        t += max(n * f / (peak_tflops * 1e12), (n * io + w) / (hbm_gbs * 1e9))
    return t


def survey_fused_ideal_s(plan, n, hbm_gbs, peak_tflops):
    F = sum(unit_work(u)[0] for u in plan.units)
    W = sum(unit_work(u)[2] for u in plan.units)
    io = 4 * (sum(plan.tensors[t].elements for t in plan.input_ids)
              + sum(plan.tensors[t].elements for t in plan.output_ids))
    return max(n * F / (peak_tflops * 1e12), (n * io + W) / (hbm_gbs * 1e9))


def total_flops(plan):
    return sum(unit_work(u)[0] for u in plan.units)
