"""compile() front half: lower the graph to launch units and fuse them.

Two groups of rewrites run in order:

1. The reference fusions, restated from pkg/src/nnjit/optimizer.py so that
   folded weights are bit-identical to the reference's:

   * ``fuse_activation`` (:220-242) -- a standalone activation joins the
     matvec unit immediately before it;
   * ``fuse_batchnorm`` (:286-325) -- BatchNorm folds into the producer's
     weights (case a), into the next Dense / 'valid' conv (case b, float64
     bias correction), or becomes a post-activation affine (case c);
   * both alternate to a fixpoint (``build_plan`` :328-341).

   A fusion needs the intermediate tensor to have exactly one consumer and to
   not be a network input/output (:189-193).

2. B200 epilogue fusions (new; each removes one launch and one HBM round
   trip of the intermediate tensor):

   * ``fuse_pool``     -- MaxPool 2x2/2 into the producing Conv2D's epilogue;
   * ``fuse_residual`` -- a binary Add into the epilogue of its later producer;
   * ``fuse_softmax``  -- a softmax over <= 32 values per row into the
     producing Dense / Conv2D epilogue.

The result is a :class:`FusionPlan` whose units map one-to-one onto
specialised sm_100a kernels (kernels.py).
"""

from dataclasses import dataclass, field, replace

import numpy as np

from .errors import UnsupportedLayer
from .graph import TensorShape
from .model_format import layer_weights

F32 = np.float32
MATVEC_KINDS = ("Dense", "Conv2D", "DepthwiseConv2D")
GEMM_KINDS = ("Dense", "Conv2D")
SOFTMAX_FUSE_MAX = 32


@dataclass
class CompilationUnit:
    uid: int
    kind: str          # Dense Conv2D DepthwiseConv2D Pool ElementwiseActivation
                       # Add Softmax Upsample Concat Copy Pad
    name: str
    input_ids: tuple
    output_id: int
    input_shapes: tuple
    output_shape: object
    kernel: object = None
    bias: object = None
    activation: str = "linear"
    post_scale: object = None
    post_offset: object = None
    scale: object = None
    offset: object = None
    stride: int = 1
    padding: str = "valid"
    kernel_hw: tuple = None
    pool_op: str = None
    factor: int = 1
    in_place_preference: int = None
    # -- B200 additions --
    pad: tuple = None               # Pad: ((top, bottom), (left, right))
    pool_after: bool = False        # fused 2x2/2 max-pool epilogue
    pre_pool_shape: object = None   # conv output shape before the fused pool
    residual_id: int = None         # fused residual Add: tensor added last
    softmax_after: bool = False     # fused row softmax epilogue
    upsample_after: int = 1         # fused nearest upsampling of the output
    pre_up_shape: object = None     # output shape before the fused upsampling
    concat_in: bool = False         # conv reads the channel concat of input_ids
    dw: object = None               # fused depthwise producer (a CompilationUnit)
    steps: list = None              # Chain: the fused units, in order
    dual_pool: object = None        # a 2x2 max-pool (Pool unit) computed from this conv's
                                    # output in its epilogue while the full output is stored
    gap: object = None              # Dense: the GlobalAveragePooling2D (a Pool unit) producing its
                                    # input, computed by the same launch (fuse_gap_dense)
    dw_after: object = None         # the DepthwiseConv2D (a unit) consuming this 1x1 conv's output,
                                    # computed in the conv's tcgen05 epilogue (fuse_pw_dw): the unit
                                    # then writes the depthwise output; its own output_id is only
                                    # written at batch sizes whose kernel lacks that epilogue

    def describe(self):
        bits = [self.kind, ",".join(map(str, self.input_shapes)) + f" -> {self.output_shape}"]
        if self.kind in ("Conv2D", "DepthwiseConv2D", "Pool"):
            kh, kw = self.kernel_hw
            bits.append(f"{self.pool_op or ''}{kh}x{kw}/s{self.stride} {self.padding}")
        if self.activation != "linear":
            bits.append(f"act={self.activation}")
        if self.post_scale is not None:
            bits.append("post_bn")
        if self.scale is not None:
            bits.append("affine")
        if self.pool_after:
            bits.append("+maxpool2")
        if self.residual_id is not None:
            bits.append(f"+add(t{self.residual_id})")
        if self.softmax_after:
            bits.append("+softmax")
        if self.upsample_after > 1:
            bits.append(f"+upsample{self.upsample_after}")
        if self.concat_in:
            bits.append("concat-loader")
        if self.dual_pool is not None:
            bits.append(f"+maxpool2->t{self.dual_pool.output_id}"
                        + (f"+upsample{self.dual_pool.upsample_after}"
                           if self.dual_pool.upsample_after > 1 else ""))
        if self.gap is not None:
            bits.append("gap-loader")
        if self.dw_after is not None and self.dw_after.kind == "Pool":
            bits.append(f"+gap->t{self.dw_after.output_id}")
        elif self.dw_after is not None:
            kh, kw = self.dw_after.kernel_hw
            bits.append(f"+dw{kh}x{kw}/s{self.dw_after.stride}->t{self.dw_after.output_id}")
        if self.steps:
            bits.append("[" + " | ".join(
                f"{st.kind}{'%dx%d/s%d' % (*st.kernel_hw, st.stride) if st.kernel_hw else ''}"
                f"->{st.output_shape}" for st in self.steps) + "]")
        if self.dw is not None:
            kh, kw = self.dw.kernel_hw
            bits.append(f"dw{kh}x{kw}/s{self.dw.stride}-loader"
                        + (f"(act={self.dw.activation})" if self.dw.activation != "linear" else ""))
        if self.in_place_preference is not None:
            bits.append("in_place?")
        return " ".join(bits)


@dataclass
class FusionPlan:
    units: list
    tensors: dict                  # tensor id -> TensorShape (per image)
    input_ids: tuple
    output_ids: tuple
    node_units: dict = field(default_factory=dict)

    def producer_positions(self):
        return {t: p for p, u in enumerate(self.units) for t in unit_writes(u)}

    def consumer_count(self, tid):
        return (sum(t == tid for u in self.units for t in self._reads(u))
                + sum(t == tid for t in self.output_ids))

    @staticmethod
    def _reads(u):
        return u.input_ids + ((u.residual_id,) if u.residual_id is not None else ())

    def describe(self):
        return "\n".join(f"  [{p:2d}] t{u.output_id:<3d} {u.describe()}"
                         for p, u in enumerate(self.units))


# ---------------------------------------------------------------------------
# lowering

def lower_to_units(graph):
    """One unit per layer; Flatten is a relabel (NHWC row-major == flat)."""
    alias = {}

    def res(t):
        while t in alias:
            t = alias[t]
        return t

    units, tensors, node_units = [], {}, {}
    next_tid = len(graph.nodes)

    def add_unit(**kw):
        u = CompilationUnit(uid=len(units), **kw)
        units.append(u)
        tensors[u.output_id] = u.output_shape
        return u

    for idx in graph.order:
        node = graph.nodes[idx]
        kind, cfg, shape = node.kind, node.config, node.output_shape
        w = layer_weights(node.spec, graph.weights) if node.spec.weight_refs else {}
        ins = tuple(res(i) for i in node.input_ids)
        in_shapes = tuple(graph.nodes[i].output_shape for i in node.input_ids)
        common = dict(name=node.name, input_ids=ins, output_id=idx,
                      input_shapes=in_shapes, output_shape=shape)
        if kind == "Input":
            tensors[idx] = shape
            node_units[idx] = None
            continue
        if kind == "Flatten":
            alias[idx] = ins[0]
            node_units[idx] = None
            continue
        zeros = lambda n: np.zeros(n, dtype=F32)
        if kind == "Dense":
            u = add_unit(kind="Dense", kernel=w["kernel"],
                         bias=w.get("bias", zeros(cfg["units"])),
                         activation=cfg["activation"], **common)
        elif kind in ("Conv2D", "DepthwiseConv2D"):
            nb = cfg["filters"] if kind == "Conv2D" else in_shapes[0].c
            u = add_unit(kind=kind, kernel=w["kernel"], bias=w.get("bias", zeros(nb)),
                         activation=cfg["activation"], stride=cfg["strides"],
                         padding=cfg["padding"], kernel_hw=cfg["kernel_size"], **common)
        elif kind == "SeparableConv2D":
            x = in_shapes[0]
            mid = TensorShape((shape.h, shape.w, x.c))
            dw = add_unit(kind="DepthwiseConv2D", name=node.name + "/depthwise",
                          input_ids=ins, output_id=next_tid, input_shapes=in_shapes,
                          output_shape=mid, kernel=w["depthwise"], bias=zeros(x.c),
                          stride=cfg["strides"], padding=cfg["padding"],
                          kernel_hw=cfg["kernel_size"])
            next_tid += 1
            u = add_unit(kind="Conv2D", name=node.name + "/pointwise",
                         input_ids=(dw.output_id,), output_id=idx, input_shapes=(mid,),
                         output_shape=shape, kernel=w["pointwise"],
                         bias=w.get("bias", zeros(cfg["filters"])),
                         activation=cfg["activation"], kernel_hw=(1, 1))
        elif kind in ("MaxPool2D", "AvgPool2D"):
            u = add_unit(kind="Pool", pool_op="max" if kind == "MaxPool2D" else "avg",
                         stride=cfg["strides"], padding=cfg["padding"],
                         kernel_hw=cfg["pool_size"], **common)
        elif kind == "GlobalAveragePooling2D":
            x = in_shapes[0]
            u = add_unit(kind="Pool", pool_op="avg", stride=1, padding="valid",
                         kernel_hw=(x.h, x.w), **common)
        elif kind == "ZeroPadding2D":
            u = add_unit(kind="Pad", pad=cfg["padding"], **common)
        elif kind == "BatchNorm":
            u = add_unit(kind="ElementwiseActivation", scale=w["scale"],
                         offset=w["offset"], in_place_preference=0, **common)
        elif kind == "Activation":
            u = add_unit(kind="ElementwiseActivation", activation=cfg["activation"],
                         in_place_preference=0, **common)
        elif kind == "Softmax":
            u = add_unit(kind="Softmax", in_place_preference=0, **common)
        elif kind == "UpSample2D":
            u = add_unit(kind="Upsample", factor=cfg["factor"], **common)
        elif kind == "Add":
            u = add_unit(kind="Add", in_place_preference=0, **common)
        elif kind == "Concatenate":
            u = add_unit(kind="Concat", **common)
        else:
            raise UnsupportedLayer(f"cannot lower layer kind '{kind}'")
        node_units[idx] = u.uid

    return FusionPlan(units=units, tensors=tensors,
                      input_ids=tuple(res(i) for i in graph.input_ids),
                      output_ids=tuple(res(o) for o in graph.output_ids),
                      node_units=node_units)


# ---------------------------------------------------------------------------
# reference fusions (pkg/src/nnjit/optimizer.py:189-341)

def _private(plan, tid):
    """Exactly one consumer and not network I/O."""
    return (tid not in plan.input_ids and tid not in plan.output_ids
            and plan.consumer_count(tid) == 1)


def _absorb_forward(plan, pos, into):
    """Delete units[pos]; ``into`` now produces the victim's output."""
    victim = plan.units[pos]
    plan.tensors.pop(into.output_id, None)
    into.output_id = victim.output_id
    _delete(plan, pos, into)


def _absorb_backward(plan, pos, into):
    """Delete units[pos]; ``into`` now reads the victim's input."""
    victim = plan.units[pos]
    into.input_ids = tuple(victim.input_ids[0] if t == victim.output_id else t
                           for t in into.input_ids)
    into.input_shapes = victim.input_shapes
    plan.tensors.pop(victim.output_id, None)
    _delete(plan, pos, into)


def _delete(plan, pos, into):
    victim = plan.units.pop(pos)
    plan.node_units = {n: (into.uid if u == victim.uid else u)
                       for n, u in plan.node_units.items()}


def fuse_activation(plan):
    progress = True
    while progress:
        progress = False
        for pos in range(1, len(plan.units)):
            u, p = plan.units[pos], plan.units[pos - 1]
            if (u.kind == "ElementwiseActivation" and u.scale is None
                    and p.kind in MATVEC_KINDS and p.output_id == u.input_ids[0]
                    and p.activation == "linear" and p.post_scale is None
                    and _private(plan, u.input_ids[0])):
                p.activation = u.activation
                _absorb_forward(plan, pos, p)
                progress = True
                break
    return plan


def _fold_after(u, s, o):
    # output channels are the last axis of all three kernel layouts
    u.kernel = np.multiply(u.kernel, s, dtype=F32)
    u.bias = np.add(np.multiply(u.bias, s, dtype=F32), o, dtype=F32)


def _fold_before(u, s, o):
    k = u.kernel
    if u.kind == "Dense":
        if k.shape[0] != len(s):          # channelwise affine seen through Flatten
            reps = k.shape[0] // len(s)
            s, o = np.tile(s, reps), np.tile(o, reps)
        extra = k.astype(np.float64).T @ o.astype(np.float64)
        u.kernel = np.multiply(k, s[:, None], dtype=F32)
    elif u.kind == "Conv2D":
        extra = np.tensordot(k.astype(np.float64), o.astype(np.float64),
                             axes=([2], [0])).sum((0, 1))
        u.kernel = np.multiply(k, s[None, None, :, None], dtype=F32)
    else:
        extra = (k.astype(np.float64) * o.astype(np.float64)).sum((0, 1))
        u.kernel = np.multiply(k, s, dtype=F32)
    u.bias = (u.bias.astype(np.float64) + extra).astype(F32)


def _post_affine(u, s, o):
    if u.post_scale is None:
        u.post_scale, u.post_offset = s.astype(F32), o.astype(F32)
    else:
        u.post_offset = np.add(np.multiply(u.post_offset, s, dtype=F32), o, dtype=F32)
        u.post_scale = np.multiply(u.post_scale, s, dtype=F32)


def fuse_batchnorm(plan):
    progress = True
    while progress:
        progress = False
        for pos, u in enumerate(plan.units):
            if u.kind != "ElementwiseActivation" or u.scale is None:
                continue
            bn_in, bn_out = u.input_ids[0], u.output_id
            if pos > 0:
                p = plan.units[pos - 1]
                if (p.kind in MATVEC_KINDS and p.output_id == bn_in
                        and len(u.scale) == p.output_shape.dims[-1]
                        and _private(plan, bn_in)):
                    if p.activation == "linear" and p.post_scale is None:
                        _fold_after(p, u.scale, u.offset)
                    else:
                        _post_affine(p, u.scale, u.offset)
                    _absorb_forward(plan, pos, p)
                    progress = True
                    break
            if pos + 1 < len(plan.units):
                c = plan.units[pos + 1]
                folds = c.kind == "Dense" or (c.kind in ("Conv2D", "DepthwiseConv2D")
                                              and c.padding == "valid")
                if folds and bn_out in c.input_ids and _private(plan, bn_out):
                    _fold_before(c, u.scale, u.offset)
                    _absorb_backward(plan, pos, c)
                    progress = True
                    break
    return plan


def build_reference_plan(graph):
    """The reference's unit list (lowering + fusion fixpoint)."""
    plan = lower_to_units(graph)
    while True:
        n = len(plan.units)
        fuse_batchnorm(fuse_activation(plan))
        if len(plan.units) == n:
            return plan


# ---------------------------------------------------------------------------
# B200 epilogue fusions

def _pool_fusable(p, u):
    if not (u.kind == "Pool" and u.pool_op == "max" and u.kernel_hw == (2, 2)
            and u.stride == 2):
        return False
    h, w = p.output_shape.h, p.output_shape.w
    return u.padding == "valid" or (h % 2 == 0 and w % 2 == 0)


def fuse_pool(plan):
    pos = 1
    while pos < len(plan.units):
        u, p = plan.units[pos], plan.units[pos - 1]
        if (p.kind == "Conv2D" and not p.pool_after and p.residual_id is None
                and not p.softmax_after and p.output_id == u.input_ids[0]
                and _pool_fusable(p, u) and _private(plan, p.output_id)):
            p.pre_pool_shape = p.output_shape
            p.output_shape = u.output_shape
            p.pool_after = True
            _absorb_forward(plan, pos, p)
            continue
        pos += 1
    return plan


def fuse_residual(plan):
    pos = 0
    while pos < len(plan.units):
        u = plan.units[pos]
        if u.kind == "Add" and len(u.input_ids) == 2 and u.input_ids[0] != u.input_ids[1]:
            where = plan.producer_positions()
            cand = [(where.get(t, -1), k) for k, t in enumerate(u.input_ids)]
            ppos, k = max(cand)
            if ppos >= 0:
                p = plan.units[ppos]
                tid = u.input_ids[k]
                if (p.kind in GEMM_KINDS and not p.pool_after and p.residual_id is None
                        and not p.softmax_after and _private(plan, tid)):
                    p.residual_id = u.input_ids[1 - k]
                    plan.tensors.pop(p.output_id, None)
                    p.output_id = u.output_id
                    _delete(plan, pos, p)
                    continue
        pos += 1
    return plan


def fuse_softmax(plan):
    pos = 1
    while pos < len(plan.units):
        u, p = plan.units[pos], plan.units[pos - 1]
        if (u.kind == "Softmax" and p.kind in GEMM_KINDS and p.output_id == u.input_ids[0]
                and not p.pool_after and not p.softmax_after
                and p.output_shape.dims[-1] <= SOFTMAX_FUSE_MAX
                and _private(plan, p.output_id)):
            p.softmax_after = True
            _absorb_forward(plan, pos, p)
            continue
        pos += 1
    return plan


def fuse_upsample(plan):
    """Nearest UpSample2D into the epilogue of its producer (Conv2D / Pool):
    each computed pixel is stored to its f x f replicas."""
    pos = 0
    while pos < len(plan.units):
        u = plan.units[pos]
        if u.kind == "Upsample":
            where = plan.producer_positions()
            ppos = where.get(u.input_ids[0], -1)
            if ppos >= 0:
                p = plan.units[ppos]
                if (p.kind in ("Conv2D", "Pool") and p.upsample_after == 1 and not p.pool_after
                        and not p.softmax_after and p.residual_id is None
                        and p.output_shape.rank == 3 and _private(plan, p.output_id)):
                    p.pre_up_shape = p.output_shape
                    p.output_shape = u.output_shape
                    p.upsample_after = u.factor
                    plan.tensors.pop(p.output_id, None)
                    p.output_id = u.output_id
                    _delete(plan, pos, p)
                    continue
        pos += 1
    return plan


def unit_writes(u):
    """Tensors a unit writes: its output, a dual-stored pooled map, and the
    output of a depthwise conv computed in its epilogue."""
    dp = getattr(u, "dual_pool", None)
    da = getattr(u, "dw_after", None)
    return ((u.output_id,) + ((dp.output_id,) if dp is not None else ())
            + ((da.output_id,) if da is not None else ()))


def fuse_pool_dual(plan):
    """A 2x2/2 max-pool whose input is a conv output that other units read
    as well (an encoder skip of cfg4) becomes a second store of that conv's
    epilogue: the conv writes its full output AND the pooled (and, if the
    pool's output is upsampled, replicated) map, so the pooled tensor costs
    no re-read of the full one and no launch.  Kernels that do not implement
    the second store get the pool as a separate launch (kernels.py)."""
    pos = 1
    while pos < len(plan.units):
        u = plan.units[pos]
        where = plan.producer_positions()
        ppos = where.get(u.input_ids[0], -1) if u.kind == "Pool" else -1
        if ppos >= 0:
            p = plan.units[ppos]
            if (p.kind == "Conv2D" and not p.pool_after and p.residual_id is None
                    and not p.softmax_after and p.upsample_after == 1 and p.dual_pool is None
                    and p.dw is None and p.output_shape.rank == 3 and _pool_fusable(p, u)
                    and u.residual_id is None and not _private(plan, p.output_id)
                    and ppos == pos - 1):
                p.dual_pool = u
                _delete(plan, pos, p)
                continue
        pos += 1
    return plan


def fuse_concat(plan):
    """A two-way channel Concatenate feeding only a stride-1 Conv2D becomes a
    two-source operand loader of that conv (no concatenated tensor)."""
    pos = 0
    while pos < len(plan.units):
        u = plan.units[pos]
        if (u.kind == "Concat" and len(u.input_ids) == 2 and u.output_shape.rank == 3
                and u.input_ids[0] != u.input_ids[1] and _private(plan, u.output_id)):
            cons = [c for c in plan.units if u.output_id in FusionPlan._reads(c)]
            c0 = u.input_shapes[0].c
            ctot = u.output_shape.c
            if (len(cons) == 1 and cons[0].kind == "Conv2D" and cons[0].stride == 1
                    and not cons[0].concat_in and cons[0].input_ids == (u.output_id,)
                    and c0 % 4 == 0 and ctot > 8):
                c = cons[0]
                c.input_ids = u.input_ids
                c.input_shapes = u.input_shapes
                c.concat_in = True
                plan.tensors.pop(u.output_id, None)
                _delete(plan, pos, c)
                continue
        pos += 1
    return plan


SEP_SMEM_MAX = 232448      # dynamic shared memory per block (227 KB opt-in)
SEP_CI_MAX = 32            # depthwise channels = pointwise K of the fused kernel
SEP_CO_MAX = 32            # pointwise outputs (weights as FFMA immediates)
SEP_SPLIT_MAX_WARPS = 0    # resident warps per SM up to which a pixel is shared by two threads
                           # (0: never -- measured slower on B200, see sep_narrow_geometry.split)


def sep_narrow_geometry(d, u, smem_max=SEP_SMEM_MAX, force=None):
    """Tile geometry (TH output rows, NS ring stages, NT threads, shared bytes)
    of the fused depthwise + narrow pointwise kernel (nnb_sep.cuh) for the
    depthwise unit ``d`` feeding the 1x1 conv ``u``, or None when the pair is
    outside that kernel: pointwise with <= 32 output channels over <= 32
    input channels (weights as FFMA immediates) and a zero-haloed input band
    that leaves >= 2 CTAs of >= 128 threads per SM.  Stride-2 depthwise
    layers need 4x the band per output pixel and fall outside."""
    h, w, c = d.input_shapes[0].dims
    ho, wo, _ = d.output_shape.dims
    co = u.output_shape.c
    kh, kw = d.kernel_hw
    s = d.stride
    if not (c % 4 == 0 and c <= SEP_CI_MAX and co <= SEP_CO_MAX and wo <= 512 and kh <= 7 and kw <= 7
            and not u.pool_after and u.upsample_after == 1 and not u.softmax_after
            and not u.concat_in):
        return None
    cp = c + 4 if ((c + 4) // 4) % 2 else c + 8
    wb = (wo - 1) * s + kw
    rs = (co | 1) if co % 4 else (co + 4 if ((co + 4) // 4) % 2 else co + 8)
    def split(g):
        """Two threads per pixel (nnb_sep.cuh SP) when the band leaves the SM
        at most SEP_SPLIT_MAX_WARPS warps: the same shared memory then feeds
        twice the warps (cfg3's 32-channel blocks run 2 CTAs x 4 warps per
        SM).  Measured on B200 (bit-identical outputs): cfg3 @256 dw C=16 +
        pw 32 27.2 -> 29.2 us, dw C=32 + pw 32 26.3 -> 31.2 us, cfg2 @1024 dw
        C=16 + pw 32 63.7 -> 73.9 us -- these kernels are bound by shared-memory
        wavefronts and issue slots (ncu: short scoreboard / MIO stalls), not by
        latency, and the exchange row adds to both.  Kept behind
        ``sep_geo=(TH, NS, 2)``; off by default."""
        nt, smem = g["NT"], g["smem"]
        warps = max(1, min(smem_max // (smem + 1024), 2048 // nt)) * nt // 32
        px = g["TH"] * wo
        smem2 = smem + 4 * px * max(0, cp - rs)      # the exchange rows share the output staging
        if (c % 8 == 0 and co % 8 == 0 and warps <= SEP_SPLIT_MAX_WARPS and 2 * nt <= 1024
                and smem2 + 1024 <= smem_max):
            return dict(g, NT=2 * nt, smem=smem2, SP=2)
        return dict(g, SP=1)

    if force:                                       # (TH, NS[, SP]) for experiments
        th, ns = force[:2]
        ri = (th - 1) * s + kh
        smem = 4 * (ns * ri * wb * cp + th * wo * rs)
        g = dict(TH=th, NS=ns, NT=-(-th * wo // 32) * 32, smem=smem)
        if len(force) > 2:
            return (dict(g, NT=2 * g["NT"], smem=smem + 4 * th * wo * max(0, cp - rs), SP=2) if force[2] == 2
                    else dict(g, SP=1))
        return split(g)
    # two ring stages, tiles of 4-8 warps; the band height that issues the
    # fewest warps per image (idle lanes of a tile's last warp, ragged last
    # band), then the smaller tile (more CTAs per SM).  Measured (cfg2 block 1,
    # 1024 images): TH 2/3/4/5/6/8 -> 73.9/63.9/70.6/74.0/70.5/74.3 us (three
    # stages never helped); cfg3 block 1 (64 px rows): TH 2/4 -> 31.1/29.2 us.
    best = None
    for th in range(1, ho + 1):
        if th * wo < min(97, ho * wo):
            continue
        ri = (th - 1) * s + kh
        nt = -(-th * wo // 32) * 32
        if nt > max(256, -(-wo // 32) * 32):
            break
        smem = 4 * (2 * ri * wb * cp + th * wo * rs)
        if smem + 1024 > smem_max:
            break
        key = (nt // 32 * -(-ho // th), th)
        if best is None or key < best[0]:
            best = (key, dict(TH=th, NS=2, NT=nt, smem=smem))
    if best:
        return split(best[1])
    return None


def fuse_dw_pw(plan, narrow_only=False):
    """DepthwiseConv2D feeding only a pointwise (1x1, stride 1) Conv2D becomes
    that conv's operand loader: the depthwise output is computed on the fly
    and never written to memory (separable-conv blocks of cfg2/cfg3).  With
    ``narrow_only`` only pairs the fused depthwise + narrow pointwise kernel
    takes (``sep_narrow_geometry``) are fused."""
    pos = 1
    while pos < len(plan.units):
        u, d = plan.units[pos], plan.units[pos - 1]
        if (u.kind == "Conv2D" and d.kind == "DepthwiseConv2D" and u.kernel_hw == (1, 1)
                and u.stride == 1 and u.input_ids == (d.output_id,) and u.dw is None
                and not u.concat_in and d.residual_id is None and not d.pool_after
                and d.upsample_after == 1 and d.input_shapes[0].c % 4 == 0
                and (not narrow_only or sep_narrow_geometry(d, u) is not None)
                and _private(plan, d.output_id)):
            u.dw = d
            u.input_ids = d.input_ids
            u.input_shapes = d.input_shapes
            plan.tensors.pop(d.output_id, None)
            _delete(plan, pos - 1, u)
            continue
        pos += 1
    return plan


GAP_DENSE_MAX_CO = 32      # one output per lane (nnb_small.cuh GapDense)


def fuse_gap_dense(plan):
    """GlobalAveragePooling2D feeding only a Dense with <= 32 outputs (cfg2's
    128 -> 4 head) becomes that Dense's loader: one warp per image pools the
    map and forms the outputs, one launch instead of two that each move a few
    kilobytes per image."""
    pos = 1
    while pos < len(plan.units):
        u, p = plan.units[pos], plan.units[pos - 1]
        if (u.kind == "Dense" and p.kind == "Pool" and p.pool_op == "avg" and u.gap is None
                and u.input_ids == (p.output_id,) and p.input_shapes[0].rank == 3
                and tuple(p.kernel_hw) == tuple(p.input_shapes[0].dims[:2])
                and p.output_shape.elements == p.input_shapes[0].c and p.padding == "valid"
                and p.upsample_after == 1 and p.residual_id is None and u.residual_id is None
                and p.input_shapes[0].c % 4 == 0 and u.kernel.shape[1] <= GAP_DENSE_MAX_CO
                and u.kernel.shape[0] == p.input_shapes[0].c and _private(plan, p.output_id)):
            u.gap = p
            u.input_ids = p.input_ids
            u.input_shapes = p.input_shapes
            plan.tensors.pop(p.output_id, None)
            _delete(plan, pos - 1, u)
            continue
        pos += 1
    return plan


PW_DW_TILE_ROWS = 128      # rows of a tcgen05 row tile (nnb_gemm_tc.cuh BM)
PW_DW_MIN_CO = 32


def pw_dw_ok(u, d, bands=False):
    """Geometry of a pointwise conv ``u`` whose consumer ``d`` (depthwise) the
    tcgen05 epilogue can compute: a 128-row tile holds whole images (8x8 and
    4x4 maps: 2 and 8 images), so every tap of the depthwise window lies in
    the tile the CTA has just finished."""
    h, w, c = u.output_shape.dims
    kh, kw = d.kernel_hw
    whole = PW_DW_TILE_ROWS % (h * w) == 0
    if d.kind == "Pool":
        # GlobalAveragePooling2D of a map the tile holds whole: the same parked
        # tile, summed over each image's rows (cfg3's 4x4x256 map ahead of the classifier)
        return (whole and w <= 16 and c % 4 == 0 and c >= PW_DW_MIN_CO and d.pool_op == "avg"
                and (kh, kw) == (h, w) and d.padding == "valid" and d.output_shape.elements == c
                and u.input_shapes[0].c % 4 == 0)
    # larger maps of <= 16 columns as bands of 128 / w image rows: the overlap
    # rows of neighbouring bands are recomputed by the 1x1 conv (cfg3's 16x16
    # stage: 3 bands of 8 rows per image for 3x3 taps, stride 1 or 2)
    # Measured on B200 (cfg3 @256): the two band kernels take 19.6 + 17.2 us
    # against 11.4 + 11.3 and 13.8 + 7.2 us for the separate launches, but the
    # replay goes 0.2377 -> 0.2452 ms: a CTA walks ~5 band tiles and its eight
    # epilogue warps run drain, park, taps and stores of each one after the
    # other, while the separate depthwise launch overlaps its neighbours
    # (PDL).  Opt-in (``pw_dw="bands"``).
    band = (bands and not whole and PW_DW_TILE_ROWS % w == 0 and PW_DW_TILE_ROWS // w >= max(8, kh)
            and h * w > PW_DW_TILE_ROWS)
    return ((whole or band) and w <= 16 and c % 4 == 0 and c >= PW_DW_MIN_CO
            and kh <= 5 and kw <= 5 and d.stride in (1, 2)
            and u.input_shapes[0].c % 4 == 0)


def fuse_pw_dw(plan, bands=False):
    """A pointwise (1x1, stride 1) Conv2D whose only consumer is a
    DepthwiseConv2D over a map small enough that a 128-row GEMM tile holds
    whole images (cfg3's 8x8 and 4x4 stages) or a band of 8 or more rows of a
    map at most 16 pixels wide (its 16x16 stage) computes that depthwise conv in
    its tcgen05 epilogue (nnb_gemm_tc.cuh EDW): the finished tile stays in
    shared memory, the depthwise taps read it there, and only the depthwise
    output is stored -- one launch and one round trip through memory less per
    separable block.  The pointwise output keeps its buffer: batch sizes
    served by kernels without that epilogue write it and run the depthwise
    conv as its own launch (kernels.py)."""
    pos = 0
    while pos + 1 < len(plan.units):
        u, d = plan.units[pos], plan.units[pos + 1]
        if (u.kind == "Conv2D" and d.kind in ("DepthwiseConv2D", "Pool") and u.kernel_hw == (1, 1)
                and u.stride == 1 and d.input_ids == (u.output_id,) and u.dw is None
                and u.dw_after is None and u.dual_pool is None and not u.concat_in
                and not u.pool_after and u.upsample_after == 1 and not u.softmax_after
                and u.residual_id is None and d.residual_id is None and not d.pool_after
                and d.upsample_after == 1 and not d.softmax_after and d.dw_after is None
                and u.output_shape.rank == 3 and pw_dw_ok(u, d, bands)
                and _private(plan, u.output_id)):
            u.dw_after = d
            _delete(plan, pos + 1, u)
        pos += 1
    return plan


# ---------------------------------------------------------------------------
# layer chains: a run of small depthwise / pointwise layers in one kernel

CHAIN_THREADS = 256          # nnb_chain.cuh block size
CHAIN_SMEM_MAX = 200 * 1024  # staged input + two activation buffers per CTA
CHAIN_MIN_STEPS = 4


def chain_stride(pixels):
    """Channel stride (floats) of a channel-major activation in the chain's
    shared memory: odd, so lanes reading different channels of one pixel hit
    different banks."""
    return pixels | 1


def chain_bytes(shape):
    h, w, c = shape.dims
    return 4 * chain_stride(h * w) * c


def chain_pw_tile(pixels, co):
    """(TP pixels, TC channels) per thread of a chain pointwise step with
    CHAIN_THREADS threads covering pixels x co outputs, or None."""
    e = pixels * co
    if e % CHAIN_THREADS:
        return None
    e //= CHAIN_THREADS
    for tc in (8, 4):
        if e % tc == 0 and co % tc == 0:
            tp = e // tc
            if 1 <= tp <= 8 and pixels % tp == 0:
                return tp, tc
    return None


def _chain_step_ok(u):
    if (u.residual_id is not None or u.pool_after or u.upsample_after != 1 or u.softmax_after
            or u.concat_in or u.dw is not None or u.scale is not None or u.steps
            or len(u.input_ids) != 1 or u.input_shapes[0].rank != 3):
        return False
    if u.kind == "DepthwiseConv2D":
        return u.kernel_hw[0] <= 5 and u.kernel_hw[1] <= 5
    if u.kind == "Conv2D":
        h, w, co = u.output_shape.dims
        return (u.kernel_hw == (1, 1) and u.stride == 1
                and chain_pw_tile(h * w, co) is not None)
    return False


def _chain_gap(u):
    """A global average pool (GlobalAveragePooling2D / AvgPool2D over the
    whole map) closing a chain."""
    x = u.input_shapes[0]
    return (u.kind == "Pool" and u.pool_op == "avg" and x.rank == 3
            and tuple(u.kernel_hw) == (x.h, x.w) and u.padding == "valid"
            and u.upsample_after == 1 and u.residual_id is None)


def chain_smem(steps):
    """Shared bytes of a chain: its staged input and two buffers sized for
    the largest intermediate."""
    inner = [chain_bytes(st.output_shape) for st in steps[:-1]]
    return chain_bytes(steps[0].input_shapes[0]) + 2 * max(inner)


def fuse_chain(plan, smem_max=CHAIN_SMEM_MAX, min_steps=CHAIN_MIN_STEPS):
    """Runs of depthwise and pointwise (1x1) convs over small maps -- the
    8x8 / 4x4 tail of MobileNet-style nets, ending in an optional global
    average pool -- become one ``Chain`` unit: one CTA per image keeps every
    intermediate in shared memory (nnb_chain.cuh), so the run costs one
    launch and one HBM round trip instead of one per layer.  A run starts at
    the earliest layer whose staged input plus two intermediate buffers fit
    ``smem_max``.

    Opt-in (``tuning={"chain": True}``): measured on B200 (cfg3, 20 steps from
    16x16x32 to the GAP) 0.399 ms at 256 images and 0.199 ms at one image,
    against 0.126 / 0.07 ms for the same layers as per-layer launches (tcgen05
    row GEMMs + depthwise kernels).  One CTA per image is bound by its FFMA
    issue and L2 weight-load latency (9.5 M FMA per image on one SM), where
    the per-layer kernels spread every layer over all SMs on tensor cores."""
    pos = 0
    while pos < len(plan.units):
        run = [pos]
        while (_chain_step_ok(plan.units[run[-1]]) and run[-1] + 1 < len(plan.units)):
            nxt = plan.units[run[-1] + 1]
            prev = plan.units[run[-1]]
            if not (nxt.input_ids == (prev.output_id,) and _private(plan, prev.output_id)):
                break
            if _chain_step_ok(nxt):
                run.append(run[-1] + 1)
            elif _chain_gap(nxt):
                run.append(run[-1] + 1)
                break
            else:
                break
        if not _chain_step_ok(plan.units[run[0]]):
            pos += 1
            continue
        units = [plan.units[i] for i in run]
        start = 0
        while start + min_steps <= len(units) and chain_smem(units[start:]) > smem_max:
            start += 1
        units = units[start:]
        if len(units) < min_steps or chain_smem(units) > smem_max:
            pos = run[-1] + 1
            continue
        first, last = units[0], units[-1]
        chain = CompilationUnit(uid=first.uid, kind="Chain", name=f"chain({first.name}..{last.name})",
                                input_ids=first.input_ids, output_id=last.output_id,
                                input_shapes=first.input_shapes, output_shape=last.output_shape,
                                steps=units)
        p0 = run[0] + start
        for st in units[:-1]:
            plan.tensors.pop(st.output_id, None)
        for _ in units:
            victim = plan.units.pop(p0)
            plan.node_units = {n: (chain.uid if u == victim.uid else u)
                               for n, u in plan.node_units.items()}
        plan.units.insert(p0, chain)
        pos = p0 + 1
    return plan


TC_CHAIN_ROWS = 128          # nnb_tcchain.cuh: two images of <= 64 pixels per M=128 tile
TC_CHAIN_MIN_PW = 3


def _tcc_ok_dw(u, first):
    if (u.kind != "DepthwiseConv2D" or u.residual_id is not None or u.pool_after
            or u.upsample_after != 1 or u.softmax_after or u.scale is not None
            or len(u.input_ids) != 1 or u.input_shapes[0].rank != 3):
        return False
    h, w, c = u.input_shapes[0].dims
    ho, wo, _ = u.output_shape.dims
    return (c % 32 == 0 and c <= 128 and ho * wo <= 64 and u.kernel_hw[0] <= 5
            and u.kernel_hw[1] <= 5 and (first or h * w <= 64))


def _tcc_ok_pw(u):
    if (u.kind != "Conv2D" or u.kernel_hw != (1, 1) or u.stride != 1 or u.residual_id is not None
            or u.pool_after or u.upsample_after != 1 or u.softmax_after or u.concat_in
            or u.dw is not None or u.dual_pool is not None):
        return False
    h, w, n = u.output_shape.dims
    k = u.input_shapes[0].c
    return h * w <= 64 and k % 32 == 0 and k <= 128 and n % 16 == 0 and n <= 128


def fuse_tc_chain(plan, min_pw=TC_CHAIN_MIN_PW):
    """Alternating pointwise / depthwise layers over maps of <= 64 pixels (the
    8x8 stage of MobileNet-style nets) become one ``TcChain`` unit run by a
    tensor-core kernel holding two images per CTA for the whole run
    (nnb_tcchain.cuh): pw (tcgen05 3xTF32; the first one reads its input from
    the arena straight into TMEM), dw (CUDA cores, into TMEM), pw, ...,
    optionally a closing depthwise.  Every intermediate stays on chip.  The
    run needs ``min_pw`` pointwise layers.  (A run starting at a depthwise
    layer would read that layer's 3x3 input windows from L2 -- 4.6x the input
    bytes through a CTA's load path; the standalone depthwise kernel does that
    step faster.)

    Opt-in (``tuning={"tc_chain": True}``).  Measured on B200, cfg3 @256 (12
    layers, 8x8x64 -> 4x4x128): 73 us for the chain against ~80 us for the
    same layers as 12 launches (replay 0.264 vs 0.263 ms with the extra
    depthwise launch ahead of it); batch 1: 68 us vs ~45 us.  Ablations
    (NNB_TCC_DBG): the depthwise layers are 35 us of it (shared-memory
    bandwidth: every output re-reads its 9 taps, 590 KB per layer per CTA),
    the 3xTF32 MMAs 10 us, epilogues / barriers 25 us -- one CTA per image
    pair serialises all three, where per-layer launches spread every layer
    over all SMs."""
    pos = 0
    while pos < len(plan.units):
        u0 = plan.units[pos]
        if not (_tcc_ok_pw(u0) and u0.input_shapes[0].rank == 3
                and u0.input_shapes[0].h * u0.input_shapes[0].w <= 64):
            pos += 1
            continue
        run = [pos]
        while run[-1] + 1 < len(plan.units):
            prev, nxt = plan.units[run[-1]], plan.units[run[-1] + 1]
            if not (nxt.input_ids == (prev.output_id,) and _private(plan, prev.output_id)):
                break
            want_pw = prev.kind == "DepthwiseConv2D"
            if want_pw and _tcc_ok_pw(nxt) and nxt.input_shapes[0].c == prev.output_shape.c:
                run.append(run[-1] + 1)
            elif not want_pw and _tcc_ok_dw(nxt, False):
                run.append(run[-1] + 1)
            else:
                break
        n_pw = sum(plan.units[i].kind == "Conv2D" for i in run)
        if n_pw < min_pw:
            pos = run[-1] + 1
            continue
        units = [plan.units[i] for i in run]
        first, last = units[0], units[-1]
        chain = CompilationUnit(uid=first.uid, kind="TcChain",
                                name=f"tcchain({first.name}..{last.name})",
                                input_ids=first.input_ids, output_id=last.output_id,
                                input_shapes=first.input_shapes, output_shape=last.output_shape,
                                steps=units)
        for st in units[:-1]:
            plan.tensors.pop(st.output_id, None)
        for _ in units:
            victim = plan.units.pop(run[0])
            plan.node_units = {n: (chain.uid if u == victim.uid else u)
                               for n, u in plan.node_units.items()}
        plan.units.insert(run[0], chain)
        pos = run[0] + 1
    return plan


def build_plan(graph, gpu_fusion=True, dw_fusion="narrow", chain=False, tc_chain=False,
               pw_dw=True, gap_dense=True):
    """Reference fusions to a fixpoint, then the B200 epilogue fusions.
    ``dw_fusion`` folds depthwise convs into the pointwise conv that consumes
    them.  "narrow" (default): only pairs whose pointwise conv has <= 32
    output channels, run by the fused depthwise + narrow pointwise kernel
    (nnb_sep.cuh).  True: every pair, the wider ones through the FFMA GEMM's
    operand loader or the tcgen05 GEMM's split warps (kernels.py tc_dwf) --
    measured on B200 that only breaks even with a depthwise kernel followed by
    the tcgen05 pointwise GEMM (cfg3 @256: 30.6 vs 32.4 us, 37.7 vs 34.0 us
    per block; cfg2 @1024: 113 vs 109 us): the fused kernel is bound by the
    depthwise math on its four split warps.  False: no depthwise fusion."""
    plan = build_reference_plan(graph)
    if gpu_fusion:
        apply_gpu_fusions(plan, dw_fusion, chain, tc_chain, pw_dw, gap_dense)
    return plan


def apply_gpu_fusions(plan, dw_fusion="narrow", chain=False, tc_chain=False, pw_dw=True,
                      gap_dense=True):
    """The B200 epilogue fusions, in place, on a reference-fused plan."""
    fuse_pool(plan)
    fuse_residual(plan)
    fuse_softmax(plan)
    fuse_upsample(plan)
    fuse_pool_dual(plan)
    fuse_concat(plan)
    if dw_fusion:
        fuse_dw_pw(plan, narrow_only=dw_fusion == "narrow")
    if tc_chain:
        fuse_tc_chain(plan)
    if chain:
        fuse_chain(plan)
    if pw_dw and not chain and not tc_chain:
        fuse_pw_dw(plan, bands=pw_dw == "bands")
    if gap_dense and not chain and not tc_chain:
        fuse_gap_dense(plan)
    return plan


# fields of the reference's CompilationUnit (pkg/src/nnjit/optimizer.py:35-57)
REFERENCE_UNIT_FIELDS = ("uid", "kind", "name", "input_ids", "output_id", "input_shapes",
                         "output_shape", "kernel", "bias", "activation", "post_scale",
                         "post_offset", "scale", "offset", "stride", "padding", "kernel_hw",
                         "pool_op", "factor", "in_place_preference")


def adopt_plan(plan, gpu_fusion=True, dw_fusion="narrow", chain=False, tc_chain=False,
               pw_dw=True, gap_dense=True):
    """A plan made by the REFERENCE's planner (``nnjit.build_plan``,
    pkg/src/nnjit/optimizer.py:328-341: a FusionPlan of CompilationUnits,
    :35-91) as this package's FusionPlan, with the B200 epilogue fusions
    applied on top -- the binding that lets a maintainer keep the reference's
    planner and hand its output to ``kernels.specialize`` (INTEGRATION.md
    section 3).  A plan of this package passes through unchanged.  Unit
    fields are copied by name, tensor shapes re-made as graph.TensorShape;
    the folded arrays are used as they are (bit-identical either way,
    tests/test_planner.py)."""
    if isinstance(plan, FusionPlan):
        return plan

    def shape(s):
        return TensorShape(tuple(int(d) for d in s.dims))

    units = []
    for u in plan.units:
        kw = {f: getattr(u, f) for f in REFERENCE_UNIT_FIELDS}
        kw["input_ids"] = tuple(kw["input_ids"])
        kw["input_shapes"] = tuple(shape(s) for s in kw["input_shapes"])
        kw["output_shape"] = shape(kw["output_shape"])
        if kw["kernel_hw"] is not None:
            kw["kernel_hw"] = tuple(kw["kernel_hw"])
        units.append(CompilationUnit(**kw))
    ours = FusionPlan(units, {t: shape(s) for t, s in plan.tensors.items()},
                      tuple(plan.input_ids), tuple(plan.output_ids), dict(plan.node_units))
    if gpu_fusion:
        apply_gpu_fusions(ours, dw_fusion, chain, tc_chain, pw_dw, gap_dense)
    return ours


def describe_plan(plan):
    return plan.describe()
