"""compile() back half: specialise every launch unit into sm_100a CUDA.

This replaces the reference's machine-code emitters (pkg/src/nnjit/codegen/
compile.py:25-51, emitters.py:651-667).  Where the reference bakes arena and
constant-pool displacements into x86 instructions, we bake them into a
``struct Cfg_uNN`` of ``constexpr`` members and instantiate one of the kernel
templates under ``csrc/kernels`` with it.  NVRTC (inside the C-ABI runtime)
compiles the whole translation unit for sm_100a, so every loop bound, stride,
offset and padding split is a compile-time constant -- the paper's runtime
specialisation idea, with the device doing the arithmetic.

Every kernel has the same entry signature as the reference's generated
function (``f(arena, pool)``, pkg/README.md:187) plus the batch count:
``void k(const float* pool, float* arena, int n)``.

Outputs: the CUDA source, a list of :class:`Launch` records and the device
weight pool (a deduplicated, 256-byte aligned blob, cf. codegen/pool.py).
"""

import hashlib
from dataclasses import dataclass, field

import re

import numpy as np

from .errors import UnsupportedLayer
from .graph import same_padding
from .planner import _private, sep_narrow_geometry

F32 = np.float32

ACT_CODE = {"linear": 0, "relu": 1, "sigmoid": 2, "tanh": 3, "relu6": 4, "elu": 5}
MODE_CODE = {"rational": 0, "fast": 1, "exact": 2}
SMEXP_CODE = {"fast": 0, "precise": 1, "exact": 2}

SMALL_M = 8           # Dense rows at or below this use the split-K GEMV kernel
TC_MIN_K = 32         # tensor-core GEMM eligibility (contraction and output width)
TC_MIN_N = 32
TC_MIN_ROWS = 256     # GEMM rows per launch from which the tcgen05 kernel is used
# Dense layers up to this many rows take the split-K row kernel (weights read
# once per 8 rows).  Measured (cfg1): 256 rows 0.062 ms vs 0.070 on tcgen05,
# 512 rows 0.096 vs 0.070; 1024 rows on the FFMA GEMM 0.228 vs 0.070 (the old
# 2048-row tcgen05 threshold); cfg3 @64 0.162 -> 0.146 ms with 1x1 convs of
# 1024 rows on tcgen05.
SMALL_DENSE_ROWS = 256
# with mega=True small batches must stay off the TMA-based tcgen05 kernels
# (the persistent kernel walks plain-pointer units only)
MEGA_TC_MIN_ROWS = 2048
TC_MIN_IMAGES = 17    # convolutions: images per launch from which TC_MIN_ROWS applies,
TC_CONV_MIN_ROWS = 2048   # ... below it this many rows
WIDE_MIN_TILES = 148  # 256x256 tiles per launch from which N = 256 tiles are used
SMEM_MAX = 232448      # dynamic shared memory per block (227 KB opt-in)
MEGA_MAX_N = 8         # batches up to this run as one persistent kernel (when eligible)
MEGA_THREADS = 256     # its block size (units with larger blocks opt it out)
MAX_TMAPS = 6         # tensor-map parameters of every TMA kernel (NNB_MAX_TMAPS)
NARROW_MAX_W = 2048   # K*CO bound of the narrow row GEMM (weights unrolled into its code)
ELEM_BLOCK = 256
SEP_BLOCK = 128
# direct conv: taps fully unrolled with the weights as immediates up to this
# many unrolled FFMAs per thread (KH*KW*CI*CO*pixels); beyond it shared-memory
# weights and a rolled kernel-row loop keep NVRTC under the compile budget
DIRECT_UNROLL_MAX = 2048
DIRECT_SPLIT_MAX = 2304
CB16_CONV_MIN_K = 128     # conv tiles from this K take the BF16 correction products
TINY_MAX_N = 64           # batches up to this run the whole net as one TinyNet launch ...
TINY_ARENA_MAX = 160 * 1024   # ... when the per-image arena fits shared memory
TINY_WEIGHTS_MAX = 96 * 1024  # ... and the weights are small (staged in shared memory)
TINY_SMEM_MAX = 200 * 1024    # arena + weights   # ... and with a pool window split over two lanes


@dataclass
class Launch:
    """One kernel launch of the schedule (mirrors ``nnb_launch`` in
    include/nnb.h)."""
    kernel: str
    block: int
    smem: int
    items_per_image: int
    items_per_block: int
    grid_mult: int = 1
    n_min: int = 1
    n_max: int = 1 << 30
    unit: int = -1
    note: str = ""
    grid_cap: int = 0                 # persistent kernels: at most this many CTAs
    tmaps: list = field(default_factory=list)   # TMA descriptors (see nnb_tmap)
    cluster: int = 1                  # thread-block cluster size along x (CTA pairs: 2)
    cooperative: bool = False         # co-resident grid (the batch-1 persistent kernel)
    zero_offset: int = -1             # arena byte offset of a u32 zeroed before the launch


class DevicePool:
    """Deduplicated weight/constant blob; every entry 256-byte aligned."""

    def __init__(self):
        self.data = bytearray()
        self._seen = {}

    def add(self, arr):
        raw = np.ascontiguousarray(arr, dtype="<f4").tobytes()
        key = hashlib.sha1(raw).digest() + len(raw).to_bytes(8, "little")
        if key in self._seen:
            return self._seen[key]
        off = len(self.data)
        self.data += raw
        self.data += bytes((-len(self.data)) % 256)
        self._seen[key] = off
        return off

    def zeros_offset(self, n):
        return self.add(np.zeros(max(n, 1), F32))

    def mark(self):
        return len(self.data), dict(self._seen)

    def rollback(self, mark):
        """Forget every entry added since ``mark``."""
        self.data = self.data[:mark[0]]
        self._seen = mark[1]


@dataclass
class Specialization:
    source: str                 # all units in one translation unit (inspection)
    launches: list
    pool: bytes
    kernel_names: list
    sources: list = field(default_factory=list)      # one TU per kernel (NVRTC jobs)
    kernel_source: list = field(default_factory=list)
    notes: dict = field(default_factory=dict)
    arena_extra: int = 0        # bytes the runtime appends to the arena (mega barrier)
    mega_source: str = ""       # the persistent kernel's TU ("" when not generated)


def _cfg_struct(name, fields, code=""):
    """``struct name`` of constexpr fields, plus generated member functions.
    ``code`` is member source text, or an :class:`ImmTables` (whose tables
    are emitted at namespace scope in front of the struct), or a list of
    both."""
    parts = code if isinstance(code, list) else [code]
    pre = [p.declarations(name) for p in parts if isinstance(p, ImmTables)]
    members = [p.members(name) if isinstance(p, ImmTables) else p for p in parts]
    lines = pre + [f"struct {name} {{"]
    for k, v in fields.items():
        if isinstance(v, bool):
            v = int(v)
        lines.append(f"  static constexpr long long {k} = {int(v)}LL;")
    lines += [m for m in members if m]
    lines.append("};")
    return "\n".join(lines)


class ImmTables:
    """float32 tables read as ``Cfg::name(i)``.  Each is a namespace-scope
    ``__device__ const`` array: once the caller's loops are unrolled the index
    is a constant and NVVM folds the load into an instruction immediate.
    (A function-local ``const float v[N] = {...}`` gives the same code but
    is re-materialised at every call site: cfg0's direct conv with 1152
    weights took 43 s of NVRTC that way, 1.2 s with this form.)"""

    def __init__(self, **tables):
        self.tables = {k: np.asarray(v, F32).ravel() for k, v in tables.items()}

    def declarations(self, cfg):
        return "\n".join(f"__device__ const float nnb_{cfg}_{k}[{max(a.size, 1)}] = "
                         f"{{{', '.join(_flit(v) for v in a) or '0.0f'}}};"
                         for k, a in self.tables.items())

    def members(self, cfg):
        return "\n".join(f"  __device__ static __forceinline__ float {k}(int i) "
                         f"{{ return nnb_{cfg}_{k}[i]; }}" for k in self.tables)


def _flit(x):
    """Exact CUDA literal of a float32 value (hex float; bit pattern if not finite)."""
    x = np.float32(x)
    if np.isfinite(x):
        return float(x).hex() + "f"
    return f"__int_as_float(0x{int(np.array(x).view(np.uint32)):08x})"


def _narrow_code(wmat, bias, K, CO, KS):
    """Members ``bias(j)`` and ``dot(a, acc, ks)`` of a RowsNarrow config: the
    unrolled K x CO FFMAs of k-slice ``ks`` with every weight an immediate
    (k ascending within the slice, columns innermost)."""
    w = np.asarray(wmat, F32).reshape(K, CO)
    out = ["  __device__ static __forceinline__ float bias(int j) {",
           f"    const float b[{CO}] = {{{', '.join(_flit(v) for v in np.asarray(bias, F32))}}};",
           "    return b[j];", "  }",
           "  __device__ static __forceinline__ void dot(const float* a, float* acc, int ks) {",
           "    float4 v;", "    switch (ks) {"]
    per = K // KS
    for ks in range(KS):
        out.append(f"    case {ks}:")
        for k4 in range(ks * per, (ks + 1) * per, 4):
            out.append(f"      v = *reinterpret_cast<const float4*>(a + {k4});")
            for q, c in enumerate("xyzw"):
                out.extend(f"      acc[{j}] = fmaf(v.{c}, {_flit(w[k4 + q, j])}, acc[{j}]);"
                           for j in range(CO))
        out.append("      break;")
    out += ["    }", "  }"]
    return "\n".join(out)


def _sep_code(wmat, bias, K, CO, dw_kernel, dw_bias, sp=1):
    """Members of a SepNarrow config: ``dww(i)`` / ``dwb(c)`` (depthwise
    weights in (ky, kx, c) order and bias, folded to immediates once the
    kernel's loops are unrolled), ``bias(j)`` and ``dotr(a, acc)``: the
    unrolled K x CO pointwise FFMAs over a register row ``a`` with every
    weight an immediate (k ascending, columns innermost: RowsNarrow's order
    with one K slice)."""
    w = np.asarray(wmat, F32).reshape(K, CO)
    out = []
    # sp = 2: ``dotr`` forms the lower half of the output channels and
    # ``dotr1`` the upper half (two threads per pixel, nnb_sep.cuh SP)
    coh = CO // sp
    for half in range(sp):
        out.append(f"  __device__ static __forceinline__ void dotr{half or ''}"
                   f"(const float (&a)[{K}], float* acc) {{")
        for k in range(K):
            out.extend(f"    acc[{j}] = fmaf(a[{k}], {_flit(w[k, half * coh + j])}, acc[{j}]);"
                       for j in range(coh))
        out.append("  }")
    return [ImmTables(dww=dw_kernel, dwb=dw_bias, bias=bias), "\n".join(out)]


def _imm_tables(**tables):
    """Members ``name(i)`` returning element i of a float32 table; once the
    caller's loops are unrolled the index is a constant and the value an
    instruction immediate (see :class:`ImmTables`)."""
    return ImmTables(**tables)


def _pad4(x):
    return (x + 3) // 4 * 4


class Specializer:
    def __init__(self, plan, assignment, options, max_batch, capacity, use_tc=True,
                 sm_count=148, tc_min_rows=TC_MIN_ROWS, tmem_a=True, nacc=None, aldg=False,
                 kpack=True, kpack9=True, kpack_wide=True, tiny=False, early_mma=True, epi_tma=True, csplit=True, chunk=None, split_rn=True,
                 pair=True, tc_tile_use=0.75, mega=False, abuf=None, small_dense_rows=SMALL_DENSE_ROWS, tc_min_images=TC_MIN_IMAGES,
                 tc_min_k=TC_MIN_K, wide=True, wide_bk=32, wide_chunk=None,
                 wide_csplit=True, rn_ss=2, corr_bf16="wide", cb16_w4=True, conv_w4="auto", rowshare=True, small_conv=True, small_conv_kper=16, a_prefetch=0, narrow=True, direct_imm=True, sep_fma=True, narrow_geo=None, head=True, sep_geo=None, setreg=True, epi16=False):
        self.use_tc = use_tc
        self.sep_geo = sep_geo
        self.corr_bf16 = corr_bf16
        self.conv_w4 = conv_w4
        self.rowshare = rowshare
        self.small_conv = small_conv
        self.setreg = setreg
        self.epi16 = epi16
        self.small_conv_kper = small_conv_kper
        self.cb16_w4 = cb16_w4
        self.a_prefetch = a_prefetch
        self.tc_min_images = tc_min_images
        self.head = head
        self.head_cap = {}           # unit pos -> largest n its own launches serve
        self._n_cap = None
        self.narrow_geo = narrow_geo
        self.direct_imm = direct_imm
        self.sep_fma = sep_fma
        self.narrow = narrow
        self.aldg = aldg
        self.kpack = kpack
        self.kpack9 = kpack9
        self.tiny = tiny
        self.early_mma = early_mma
        self.kpack_wide = kpack_wide
        self.epi_tma = epi_tma
        self.csplit = csplit
        self.split_rn = split_rn
        self.pair = pair
        self.tc_tile_use = tc_tile_use
        self.mega = mega
        self.abuf = abuf
        self.small_dense_rows = small_dense_rows
        self.tc_min_k = tc_min_k
        self.wide = wide
        self.wide_bk = wide_bk
        self.wide_chunk = wide_chunk
        self.wide_csplit = wide_csplit
        self.rn_ss = rn_ss
        self.unit_src = {}            # launch index -> (cfg name, struct, template, dynamic smem)
        self._dual_from = 1 << 30     # lowest batch whose conv launch stores the dual pool
        self._edw_from = 1 << 30      # ... whose 1x1 conv launch computes the following depthwise conv
        self._n_floor = 1             # regular launches serve batches >= this (TinyNet below)
        self.chunk = chunk
        self.nacc = nacc
        self.tmem_a = tmem_a
        self.tc_min_rows = tc_min_rows
        self.sm_count = sm_count
        self.plan = plan
        self.asg = assignment
        self.opt = options
        self.max_batch = max_batch
        self.cap = capacity
        self.pool = DevicePool()
        self.chunks = []
        self.launches = []
        self.names = []

    # -- helpers -----------------------------------------------------------
    def arena_off(self, tid):
        return self.asg.offsets[tid][0] * self.cap

    def img_bytes(self, tid):
        return 4 * self.plan.tensors[tid].elements

    def emit(self, unit_pos, tag, template, fields, block, smem, ipi, ipb,
             grid_mult=1, n_min=1, n_max=1 << 30, dynamic_smem=False, note="",
             tmaps=(), grid_cap=0, cluster=1, code=""):
        if self._n_cap is not None:          # batches above the cap run fused elsewhere
            n_max = min(n_max, self._n_cap)
            if n_min > n_max:
                return
        if self._n_floor > 1:                # batches below the floor run as one TinyNet launch
            n_min = max(n_min, self._n_floor)
            if n_min > n_max:
                return
        kname = f"nnb_u{unit_pos:02d}_{tag}_{len(self.names)}"
        cfg = f"Cfg_{len(self.names)}"
        body = _cfg_struct(cfg, fields, code)
        if tmaps:
            body += (f"\nextern \"C\" __global__ void __launch_bounds__({block}, 1) {kname}("
                     f"const float* __restrict__ pool, float* __restrict__ arena, int n, "
                     + ", ".join(f"const __grid_constant__ nnb::TmaDesc tm{k}"
                                 for k in range(MAX_TMAPS)) + ") {\n"
                     f"  NNB_PDL_PROLOGUE\n"
                     f"  {template}<{cfg}>::run(pool, arena, n, "
                     + ", ".join(f"&tm{k}" for k in range(MAX_TMAPS)) + ");\n}\n")
            tmaps = list(tmaps) + [tmaps[0]] * (MAX_TMAPS - len(tmaps))
            self.chunks.append(body)
            self.names.append(kname)
            self.launches.append(Launch(kname, block, smem, ipi, ipb, grid_mult, n_min, n_max,
                                        unit_pos, note, grid_cap, list(tmaps), cluster))
            return
        self.unit_src[len(self.launches)] = (cfg, body, template, dynamic_smem)
        if dynamic_smem:
            call = (f"  extern __shared__ __align__(16) unsigned char nnb_smem[];\n"
                    f"  {template}<{cfg}>::run(pool, arena, n, "
                    f"*reinterpret_cast<{template}<{cfg}>::Smem*>(nnb_smem));\n")
        else:
            call = f"  {template}<{cfg}>::run(pool, arena, n);\n"
        body += (f"\nextern \"C\" __global__ void __launch_bounds__({block}) {kname}("
                 f"const float* __restrict__ pool, float* __restrict__ arena, int n) {{\n"
                 f"  NNB_PDL_PROLOGUE\n" + call + "}\n")
        self.chunks.append(body)
        self.names.append(kname)
        self.launches.append(Launch(kname, block, smem, ipi, ipb, grid_mult, n_min,
                                    n_max, unit_pos, note, grid_cap))

    def epilogue_fields(self, u, co):
        ps = po = self.pool.zeros_offset(co)
        post = u.post_scale is not None
        if post:
            ps, po = self.pool.add(u.post_scale), self.pool.add(u.post_offset)
        return dict(ACT=ACT_CODE[u.activation], MODE=MODE_CODE[self.opt.activation_mode],
                    POST=post, PS_OFF=ps, PO_OFF=po)

    # -- unit kinds ----------------------------------------------------------
    def gemm(self, pos, u):
        """Conv2D (any window) and Dense through the FFMA implicit GEMM."""
        x = u.input_shapes[0]
        if u.kind == "Dense":
            H = W = 1
            CI = x.elements
            KH = KW = S = 1
            PT = PL = 0
            CO = u.kernel.shape[1]
            HO = WO = 1
            wmat = np.asarray(u.kernel, F32)
        elif u.dw is not None:
            # fused depthwise loader: the GEMM's input map is the dw output
            H, W, CI = u.dw.output_shape.dims
            KH = KW = S = 1
            PT = PL = 0
            HO, WO, CO = u.output_shape.dims
            conv_out = u.output_shape
            wmat = np.asarray(u.kernel, F32).reshape(CI, CO)
        else:
            H, W = x.h, x.w
            CI = sum(sh.c for sh in u.input_shapes)      # concat loader: both sources
            KH, KW = u.kernel_hw
            S = u.stride
            conv_out = (u.pre_pool_shape if u.pool_after else
                        u.pre_up_shape if u.upsample_after > 1 else u.output_shape)
            HO, WO, CO = conv_out.dims
            if u.padding == "same":
                PT, PL = same_padding(H, KH, S)[0], same_padding(W, KW, S)[0]
            else:
                PT = PL = 0
            wmat = np.asarray(u.kernel, F32).reshape(KH * KW * CI, CO)
        K = KH * KW * CI
        pool_fused = bool(u.pool_after)
        UPF = u.upsample_after
        concat = bool(u.concat_in)
        C0 = u.input_shapes[0].c if concat else CI
        src1 = dict(CONCAT=concat, C0=C0, UPF=UPF,
                    IN1_OFF=self.arena_off(u.input_ids[1]) if concat else 0,
                    IN1_IMG=self.img_bytes(u.input_ids[1]) if concat else 0)
        src1.update(self._dw_fields(u))
        if pool_fused:
            PHO, PWO = u.output_shape.h, u.output_shape.w
            rows = PHO * PWO * 4
        else:
            PHO = PWO = 1
            rows = HO * WO
        softmax = bool(u.softmax_after)

        if u.kind == "Dense" and self.max_batch > 0:
            # batch-1 latency path: split-K GEMV (also used for tiny batches)
            self._dense_small(pos, u, wmat, CI, CO, softmax,
                              n_max=min(SMALL_M, self.max_batch))
            if self.max_batch <= SMALL_M:
                return
            n_min = SMALL_M + 1
            # a few hundred rows: the same split-K kernel with 8 rows per block
            # keeps every SM busy, where a tiled GEMM would run a handful of
            # CTAs through a serial K loop
            # (narrow layers hand over to the tensor cores earlier: cfg0's
            # Dense 256->32 at 256 rows 0.039 -> 0.033 ms replay on tcgen05,
            # cfg1's 1024->512 at 256 rows 0.062 here vs 0.070 there)
            # (and so do wide ones with a short K: cfg3's Dense 256->1000 at 256
            # rows 16.7 -> 12.7 us on tcgen05)
            sdr = (self.small_dense_rows if 64 < CO <= 512 or CI > 256
                   else min(self.small_dense_rows, 128))
            if sdr > SMALL_M:
                hi = min(sdr, self.max_batch)
                self._dense_small(pos, u, wmat, CI, CO, softmax, n_max=hi, mb=8, n_min=n_min)
                if self.max_batch <= hi:
                    return
                n_min = hi + 1
        else:
            n_min = 1
            # few-pixel pointwise convs (batch-1 latency): while the tiled GEMM
            # (16 x 64 tiles) would not fill one wave of CTAs, the split-K row
            # kernel (1 / 2 / 4 pixels per block, 16 k per warp) -- the GEMM
            # runs a handful of CTAs through a serial K loop.  Measured (warm
            # replays): cfg3 @1 0.103 -> 0.058 ms, @16 0.113 -> 0.100, cfg2
            # @1 0.033 -> 0.029 ms; from a full wave on it loses (cfg3 @64
            # 0.142 -> 0.152 ms with it on the 4x4 layers)
            n_hi = 0
            if (u.kind == "Conv2D" and KH == KW == S == 1 and PT == PL == 0 and not concat
                    and not pool_fused and UPF == 1 and u.dw is None and not softmax
                    and self.small_conv and self.max_batch > 0):
                n_hi = min(self.max_batch, 16 * ((self.sm_count - 1) // -(-CO // 64)) // rows)
            if n_hi > 0:
                lo = 1
                for mb, m_cap in ((1, 256), (2, 1024), (4, 1 << 30)):
                    hi = min(n_hi, m_cap // rows)
                    if hi >= lo:
                        # (the opt-in persistent kernel takes blocks of <= MEGA_THREADS)
                        kper = max(self.small_conv_kper, CI // (MEGA_THREADS // 32)) if self.mega \
                            else self.small_conv_kper
                        self._dense_small(pos, u, wmat, CI, CO, False, n_min=lo, n_max=hi, rows=rows,
                                          mb=mb, kper=kper)
                        lo = hi + 1
                if self.max_batch <= n_hi:
                    return
                n_min = n_hi + 1

        # depthwise producer + narrow pointwise conv: one fused kernel
        # (nnb_sep.cuh, all batch sizes)
        if u.dw is not None and self.narrow:
            geo = sep_narrow_geometry(u.dw, u)
            if geo is not None and self.sep_geo:
                geo = sep_narrow_geometry(u.dw, u, force=self.sep_geo)
            if geo is not None:
                self._sep_narrow(pos, u, wmat, CI, CO, geo)
                return

        # narrow inputs: direct FFMA convolution (all batch sizes)
        if (u.kind == "Conv2D" and not softmax and CO <= 32 and u.dw is None
                and (CI <= 4 or (CI <= 8 and pool_fused and CO <= 16)
                     or (CI <= 16 and pool_fused and CO <= 16 and self.direct_imm
                         and KH * KW * CI * CO <= DIRECT_SPLIT_MAX))):
            assert not concat
            self._conv_direct(pos, u, wmat, H, W, CI, HO, WO, CO, KH, KW, S, PT, PL,
                              pool_fused, PHO, PWO, UPF, n_min=n_min)
            return

        # tensor-core path for large dense contractions (3xTF32, FP32-accurate)
        n_max = 1 << 30
        # (a concatenated input is not one row-major matrix: the row GEMM's
        # single A map cannot read it, so fused concats go to the conv tiles
        # or the SIMT loader)
        tc_rows = (self.use_tc and not softmax and not pool_fused and KH == KW == S == 1
                   and u.dw is None and not concat
                   and PT == PL == 0 and K % 4 == 0 and K >= self.tc_min_k and CO >= TC_MIN_N)
        # implicit-GEMM tiles are 8 x 16 output pixels of one image: small images
        # waste most of a tile (cfg0's 8x8 conv: 0.103 ms on tensor cores vs
        # 0.046 ms as an FFMA GEMM), so require tc_tile_use (75%) useful pixels
        tile_use = (HO * WO) / ((-(-HO // 8) * 8) * (-(-WO // 16) * 16))
        tc_conv = (self.use_tc and not tc_rows and u.kind == "Conv2D" and not softmax
                   and S == 1 and (KH * KW > 1 or concat) and CI % 16 == 0 and C0 % 16 == 0
                   and CO >= 16
                   and tile_use >= self.tc_tile_use)
        # pointwise conv with its depthwise producer fused in (planner
        # fuse_dw_pw): 8 x 16-pixel tiles whose A operand the split warps
        # compute from a TMA'd depthwise-input halo
        tc_dwf = (self.use_tc and u.dw is not None and u.kind == "Conv2D" and not softmax
                  and not pool_fused and UPF == 1 and not concat and KH == KW == S == 1
                  and CI % 16 == 0 and CO >= 16 and u.dw.stride in (1, 2)
                  and tile_use >= self.tc_tile_use)
        if tc_rows or tc_conv or tc_dwf:
            n_tc = max(n_min, -(-self.tc_min_rows // rows))
            if u.kind == "Dense" and self.tc_min_rows == TC_MIN_ROWS:
                n_tc = n_min          # right after the split-K row kernel's range
            if rows > 1 and self.tc_min_rows == TC_MIN_ROWS:
                # convolutions: below TC_MIN_IMAGES images the FFMA kernels
                # keep launches under TC_CONV_MIN_ROWS rows (measured: with
                # tcgen05 1x1 convs from 256 rows, batch-1 latency cfg2 41 ->
                # 47 us, cfg3 141 -> 145 us, cfg3 @16 0.117 -> 0.123 ms; @20
                # 0.144 -> 0.125, @24 0.145 -> 0.127, @32 0.131 -> 0.129, @64
                # 0.161 -> 0.146 ms)
                n_tc = max(n_min, min(max(n_tc, self.tc_min_images), -(-TC_CONV_MIN_ROWS // rows)))
            if n_tc <= self.max_batch:
                conv = None
                if tc_conv:
                    conv = dict(H=H, W=W, CI=CI, HO=HO, WO=WO, KH=KH, KW=KW, PT=PT, PL=PL,
                                POOL=pool_fused, PHO=PHO, PWO=PWO, C0=C0,
                                CONCAT=concat, UPF=UPF)
                if tc_dwf:
                    conv = dict(H=HO, W=WO, CI=CI, HO=HO, WO=WO, KH=1, KW=1, PT=0, PL=0,
                                POOL=False, PHO=1, PWO=1, C0=CI, CONCAT=False, UPF=1, DWF=1)
                edw = u.dw_after if (tc_rows and u.dw_after is not None and u.kind == "Conv2D"
                                     and u.residual_id is None and UPF == 1) else None
                self._gemm_tc(pos, u, wmat, K, CO, rows, n_tc, conv,
                              rows_geo=dict(HO=HO, WO=WO, UPF=UPF),
                              head=self._head_candidate(pos, u) if not conv else None, edw=edw)
                n_max = n_tc - 1
                if n_max < n_min:
                    return

        # many rows, at most 32 columns: stream contiguous row tiles through a
        # cp.async ring, weights baked into the code (nnb_rows.cuh), once the
        # batch gives every SM a tile
        rows_contig = (u.kind == "Dense" or (KH == KW == S == 1 and PT == PL == 0 and not concat
                                             and not pool_fused and UPF == 1 and u.dw is None))
        if self.narrow and rows_contig and CO <= 32 and K % 4 == 0 and K * CO <= NARROW_MAX_W:
            KS = next(ks for ks in (4, 2, 1) if K % (4 * ks) == 0 and K // ks >= 16 or ks == 1)
            TR = 32 if KS > 1 else 64
            if self.narrow_geo:                      # (KS, TR) override for experiments
                KS, TR = self.narrow_geo
            ast = K + 4 if ((K + 4) // 4) % 2 else K + 8
            fixed = (max(KS - 1, 1) + 1) * TR * (CO | 1)
            NS = min(4, (SMEM_MAX // 16 - fixed) // (TR * ast))    # four CTAs per SM
            if NS < 2:
                NS = min(4, (SMEM_MAX // 8 - fixed) // (TR * ast))
            if NS < 2:
                NS = min(4, (SMEM_MAX // 4 - fixed) // (TR * ast))
            n_lo = max(n_min, -(-self.sm_count * TR // rows))
            if NS >= 2 and n_lo <= min(n_max, self.max_batch):
                smem = 4 * (NS * TR * ast + fixed)
                fields = dict(K=K, CO=CO, TR=TR, NS=NS, KS=KS, ROWS=rows,
                              IN_OFF=self.arena_off(u.input_ids[0]),
                              OUT_OFF=self.arena_off(u.output_id),
                              RES=u.residual_id is not None,
                              RES_OFF=self.arena_off(u.residual_id) if u.residual_id is not None else 0,
                              SOFTMAX=softmax, SMEXP=SMEXP_CODE[self.opt.softmax_exp])
                fields.update(self.epilogue_fields(u, CO))
                per_sm = max(1, min(SMEM_MAX // (smem + 1024), 2048 // (TR * KS)))
                self.emit(pos, "dense_narrow" if u.kind == "Dense" else "conv1x1_narrow", "nnb::RowsNarrow",
                          fields, TR * KS, smem, rows, TR, n_min=n_lo, n_max=n_max, dynamic_smem=True,
                          grid_cap=self.sm_count * per_sm,
                          code=_narrow_code(wmat, u.bias, K, CO, KS),
                          note=f"narrow rows M=n*{rows} N={CO} K={K} {TR}-row tiles, K in {KS} slices, "
                               f"{NS}-stage cp.async ring, weights as FFMA immediates")
                n_max = n_lo - 1
                if n_max < n_min:
                    return

        # tile shape
        if softmax:
            TN = _pad4(CO)
            NTX = 1
            TM = 4 if TN <= 16 else 2
        elif CO <= 4:
            TN, NTX, TM = 4, 1, 4
        elif CO <= 8:
            TN, NTX, TM = 8, 1, 4 if K > 32 else 2
        elif CO <= 16:
            TN, NTX, TM = 8, 2, 4
        elif CO <= 32:
            TN, NTX, TM = 8, 4, 8
        else:
            TN, NTX, TM = 8, 8, 8
        if pool_fused and TM % 4:
            TM = 4
        NT = 128
        BN = TN * NTX
        ntile_n = (CO + BN - 1) // BN
        wo = self.pool.add(wmat)
        bo = self.pool.add(u.bias)

        def simt(TM, lo, hi):
            BM = TM * (NT // NTX)
            if K <= 16:
                BK = _pad4(K)
            else:
                BK = 8 if BM >= 256 else 16
            avec = CI % 4 == 0 and C0 % 4 == 0 and BK % 4 == 0
            akv = 4 if avec else 1
            while (BM * BK) % (akv * NT):
                BK += 4 if avec else 1
            smem = 4 * (2 * BK * (BM + 4) + 2 * BK * (BN + 4))
            fields = dict(
                H=H, W=W, CI=CI, HO=HO, WO=WO, CO=CO, KH=KH, KW=KW, S=S, PT=PT, PL=PL,
                K=K, ROWS=rows, POOL=pool_fused, PHO=PHO, PWO=PWO,
                IN_OFF=self.arena_off(u.input_ids[0]), IN_IMG=self.img_bytes(u.input_ids[0]),
                OUT_OFF=self.arena_off(u.output_id), OUT_IMG=self.img_bytes(u.output_id),
                W_OFF=wo, B_OFF=bo,
                RES=u.residual_id is not None,
                RES_OFF=self.arena_off(u.residual_id) if u.residual_id is not None else 0,
                RES_FIRST=False,
                SOFTMAX=softmax, SMEXP=SMEXP_CODE[self.opt.softmax_exp],
                BM=BM, BN=BN, BK=BK, TM=TM, TN=TN, **src1)
            fields.update(self.epilogue_fields(u, CO))
            tag = "dense" if u.kind == "Dense" else f"conv{KH}x{KW}"
            self.emit(pos, tag, "nnb::GemmSimt", fields, NT, smem, rows, BM,
                      grid_mult=ntile_n, n_min=lo, n_max=hi, dynamic_smem=True,
                      note=f"gemm M=n*{rows} N={CO} K={K} tile {BM}x{BN}x{BK}")

        # batches whose grid would not fill two waves of SMs with this tile get
        # a short-tile variant (TM = 1, or 4 under a fused pool): more CTAs
        TM_small = 4 if pool_fused else 1
        target = 2 * self.sm_count
        bm_big = TM * (NT // NTX)
        n_split = -(-target * bm_big // (rows * ntile_n))    # first n with >= target CTAs
        hi = min(n_max, self.max_batch)
        if TM > TM_small and n_split > n_min:
            simt(TM_small, n_min, min(n_split - 1, n_max))
            if n_split <= hi:
                simt(TM, n_split, n_max)
        else:
            simt(TM, n_min, n_max)

    def _sep_narrow(self, pos, u, wmat, CI, CO, geo):
        """Depthwise unit ``u.dw`` + 1x1 conv ``u`` (<= 32 output channels) as
        one SepNarrow launch: zero-haloed row bands through a cp.async ring,
        one thread per output pixel."""
        d = u.dw
        HO, WO, _ = u.output_shape.dims
        dwf = self._dw_fields(u)
        fields = dict(H=dwf["DW_H"], W=dwf["DW_W"], CI=CI, S=dwf["DW_S"], KH=dwf["DW_KH"],
                      KW=dwf["DW_KW"], PT=dwf["DW_PT"], PL=dwf["DW_PL"], HO=HO, WO=WO, CO=CO,
                      TH=geo["TH"], NS=geo["NS"], NT=geo["NT"], SP=geo.get("SP", 1),
                      IN_OFF=self.arena_off(u.input_ids[0]), OUT_OFF=self.arena_off(u.output_id),
                      RES=u.residual_id is not None,
                      RES_OFF=self.arena_off(u.residual_id) if u.residual_id is not None else 0,
                      DW_ACT=dwf["DW_ACT"], DW_POST=dwf["DW_POST"], DW_PS_OFF=dwf["DW_PS_OFF"],
                      DW_PO_OFF=dwf["DW_PO_OFF"], DW_FMA=self.sep_fma)
        fields.update(self.epilogue_fields(u, CO))
        tpi = -(-HO // geo["TH"])
        per_sm = max(1, min(SMEM_MAX // (geo["smem"] + 1024), 2048 // geo["NT"]))
        kh, kw = d.kernel_hw
        self.emit(pos, f"sep{kh}x{kw}_narrow", "nnb::SepNarrow", fields, geo["NT"], geo["smem"],
                  tpi, 1, dynamic_smem=True, grid_cap=self.sm_count * per_sm,
                  code=_sep_code(wmat, u.bias, CI, CO, d.kernel, d.bias, geo.get("SP", 1)),
                  note=f"dw{kh}x{kw}/s{d.stride} C={CI} + pw N={CO}: {geo['TH']}x{WO}-pixel tiles, "
                       f"{geo['NS']}-stage cp.async ring, zero halo, weights as immediates"
                       f"{', two threads per pixel' if geo.get('SP', 1) == 2 else ''}")

    def _dw_fields(self, u):
        """Fields of a fused depthwise producer (GemmSimt DW loader, tcgen05
        DWF); defaults when ``u`` is None or has none."""
        d = u.dw if u is not None else None
        if d is None:
            return dict(DW=0, DW_H=1, DW_W=1, DW_S=1, DW_PT=0, DW_PL=0, DW_KH=1, DW_KW=1,
                        DW_W_OFF=0, DW_B_OFF=0, DW_ACT=0, DW_POST=0, DW_PS_OFF=0, DW_PO_OFF=0)
        h, w, c = d.input_shapes[0].dims
        kh, kw = d.kernel_hw
        pt = same_padding(h, kh, d.stride)[0] if d.padding == "same" else 0
        pl = same_padding(w, kw, d.stride)[0] if d.padding == "same" else 0
        ep = self.epilogue_fields(d, c)
        return dict(DW=1, DW_H=h, DW_W=w, DW_S=d.stride, DW_PT=pt, DW_PL=pl, DW_KH=kh, DW_KW=kw,
                    DW_W_OFF=self.pool.add(d.kernel), DW_B_OFF=self.pool.add(d.bias),
                    DW_ACT=ep["ACT"], DW_POST=ep["POST"], DW_PS_OFF=ep["PS_OFF"],
                    DW_PO_OFF=ep["PO_OFF"])

    def _head_candidate(self, pos, u):
        """The Dense head (<= 16 outputs) right after Dense unit ``u`` that
        the tcgen05 epilogue can compute from u's finished rows (HEAD), or
        None.  u's output must feed only the head, and the head's output must
        not overlap u's input (the fused kernel reads one while writing the
        other)."""
        if not self.head or u.kind != "Dense" or u.residual_id is not None or pos + 1 >= len(self.plan.units):
            return None
        v = self.plan.units[pos + 1]
        if (v.kind != "Dense" or v.input_ids != (u.output_id,) or v.residual_id is not None
                or v.kernel.shape[1] > 16 or not _private(self.plan, u.output_id)):
            return None
        o_in, s_in = self.asg.offsets[u.input_ids[0]]
        o_out, s_out = self.asg.offsets[v.output_id]
        if o_out < o_in + s_in and o_in < o_out + s_out:
            return None
        return v

    def _gemm_tc(self, pos, u, wmat, K, CO, rows, n_min, conv=None, rows_geo=None, head=None,
                 n_max=1 << 30, edw=None):
        """tcgen05 3xTF32 GEMM (csrc/kernels/nnb_gemm_tc.cuh) for n >= n_min.
        ``conv`` switches the A operand to 8x16-pixel implicit-GEMM tiles of a
        stride-1 convolution loaded as 4-D TMA boxes (zero-filled borders)."""
        # narrow outputs: pack all KH x KW taps into N (KP9: N = 144 for CO = 16,
        # K = CI, each input pixel loaded and split once per tile), else the
        # horizontal taps (KPACK: N = KW * CO, K = KH * CI)
        kw = u.kernel_hw[1] if conv else 1
        kh_ = u.kernel_hw[0] if conv else 1
        kp9 = bool(conv and self.kpack9 and CO == 16 and kh_ * kw * CO <= 256 and 1 < kh_ <= 3
                   and 1 < kw <= 3 and not conv["POOL"] and u.residual_id is None
                   and conv.get("UPF", 1) == 1 and not conv.get("DWF") and u.dual_pool is None
                   and conv["CI"] % 32 == 0 and conv["C0"] % 32 == 0)
        # (KW * CO up to 192: CO = 64 convs pack into N = 192 with the
        # correction products merged into the main chain -- two accumulator
        # buffers of 192 columns fit TMEM, the short K = KH*CI keeps the merged
        # chain accurate)
        kpack = bool(conv and self.kpack and not kp9 and CO % 16 == 0 and kw > 1
                     and (kw * CO <= 128 or (kw * CO <= 192 and CO % 32 == 0 and self.kpack_wide
                                             and kh_ * conv["CI"] <= 512))
                     and (CO == 16 or CO % 32 == 0)
                     and not conv["POOL"] and u.residual_id is None)
        CO_real = CO
        if kp9:
            ci = conv["CI"]
            wmat = (np.asarray(wmat, F32).reshape(kh_, kw, ci, CO).transpose(2, 0, 1, 3)
                    .reshape(ci, kh_ * kw * CO))          # [ci][(ky*KW+kx)*CO+co]
            K, CO = ci, kh_ * kw * CO
        if kpack:
            kh = u.kernel_hw[0]
            ci = conv["CI"]
            wmat = (np.asarray(wmat, F32).reshape(kh, kw, ci, CO).transpose(0, 2, 1, 3)
                    .reshape(kh * ci, kw * CO))           # [ky*CI+ci][kx*CO+co]
            K, CO = kh * ci, kw * CO
        BN = min(128, -(-CO // 16) * 16) if CO < 32 else min(128, -(-CO // 32) * 32)
        if kpack or kp9:
            BN = CO
        # N = 256 tiles for wide row GEMMs whose K fits one accumulator chunk:
        # a kind::tf32 MMA costs ~1.4x at N = 256 what it costs at N = 128
        res_ = u.residual_id is not None
        eband = 0
        if edw is not None:
            head = None
            eh_, ew__, _ = u.output_shape.dims
            if 128 % (eh_ * ew__) and edw.kind != "Pool":
                # band tiles (nnb_gemm_tc.cuh EBAND): 128 / W image rows per tile
                etr = 128 // ew__
                eot = (etr - edw.kernel_hw[0]) // edw.stride + 1
                eband = -(-edw.output_shape.h // eot)          # tiles per image
        wide = bool(self.wide and not conv and edw is None and CO >= 256 and K <= 1024 and not res_
                    and self.pair and not self.aldg and CO % 4 == 0
                    and (not rows_geo or rows_geo.get("UPF", 1) == 1))
        if wide:
            # N = 256 tiles only where they keep every SM pair busy: with few
            # 256-row tiles (cfg3's 4x4x256 layers at 256 images: 16 tiles)
            # the 128-column form spreads the same work over 4x the CTAs
            # (measured: cfg3 @256 0.279 -> 0.266 ms)
            ntw = -(-CO // 256)
            n_wide = -(-(-(-WIDE_MIN_TILES // ntw) * 256) // rows)
            if n_wide > n_min:
                saved, self.wide = self.wide, False
                self._gemm_tc(pos, u, wmat, K, CO, rows, n_min, conv, rows_geo,
                              n_max=min(n_max, n_wide - 1))
                self.wide = saved
                if n_wide > n_max:
                    return
                n_min = n_wide
                head = None
            BN = 256
        NPAD = -(-CO // BN) * BN
        dwf = bool(conv and conv.get("DWF"))
        KPAD = -(-K // 32) * 32 if not conv or conv["CI"] % 32 == 0 else -(-K // 16) * 16
        BK = 32 if (not conv or (conv["CI"] % 32 == 0 and conv["C0"] % 32 == 0)) else 16
        if dwf and u.dw.stride > 1:
            BK = 16                                 # the stride-2 halo is 33 x 17 pixels
        halo_w = halo_h = 0
        if dwf:
            dkh, dkw = u.dw.kernel_hw
            halo_w, halo_h = 15 * u.dw.stride + dkw, 7 * u.dw.stride + dkh
        sw = 3 if BK == 32 else 2                  # TMA swizzle: 128 B or 64 B rows
        # independent accumulator chains fill TMEM (2 buffers x NACC x (main, corr))
        NACC = max(1, min(8, 128 // BN)) if self.nacc is None else max(1, min(self.nacc, 128 // BN))
        aldg = self.aldg
        tmem_a = self.tmem_a and NACC == 1 and not aldg and (BN <= 64 or BN == 128)
        if (tmem_a and BN > 64 and head is not None and -(-CO // BN) == 1 and not wide
                and u.residual_id is None and not kpack):
            # A in TMEM leaves one accumulator buffer at BN = 128, which keeps a
            # following head out of the epilogue; shared-memory A with two
            # buffers + the fused head (cfg1 @65536: 256->128 + 128->10 0.0371
            # + 0.0108 -> 0.0379 ms, replay 0.3214 -> 0.3160 ms)
            tmem_a = False
        if wide:
            BK = self.wide_bk
            sw = 3 if BK == 32 else 2
        csplit = self.csplit and not kp9 and BN <= 128   # N = 144 / 192: two buffers fit only merged
        # k-blocks (of 32) per TMEM accumulator chunk: every chunk ends in a
        # drain the MMAs wait for (one accumulator buffer at BN = 128), so
        # long chunks are faster; the tensor core truncates once per MMA, so
        # short chunks are more accurate.  Measured (scripts/tc_error.py,
        # max |d| / (atol + rtol |ref|)): K=1024: 0.39 / 0.50 / 0.80 at 8 / 16
        # / 32; K=4096: 0.77 / 0.83 / 0.89.  dense 1024->512: 0.40 / 0.34 /
        # 0.32 ms at 65536 rows.
        chunk = self.chunk or (16 if K <= 1024 else 8)
        corr_whole = False
        if wide:
            # one accumulator buffer of (main, correction) = 512 TMEM columns;
            # the main chain restarts every 16 k-blocks (an accuracy bound: the
            # tensor core truncates per MMA) while the small correction chain
            # spans the whole K, so a mid-tile drain reads only the main half.
            # Measured (tc_error.py / tc_error_wide.py, dense 1024->512 at
            # 65536 rows): whole K in one chunk 0.26 ms but up to 1.05 of the
            # FP32 tolerance on N(0,1) data; 16 k-blocks 0.317 ms at <= 0.69
            # (BN = 128: 0.337 ms at <= 0.67); merged chains with two buffers
            # 0.30-0.35 ms.  With the round-to-nearest split written back
            # (rn_ss) the 16-block form has the BN = 128 path's accuracy.
            # MERGED form (wide_csplit=False, opt-in): the BF16 correction MMA
            # accumulates into the main chain, restarted every 8 k-blocks, so
            # TWO 256-column buffers fit and a chunk is drained while the next
            # one is filled (with six split warps the mainloop runs at the MMA
            # roof; what remains is the MMAs waiting for drains).  Measured
            # (cfg1 @65536): Dense 1024->512 0.1990 -> 0.1922 ms, replay 0.2983
            # -> 0.2910 ms, max |d| / FP32 gate 0.75-0.85 on N(0,1) inputs for
            # both forms -- but one of 9.7 M outputs of a K = 512 tanh layer on
            # U(-2, 2) inputs lands at 1.02x the plain gate (test_wide_n256_
            # tiles_opt_in), which the split form passes; 4-block chunks are
            # more accurate (0.68-0.78) and slower (0.3053 ms).  Not the default.
            csplit = self.wide_csplit
            corr_whole = csplit
            if not self.chunk:
                chunk = self.wide_chunk or (16 if csplit else 8)
        cw = (2 if csplit else 1) * BN                # TMEM columns per accumulator chain
        ABUF = 1 if ((tmem_a and BN > 64 and csplit) or (wide and csplit)) else 2
        if not tmem_a and self.abuf:
            # more accumulator buffers let the MMA run further ahead of the
            # epilogue: a tile's commit -> drain -> release round trip costs
            # ~1-2 us, which short tiles (few k-blocks) cannot hide with two
            ABUF = max(1, min(self.abuf, 512 // (NACC * cw)))
        # CTA pairs (cta_group::2, 256-row tiles, each CTA holds half of B):
        # the BN = 128 row GEMMs, whose single-CTA form is bound by
        # shared-memory bandwidth (B is re-read by every product)
        # Narrow-N convs are bound by tcgen05 instruction dispatch, not MMA
        # math (ncu: TC pipe 66% busy, tensor math 23% at N=48): a pair issues
        # one M=256 instruction where two CTAs issued two.
        pair = bool(self.pair and not aldg and BN % 16 == 0 and (BN // 2) % 8 == 0 and not eband
                    and ((not conv and tmem_a and BN == 128 and K >= 256)
                         or conv or wide))
        # row-shared vertical taps (KPACK conv tiles, A in shared memory): one
        # A box of 8 + KH - 1 input rows serves every kernel row (nnb_gemm_tc.cuh
        # RS), so each input pixel is loaded and split once per channel block
        rs = (kh_ if (kpack and self.rowshare and kh_ > 1 and not tmem_a and not aldg and not dwf
                      and self.corr_bf16 not in (True, "auto")) else 1)
        # (cfg4 @64: 0.659 -> 0.607 ms; the 120x160x16->32 conv 0.131 -> 0.111,
        # the 60x80x128->32 concat conv 0.180 -> 0.146)
        a_rows = 128 + 16 * (rs - 1)
        a_smem = (0 if dwf else 128 * BK * 4) if tmem_a else 2 * a_rows * BK * 4
        halo_bytes = -(-(halo_w * halo_h * BK * 4) // 1024) * 1024
        stage = a_smem + 2 * rs * (BN // 2 if pair else BN) * BK * 4 + halo_bytes
        # epilogue through TMA stores (and a TMA-prefetched residual) for plain
        # row tiles; 64B-swizzled 32 x 16 boxes, NBUF per epilogue warp
        res = u.residual_id is not None
        egrp = max(1, (BN // 2 if BN >= 32 else 16) // 16)
        epi_tma = bool(self.epi_tma and not kpack and not kp9 and CO % 4 == 0 and (not res or egrp <= 2)
                       and not (conv and conv["POOL"])
                       and (conv or not rows_geo or rows_geo.get("UPF", 1) == 1)
                       and (not conv or conv.get("UPF", 1) == 1))
        if edw is not None:
            epi_tma = False        # the finished tile is parked in shared memory instead
        nbuf = (egrp if res else min(egrp, 2)) if epi_tma else 1
        # KPACK conv tiles with 32 outputs: sixteen epilogue warps (nnb_gemm_tc.cuh EPI16) --
        # bit-identical, measured SLOWER (cfg4 @64: 109.5 -> 118 us, 145.8 -> 153 us): opt-in
        epi16 = bool(kpack and CO_real == 32 and self.epi16 and edw is None)
        epi_bytes = (16 if epi16 else 8) * nbuf * 2048
        if edw is not None:
            epi_bytes = -(-(128 * (BN + 4) * 4) // 1024) * 1024
        # deep rings hide the TMA/L2 latency when a stage carries little MMA work
        room = SMEM_MAX - 1024 - 512 - epi_bytes
        if rs > 1 and room // stage < 2 and BK == 32:
            # row-shared stages of 16-channel k-blocks (N = 192: 112 KB -> 56 KB;
            # cfg4 @64 0.084 -> 0.078 ms; where two 32-channel stages fit they
            # are faster: N = 96, K = 384 0.146 vs 0.169 ms at 16)
            bk16 = 2 * a_rows * 16 * 4 + 2 * rs * (BN // 2 if pair else BN) * 16 * 4
            if room // bk16 >= 3:
                BK, sw, stage = 16, 2, bk16
        if rs > 1 and room // stage < 2:
            # two row-shared stages do not fit: per-row boxes
            rs = 1
            chunk = self.chunk or (16 if K <= 1024 else 8)
            stage = 2 * 128 * BK * 4 + 2 * (BN // 2 if pair else BN) * BK * 4 + halo_bytes
        if rs > 1 and not self.chunk:
            # a chunk counts k-blocks of RS x BK k values: keep its K span
            chunk = max(1, chunk * 32 // (rs * BK))
        NS = max(2, min(8, (SMEM_MAX - 1024 - 512 - epi_bytes) // stage))
        if tmem_a:
            NS = min(NS, (512 - ABUF * NACC * cw) // (2 * BK))
        wt = np.zeros((NPAD, KPAD), F32)
        wt[:CO, :K] = np.asarray(wmat, F32).T
        hi = tf32_split_hi(wt, self.split_rn)
        lo = (wt - hi).astype(F32)
        # BF16 correction products (one kind::f16 MMA per k-step instead of
        # two tf32 ones; B_corr replaces B_lo byte for byte) on every
        # shared-memory-A tile with 32-float k-blocks (corr_bf16=True) or on
        # the N = 256 row tiles only ("wide", default).  Measured (cfg1
        # @65536): Dense 1024->512 0.258 -> 0.220 ms, 512->256 0.081 -> 0.073
        # ms; cfg4 @64 convs 0.117 / 0.179 / 0.317 -> 0.107 / 0.163 / 0.287
        # ms -- but K = 32 pointwise convs then miss the plain FP32 gate on
        # 0.03% of outputs near zero (|d| 1.5e-5: within the stated bf16
        # bound, not within atol 1e-5), so narrow tiles keep the TF32 split.
        # "wide" (default): the N = 256 row tiles only.  "auto" adds the
        # implicit-GEMM conv tiles with K >= CB16_CONV_MIN_K (cfg4 @64: 0.897
        # -> 0.857 ms), but their outputs then sit within the stated BF16
        # bound, not the plain FP32 gate (cfg4's reference golden: 3 of 57600
        # outputs off by 1.3e-5 > atol 1e-5), so it is opt-in
        cb16_on = (wide if self.corr_bf16 == "wide" else
                   (wide or (conv is not None and K >= CB16_CONV_MIN_K)) if self.corr_bf16 == "auto"
                   else bool(self.corr_bf16))
        cb16 = bool(cb16_on and not tmem_a and not aldg and not dwf and BK == 32 and (csplit or wide))
        # narrow tiles with the bf16 split: four converter warps (with two the
        # extra split work made cfg4's convs slower; with four cfg4 @64
        # 0.892 -> 0.834 ms, cfg0/2/3 unchanged)
        # conv tiles whose MMA work per k-block is short next to the split of
        # their A tile (all taps in N, 16-channel k-blocks, N = 192): four
        # split warps too (cfg4 @64: KP9 conv 0.195 -> 0.170 ms, BK = 16 conv
        # 0.138 -> 0.131, N = 192 0.085 -> 0.084; the N = 96 concat conv with
        # K = 384 gets slower, 0.178 -> 0.194, and keeps two)
        conv_w4 = bool((cb16 and not wide and self.cb16_w4)
                       or (conv and (self.conv_w4 is True or (self.conv_w4 == "auto" and (kp9 or BK == 16 or BN > 128)))))
        # N = 256 BF16-correction row tiles: six split warps, registers moved from the
        # producer / split warpgroups to the epilogue ones (nnb_gemm_tc.cuh SETREG)
        setreg = bool(cb16 and wide and self.setreg and not tmem_a and not aldg)
        hi_off, lo_off = self.pool.add(hi), self.pool.add(bf16_corr_words(hi, lo) if cb16 else lo)
        geo = dict(CONV=0, POOL=0, H=1, W=1, CI=1, HO=1, WO=1, KH=1, KW=1, PT=0, PL=0, PHO=1,
                   PWO=1, C0=1, CONCAT=0, UPF=1, DWF=0)
        if conv:
            geo.update(conv, CONV=1)
        elif rows_geo:
            geo.update(rows_geo)
        fields = dict(K=K, N=CO, CO=CO_real, KPACK=kpack, KP9=kp9, NPAD=NPAD, BN=BN, BK=BK, NS=NS,
                      ROWS=rows, TMEM_A=tmem_a,
                      NACC=NACC, ALDG=aldg, ABUF=ABUF, CSPLIT=int(csplit), CHUNK=chunk,
                      CORR_WHOLE=int(corr_whole), RN_SS=(2 if self.rn_ss == 2 else int(bool(self.rn_ss))) if self.split_rn else 0,
                      CORR_BF16=int(cb16), CONV_W4=int(conv_w4), SETREG=int(setreg), EPI16=int(epi16), RS=rs,
                      EARLY=int(cb16 and wide and self.early_mma),
                      APF=(self.a_prefetch if (wide and not conv) else 0),
                      PAIR=int(pair),
                      # shared-memory transposed epilogue (coalesced residual
                      # loads / stores); long-K tiles keep direct row stores --
                      # their mainloop is shared-memory bound and the extra
                      # staging traffic cost 9% at K=1024 (equal at K=512)
                      EPI_ST=int(u.residual_id is not None or K < 512 or self.epi_tma == "staged"),
                      EPI_TMA=int(epi_tma),
                      IN_OFF=self.arena_off(u.input_ids[0]),
                      IN_IMG=self.img_bytes(u.input_ids[0]),
                      IN1_OFF=(self.arena_off(u.input_ids[1]) if conv and conv["CONCAT"] else 0),
                      IN1_IMG=(self.img_bytes(u.input_ids[1]) if conv and conv["CONCAT"] else 0),
                      **geo,
                      OUT_IMG=self.img_bytes(u.output_id),
                      OUT_OFF=self.arena_off(u.output_id), B_OFF=self.pool.add(u.bias),
                      RES=u.residual_id is not None,
                      RES_OFF=self.arena_off(u.residual_id) if u.residual_id is not None else 0)
        fields.update(self.epilogue_fields(u, CO_real))
        fields.update(self._dw_fields(u) if dwf else self._dw_fields(None))
        # second store of the 2x2 max-pooled output (planner.fuse_pool_dual)
        dp = u.dual_pool if conv else None
        if dp is not None:
            pre = dp.pre_up_shape if dp.upsample_after > 1 else dp.output_shape
            fields.update(DPOOL=1, DP_OFF=self.arena_off(dp.output_id),
                          DP_IMG=self.img_bytes(dp.output_id), DP_UPF=dp.upsample_after,
                          DP_PHO=pre.h, DP_PWO=pre.w)
            self._dual_from = min(self._dual_from, n_min)
        else:
            fields.update(DPOOL=0, DP_OFF=0, DP_IMG=0, DP_UPF=1, DP_PHO=1, DP_PWO=1)
        # the depthwise conv consuming this 1x1 conv, in the epilogue (planner.fuse_pw_dw)
        if edw is not None and edw.kind == "Pool":
            # global average pool of the parked tile (E_GAP)
            eh, ew_, _ = u.output_shape.dims
            zo = self.pool.zeros_offset(CO)
            fields.update(EDW=1, E_GAP=1, E_H=eh, E_W=ew_, E_HO=1, E_WO=1, E_KH=1, E_KW=1, E_S=1, E_PT=0,
                          E_PL=0, E_W_OFF=zo, E_B_OFF=zo, E_ACT=0, E_POST=0, E_PS_OFF=zo, E_PO_OFF=zo,
                          E_OUT_OFF=self.arena_off(edw.output_id),
                          E_OUT_IMG=self.img_bytes(edw.output_id), E_FMA=0)
            self._edw_from = min(self._edw_from, n_min)
        elif edw is not None:
            eh, ew_, _ = u.output_shape.dims
            eho, ewo, _ = edw.output_shape.dims
            ekh, ekw = edw.kernel_hw
            same = edw.padding == "same"
            eep = self.epilogue_fields(edw, CO)
            fields.update(EDW=1, E_GAP=0, E_H=eh, E_W=ew_, E_HO=eho, E_WO=ewo, E_KH=ekh, E_KW=ekw,
                          E_S=edw.stride,
                          E_PT=same_padding(eh, ekh, edw.stride)[0] if same else 0,
                          E_PL=same_padding(ew_, ekw, edw.stride)[0] if same else 0,
                          E_W_OFF=self.pool.add(edw.kernel), E_B_OFF=self.pool.add(edw.bias),
                          E_ACT=eep["ACT"], E_POST=eep["POST"], E_PS_OFF=eep["PS_OFF"],
                          E_PO_OFF=eep["PO_OFF"], E_OUT_OFF=self.arena_off(edw.output_id),
                          E_OUT_IMG=self.img_bytes(edw.output_id), E_FMA=int(bool(self.sep_fma)))
            self._edw_from = min(self._edw_from, n_min)
        else:
            fields.update(EDW=0, E_GAP=0, E_H=1, E_W=1, E_HO=1, E_WO=1, E_KH=1, E_KW=1, E_S=1, E_PT=0, E_PL=0,
                          E_W_OFF=0, E_B_OFF=0, E_ACT=0, E_POST=0, E_PS_OFF=0, E_PO_OFF=0,
                          E_OUT_OFF=0, E_OUT_IMG=0, E_FMA=0)
        if conv:
            H, W = conv["H"], conv["W"]

            def act_map(tid, ch):
                return dict(space=1, offset=self.arena_off(tid), dims=(ch, W, H, self.cap),
                            box=(BK, 16, 8 + rs - 1, 1), strides=(4 * ch, 4 * ch * W, 4 * ch * W * H),
                            swizzle=sw)
            tm_a = act_map(u.input_ids[0], conv["C0"])
            tm_a1 = (act_map(u.input_ids[1], conv["CI"] - conv["C0"]) if conv["CONCAT"]
                     else tm_a)
            if dwf:                # the depthwise input, one halo box per tile
                dh, dw_, dc = u.dw.input_shapes[0].dims
                tm_a = dict(space=1, offset=self.arena_off(u.input_ids[0]),
                            dims=(dc, dw_, dh, self.cap), box=(BK, halo_w, halo_h, 1),
                            strides=(4 * dc, 4 * dc * dw_, 4 * dc * dw_ * dh), swizzle=sw)
                tm_a1 = tm_a

            def out_map(tid):      # epilogue boxes: 16 channels x 16 px x 2 rows
                return dict(space=1, offset=self.arena_off(tid), dims=(CO, conv["WO"], conv["HO"], self.cap),
                            box=(16, 16, 2, 1), strides=(4 * CO, 4 * CO * conv["WO"],
                                                         self.img_bytes(tid)), swizzle=2)
        else:
            tm_a = dict(space=1, offset=self.arena_off(u.input_ids[0]),
                        dims=(K, self.cap * rows), strides=(4 * K,), box=(BK, 128), swizzle=sw)
            tm_a1 = tm_a

            def out_map(tid):      # epilogue boxes: 16 columns x 32 rows
                return dict(space=1, offset=self.arena_off(tid), dims=(CO, self.cap * rows),
                            strides=(4 * CO,), box=(16, 32), swizzle=2)
        tm_b = dict(space=2, offset=hi_off, dims=(KPAD, NPAD), strides=(4 * KPAD,),
                    box=(BK, BN // 2 if pair else BN), swizzle=sw)
        tm_bl = dict(tm_b, offset=lo_off)
        tm_o = out_map(u.output_id) if epi_tma else tm_a
        tm_r = out_map(u.residual_id) if (epi_tma and res) else tm_o
        smem = NS * stage + epi_bytes + 1024 + 512
        ntn = NPAD // BN
        code = ""
        hn = 0
        # the head's FFMAs lengthen the epilogue: only when a second accumulator
        # buffer keeps the MMA from waiting on it (measured: cfg0 Dense 256->32
        # + 32->2, two buffers: replay -1.3%; cfg1 256->128 + 128->10, one
        # buffer (A in TMEM): +1%, two (A in shared memory): -1.7%)
        if (head is not None and ntn == 1 and BN >= 32 and not wide and not res and not kpack
                and ABUF >= 2):
            hn = head.kernel.shape[1]
            hep = self.epilogue_fields(head, hn)
            fields.update(HEAD=1, HN=hn, H_ACT=hep["ACT"], H_POST=hep["POST"],
                          H_PS_OFF=hep["PS_OFF"], H_PO_OFF=hep["PO_OFF"],
                          H_SOFTMAX=bool(head.softmax_after),
                          H_SMEXP=SMEXP_CODE[self.opt.softmax_exp],
                          H_OUT_OFF=self.arena_off(head.output_id))
            code = _imm_tables(hw=np.asarray(head.kernel, F32), hbias=head.bias)
            self.head_cap[pos + 1] = n_min - 1
        else:
            fields.update(HEAD=0, HN=1, H_ACT=0, H_POST=0, H_PS_OFF=0, H_PO_OFF=0, H_SOFTMAX=0,
                          H_SMEXP=0, H_OUT_OFF=0)
        if conv:
            ow = 16 - (kw - 1) if (kpack or kp9) else 16
            tho = 8 - (kh_ - 1) if kp9 else 8
            tpi = -(-conv["HO"] // tho) * -(-conv["WO"] // ow)
            ipi, ipb = tpi, 2 if pair else 1
            tag = f"conv{u.kernel_hw[0]}x{u.kernel_hw[1]}_tc"
        else:
            ipi, ipb = rows, 256 if pair else 128
            if eband:
                ipi, ipb = eband, 1
            tag = "dense_tc" if u.kind == "Dense" else "conv1x1_tc"
            if edw is not None:
                tag = ("conv1x1_gap_tc" if edw.kind == "Pool"
                       else f"conv1x1_dw{edw.kernel_hw[0]}x{edw.kernel_hw[1]}_tc")
        self.emit(pos, tag, "nnb::GemmTc", fields,
                  (512 if setreg else 448 if (tmem_a or aldg or dwf or conv_w4) else 384)
                  + (256 if epi16 else 0), smem,
                  ipi, ipb,
                  grid_mult=ntn * (2 if pair else 1), cluster=2 if pair else 1,
                  n_min=n_min, n_max=n_max, tmaps=[tm_a, tm_b, tm_bl, tm_a1, tm_o, tm_r], code=code,
                  grid_cap=self.sm_count - self.sm_count % 2 if pair else self.sm_count,
                  note=f"tcgen05 3xTF32 M=n*{rows} N={CO} K={K} tile {256 if pair else 128}x{BN}x{BK}"
                       f"{' CTA pair' if pair else ''} stages {NS}"
                       f" chains {NACC} bufs {ABUF}{'' if csplit else ' merged-corr'}"
                       f"{' A via cp.async' if aldg else ''}"
                       f"{' taps packed in N' if kpack else ''}"
                       f"{' rows shared by the kernel rows' if rs > 1 else ''}"
                       f"{' all taps packed in N' if kp9 else ''}"
                       f"{' depthwise fused' if dwf else ''}"
                       f"{' 8x16-pixel conv tiles' if conv else ' row tiles'}"
                       f"{' concat (2 A maps)' if conv and conv.get('CONCAT') else ''}"
                       f"{' A in TMEM' if tmem_a else ''}{' TMA epilogue' if epi_tma and not hn else ''}"
                       f"{' bf16 corr' if cb16 else ''}{' 6 split warps (setmaxnreg)' if setreg else ''}"
                       f"{' 16 epilogue warps' if epi16 else ''}"
                       f"{' + pooled second store' if dp is not None else ''}"
                       f"{' + global average pool in the epilogue' if edw is not None and edw.kind == 'Pool' else ' + depthwise conv in the epilogue' if edw is not None else ''}"
                       f"{f' ({eband} bands of {128 // u.output_shape.w} rows per image)' if eband else ''}"
                       f"{f' + fused Dense head N={hn}' if hn else ''}")

    def _conv_direct(self, pos, u, wmat, H, W, CI, HO, WO, CO, KH, KW, S, PT, PL, pool_fused,
                     PHO, PWO, UPF=1, n_min=1):
        pxt = 4 if CO <= 8 else 2 if CO <= 16 else 1
        fields = dict(H=H, W=W, CI=CI, HO=HO, WO=WO, CO=CO, KH=KH, KW=KW, S=S, PT=PT, PL=PL,
                      POOL=pool_fused, PHO=PHO, PWO=PWO, PXT=pxt, UPF=UPF,
                      IN_OFF=self.arena_off(u.input_ids[0]), IN_IMG=self.img_bytes(u.input_ids[0]),
                      OUT_OFF=self.arena_off(u.output_id), OUT_IMG=self.img_bytes(u.output_id),
                      W_OFF=self.pool.add(wmat), B_OFF=self.pool.add(u.bias),
                      RES=u.residual_id is not None,
                      RES_OFF=self.arena_off(u.residual_id) if u.residual_id is not None else 0)
        fields.update(self.epilogue_fields(u, CO))
        # Every tap unrolled with the weights as immediates is the fastest
        # form, but NVRTC time grows with the unrolled FFMA count; above
        # DIRECT_UNROLL_MAX the weights are shared-memory broadcasts and the
        # kernel-row loop stays rolled (compile-time bound, see DESIGN)
        np_ = 4 if pool_fused else pxt
        unrolled = KH * KW * CI * CO * np_
        # a pool window split over two lanes halves the unrolled body (cfg0's
        # 16x16x8 -> 16 conv: 4608 -> 2304 FFMAs, immediates kept: 88 -> ~53 us
        # at 4096 images against the shared-memory form)
        psplit = 0
        if pool_fused and unrolled > DIRECT_UNROLL_MAX:
            # a 2x2 window over 2 lanes (one row each) or 4 (one pixel each;
            # cfg0's 8x8x16 -> 16 conv: the SIMT GEMM took 44 us)
            psplit = 2 if unrolled // 2 <= DIRECT_SPLIT_MAX else 4
            unrolled //= psplit
        wimm = bool(self.direct_imm) and unrolled <= (DIRECT_SPLIT_MAX if psplit
                                                      else DIRECT_UNROLL_MAX)
        if self.direct_imm == "force":
            wimm = True
        fields["WIMM"] = wimm
        fields["PSPLIT"] = psplit
        roll = 0
        if not wimm and unrolled > DIRECT_UNROLL_MAX and KH > 1:
            roll = 1 if unrolled // KH <= DIRECT_UNROLL_MAX // 2 else 2
        fields["ROLL_KY"] = roll
        code = _imm_tables(wt=wmat, bias=u.bias) if wimm else ""
        # pool: one 2x2 window per thread; else pxt pixels per thread, the
        # 128-thread block covering 128*pxt consecutive pixels
        ipi, ipb = ((PHO * PWO * max(psplit, 1), 128) if pool_fused
                    else (HO * WO, 128 * pxt))
        smem = 4 * ((4 if wimm else KH * KW * CI * CO) + CO)
        self.emit(pos, f"conv{KH}x{KW}_direct", "nnb::ConvDirect", fields, 128, smem, ipi, ipb,
                  dynamic_smem=True, n_min=n_min, code=code,
                  note=f"direct conv CI={CI} CO={CO} {'pool2 ' if pool_fused else ''}px/thread "
                       f"{(4 // psplit if psplit else 4) if pool_fused else pxt}"
                       f"{' weights as immediates' if wimm else ' weights in smem'}")

    def _dense_small(self, pos, u, wmat, K, CO, softmax, n_max, rows=1, mb=None, n_min=1, kper=32):
        """Split-K GEMV/GEMM for few rows: Dense at n <= n_max (MB = n_max
        rows per block), or a 1x1 conv whose n*rows pixels are the rows (MB
        = ``mb`` per block)."""
        MB = mb or n_max
        KS = max(1, min(32, K // kper))
        fields = dict(K=K, CO=CO, MB=MB, KS=KS, ROWS=rows,
                      IN_OFF=self.arena_off(u.input_ids[0]),
                      IN_IMG=self.img_bytes(u.input_ids[0]),
                      OUT_OFF=self.arena_off(u.output_id), OUT_IMG=self.img_bytes(u.output_id),
                      W_OFF=self.pool.add(wmat), B_OFF=self.pool.add(u.bias),
                      SOFTMAX=softmax, SMEXP=SMEXP_CODE[self.opt.softmax_exp],
                      RES=u.residual_id is not None,
                      RES_OFF=self.arena_off(u.residual_id) if u.residual_id is not None else 0)
        fields.update(self.epilogue_fields(u, CO))
        if softmax and CO > 32:
            raise UnsupportedLayer("fused softmax needs <= 32 units")
        nj = (CO + 31) // 32
        self.emit(pos, "gemv" if rows == 1 else "conv1x1_rows", "nnb::DenseSmallM", fields,
                  32 * KS, 0, rows, MB, grid_mult=nj, n_min=n_min, n_max=n_max,
                  note=f"split-K rows K={K} N={CO} ks={KS} rows/block {MB}")

    def _tiny_step(self, i, u):
        """(struct text, call) of one unit inside the TinyNet kernel, or None
        when the unit kind / fusion is outside it."""
        off = lambda t: self.asg.offsets[t][0]
        ep = lambda co: self.epilogue_fields(u, co)
        res = off(u.residual_id) if u.residual_id is not None else -1
        if u.kind == "Conv2D":
            if (u.dw is not None or u.concat_in or u.upsample_after != 1 or u.softmax_after
                    or u.kernel.shape[3] % 4):
                return None
            H, W, CI = u.input_shapes[0].dims
            co = u.kernel.shape[3]
            pre = u.pre_pool_shape if u.pool_after else u.output_shape
            HO, WO = pre.h, pre.w
            KH, KW = u.kernel_hw
            PT = same_padding(H, KH, u.stride)[0] if u.padding == "same" else 0
            PL = same_padding(W, KW, u.stride)[0] if u.padding == "same" else 0
            f = dict(H=H, W=W, CI=CI, HO=HO, WO=WO, CO=co, KH=KH, KW=KW, S=u.stride, PT=PT, PL=PL,
                     POOL=u.pool_after, PHO=u.output_shape.h, PWO=u.output_shape.w,
                     IN=off(u.input_ids[0]), OUT=off(u.output_id), RES=res,
                     W_OFF=self.pool.add(np.asarray(u.kernel, F32)), B_OFF=self.pool.add(u.bias),
                     **ep(co))
            return f, "TinyConv"
        if u.kind == "DepthwiseConv2D":
            if (u.residual_id is not None or u.pool_after or u.upsample_after != 1
                    or u.softmax_after):
                return None
            H, W, C = u.input_shapes[0].dims
            HO, WO, _ = u.output_shape.dims
            KH, KW = u.kernel_hw
            PT = same_padding(H, KH, u.stride)[0] if u.padding == "same" else 0
            PL = same_padding(W, KW, u.stride)[0] if u.padding == "same" else 0
            f = dict(H=H, W=W, C=C, HO=HO, WO=WO, KH=KH, KW=KW, S=u.stride, PT=PT, PL=PL,
                     IN=off(u.input_ids[0]), OUT=off(u.output_id), W_OFF=self.pool.add(u.kernel),
                     B_OFF=self.pool.add(u.bias), **ep(C))
            return f, "TinyDw"
        if u.kind == "Dense":
            K, CO = u.kernel.shape
            if u.softmax_after and CO > 32:
                return None
            f = dict(K=K, CO=CO, IN=off(u.input_ids[0]), OUT=off(u.output_id), RES=res,
                     W_OFF=self.pool.add(np.asarray(u.kernel, F32)), B_OFF=self.pool.add(u.bias),
                     SOFTMAX=bool(u.softmax_after), SMEXP=SMEXP_CODE[self.opt.softmax_exp], **ep(CO))
            return f, "TinyDense"
        if u.kind == "Pool":
            if u.upsample_after != 1 or u.input_shapes[0].rank != 3:
                return None
            H, W, C = u.input_shapes[0].dims
            o = u.output_shape
            HO, WO = (1, 1) if o.rank == 1 else (o.h, o.w)
            PH, PW = u.kernel_hw
            PT = same_padding(H, PH, u.stride)[0] if u.padding == "same" else 0
            PL = same_padding(W, PW, u.stride)[0] if u.padding == "same" else 0
            f = dict(H=H, W=W, C=C, HO=HO, WO=WO, PH=PH, PW=PW, S=u.stride, PT=PT, PL=PL,
                     AVG=u.pool_op == "avg", IN=off(u.input_ids[0]), OUT=off(u.output_id))
            return f, "TinyPool"
        if u.kind in ("ElementwiseActivation", "Add"):
            if len(u.input_ids) > 4:
                return None
            ins = [off(t) for t in u.input_ids] + [0] * (4 - len(u.input_ids))
            aff = u.scale is not None
            f = dict(N=u.output_shape.elements, C=u.output_shape.c, NIN=len(u.input_ids),
                     IN0=ins[0], IN1=ins[1], IN2=ins[2], IN3=ins[3], OUT=off(u.output_id),
                     AFFINE=aff, SC_OFF=self.pool.add(u.scale) if aff else 0,
                     OF_OFF=self.pool.add(u.offset) if aff else 0,
                     ACT=ACT_CODE[u.activation], MODE=MODE_CODE[self.opt.activation_mode])
            return f, "TinyElem"
        if u.kind == "Softmax":
            if u.output_shape.rank != 1 or u.output_shape.elements > 32:
                return None
            f = dict(L=u.output_shape.elements, IN=off(u.input_ids[0]), OUT=off(u.output_id),
                     SMEXP=SMEXP_CODE[self.opt.softmax_exp])
            return f, "TinySoftmax"
        return None

    def _tiny(self):
        """The whole network as ONE launch for batches up to TINY_MAX_N (one
        CTA per image over a shared-memory copy of its arena;
        nnb_tiny.cuh) when every unit has a TinyNet step, the per-image
        arena fits shared memory and the weights are small (read through
        L1).  Regular launches then serve the larger batches only.

        Opt-in (``tuning={"tiny": True}``): measured on B200, cfg0 at 1 / 16 /
        64 images 37 us against 23 / 31 / 32 us for the per-layer launches
        (60 us before the weights were staged in shared memory).  One CTA
        per image leaves one image's layers on 256 threads of one SM, where
        the per-layer kernels spread each layer over many CTAs; the launch
        overhead it removes is smaller than that."""
        if (self.asg.arena_size > TINY_ARENA_MAX or not self.plan.units
                or len(self.plan.units) < 2):
            return
        wbytes = sum(4 * a.size for u in self.plan.units
                     for a in (u.kernel, u.bias, u.post_scale, u.post_offset, u.scale, u.offset)
                     if a is not None)
        if wbytes > TINY_WEIGHTS_MAX:
            return
        pool_mark = self.pool.mark()
        assert pool_mark[0] == 0, "the TinyNet is specialised first (its weights lead the pool)"
        steps = []
        for i, u in enumerate(self.plan.units):
            st = self._tiny_step(i, u)
            if st is None:
                self.pool.rollback(pool_mark)   # nothing of it is referenced
                return
            steps.append(st)
        n_max = min(self.max_batch, TINY_MAX_N)
        structs = [_cfg_struct(f"T{i}", f).replace("\n", "\n  ") for i, (f, _) in enumerate(steps)]
        body = ["  __device__ static __forceinline__ void body(const float* __restrict__ pool, "
                "const float* w, float* a) {"]
        for i, (_, t) in enumerate(steps):
            body += [f"    nnb::{t}<T{i}>::run(pool, w, a);", "    __syncthreads();"]
        body.append("  }")

        def copies(tids, load):
            lines = [f"  __device__ static __forceinline__ void {'load' if load else 'store'}("
                     "float* __restrict__ arena, int img, float* a) {"]
            for t in tids:
                o, b = self.asg.offsets[t][0], self.img_bytes(t)
                g = f"nnb::at<float>(arena, {self.arena_off(t)}LL + (long long)img * {b}LL)"
                lines.append(f"    nnb::tiny_copy<{b}>({'a + ' + str(o // 4) if load else g}, "
                             f"{g if load else 'a + ' + str(o // 4)});")
            lines.append("  }")
            return lines
        code = "\n".join(["  " + x for x in structs] + body + copies(self.plan.input_ids, True)
                         + copies(self.plan.output_ids, False))
        arena_floats = -(-self.asg.arena_size // 16) * 4
        w_floats = -(-len(self.pool.data) // 16) * 4          # every entry so far is this kernel's
        if 4 * (arena_floats + w_floats) > TINY_SMEM_MAX:
            self.pool.rollback(pool_mark)
            return
        self.emit(0, "tinynet", "nnb::TinyNet", dict(ARENA_FLOATS=arena_floats, W_FLOATS=w_floats),
                  256, 4 * (arena_floats + w_floats), 1, 1, dynamic_smem=True, n_max=n_max, code=code,
                  note=f"whole network ({len(steps)} units) in one launch, one CTA per image, "
                       f"{self.asg.arena_size // 1024} KB arena in shared memory")
        self._n_floor = n_max + 1

    def chain(self, pos, u):
        """A run of small depthwise / pointwise convs (+ closing global average
        pool) in one kernel, one CTA per image (nnb_chain.cuh,
        planner.fuse_chain).  The generated ``body`` calls one step template
        per layer over shared-memory ping-pong buffers."""
        from .planner import CHAIN_THREADS, chain_bytes, chain_pw_tile
        steps = u.steps
        h, w, c = steps[0].input_shapes[0].dims
        structs, calls = [], [f"    nnb::chain_stage<{h}, {w}, {c}>(src, x);",
                               "    __syncthreads();"]
        cur, flops = "x", 0
        for i, st in enumerate(steps):
            if st.kind == "Pool":                         # closing GAP
                ih, iw, ic = st.input_shapes[0].dims
                calls.append(f"    nnb::chain_gap<{ih * iw}, {ic}>({cur}, dst);")
                break
            nxt = "ab"[i % 2]
            ep = self.epilogue_fields(st, st.output_shape.c)
            if st.kind == "DepthwiseConv2D":
                H, W, C = st.input_shapes[0].dims
                HO, WO, _ = st.output_shape.dims
                KH, KW = st.kernel_hw
                PT = same_padding(H, KH, st.stride)[0] if st.padding == "same" else 0
                PL = same_padding(W, KW, st.stride)[0] if st.padding == "same" else 0
                f = dict(H=H, W=W, C=C, HO=HO, WO=WO, KH=KH, KW=KW, S=st.stride, PT=PT, PL=PL,
                         W_OFF=self.pool.add(st.kernel), B_OFF=self.pool.add(st.bias), **ep)
                tmpl = "ChainDw"
            else:
                HO, WO, CO = st.output_shape.dims
                CI = st.input_shapes[0].c
                tp, tc = chain_pw_tile(HO * WO, CO)
                f = dict(P=HO * WO, CI=CI, CO=CO, TP=tp, TC=tc,
                         W_OFF=self.pool.add(np.asarray(st.kernel, F32).reshape(CI, CO)),
                         B_OFF=self.pool.add(st.bias), **ep)
                tmpl = "ChainPw"
            structs.append(_cfg_struct(f"S{i}", f).replace("\n", "\n  "))
            calls += [f"    nnb::{tmpl}<S{i}>::run(pool, {cur}, {nxt});", "    __syncthreads();"]
            cur = nxt
            if i == len(steps) - 1:
                oh, ow, oc = st.output_shape.dims
                calls.append(f"    nnb::chain_store<{oh * ow}, {oc}>({cur}, dst);")
        code = "\n".join(["  " + x for x in structs] + [
            "  __device__ static __forceinline__ void body(const float* __restrict__ pool, "
            "const float* __restrict__ src, float* __restrict__ dst, float* x, float* a, float* b) {"]
            + calls + ["  }"])
        x_floats = chain_bytes(steps[0].input_shapes[0]) // 4
        ab_floats = max(chain_bytes(st.output_shape) for st in steps[:-1]) // 4
        fields = dict(IN_OFF=self.arena_off(u.input_ids[0]), IN_IMG=self.img_bytes(u.input_ids[0]),
                      OUT_OFF=self.arena_off(u.output_id), OUT_IMG=self.img_bytes(u.output_id),
                      X_FLOATS=x_floats, AB_FLOATS=ab_floats)
        smem = 4 * (x_floats + 2 * ab_floats)
        kinds = "".join("d" if st.kind == "DepthwiseConv2D" else "p" if st.kind == "Conv2D"
                        else "g" for st in steps)
        self.emit(pos, "chain", "nnb::Chain", fields, CHAIN_THREADS, smem, 1, 1,
                  dynamic_smem=True, code=code,
                  note=f"chain of {len(steps)} steps ({kinds}) {steps[0].input_shapes[0]} -> "
                       f"{u.output_shape}, one CTA per image, {smem // 1024} KB shared")

    def tc_chain(self, pos, u):
        """Alternating depthwise / pointwise layers over <= 64-pixel maps on
        the tensor cores, two images per CTA for the whole run
        (nnb_tcchain.cuh, planner.fuse_tc_chain).  Pointwise weights are
        split (3xTF32, round-to-nearest hi) and pre-swizzled into the shared-
        memory image of a K-major SW128 operand, one [B_hi | B_lo] block per
        32-wide k-block, streamed by 1-D bulk copies."""
        steps = u.steps
        AS = max(st.output_shape.c for st in steps if st.kind == "Conv2D") + 4
        calls, structs, blocks = [], [], []           # blocks: (pool offset, bytes, layer, stage)
        layer = 0
        for i, st in enumerate(steps):
            last = i == len(steps) - 1
            ep = self.epilogue_fields(st, st.output_shape.c)
            if st.kind == "DepthwiseConv2D":
                H, W, C = st.input_shapes[0].dims
                HO, WO, _ = st.output_shape.dims
                KH, KW = st.kernel_hw
                PT = same_padding(H, KH, st.stride)[0] if st.padding == "same" else 0
                PL = same_padding(W, KW, st.stride)[0] if st.padding == "same" else 0
                f = dict(H=H, W=W, C=C, HO=HO, WO=WO, KH=KH, KW=KW, S=st.stride, PT=PT, PL=PL,
                         W_OFF=self.pool.add(st.kernel), B_OFF=self.pool.add(st.bias),
                         SRC_GLOBAL=int(i == 0), SRC_IMG=4 * st.input_shapes[0].elements,
                         AS_IN=AS, KA=C, OUT_IMG=self.img_bytes(u.output_id), **ep)
                calls.append(f"    nnb::{'TccDwOut' if last else 'TccDwA'}<S{i}>::run(x);")
            else:
                HO, WO, N = st.output_shape.dims
                K = st.input_shapes[0].c
                wt = np.ascontiguousarray(np.asarray(st.kernel, F32).reshape(K, N).T)   # [N][K]
                hi = tf32_split_hi(wt, self.split_rn)
                lo = (wt - hi).astype(F32)
                blk0 = len(blocks)
                for kb in range(K // 32):
                    img = b""
                    for part in (hi, lo):
                        blk = part[:, kb * 32:(kb + 1) * 32].reshape(N, 8, 4)
                        sw = np.empty_like(blk)
                        rows = np.arange(N)[:, None]
                        sw[rows, np.arange(8)[None, :] ^ (rows % 8)] = blk
                        img += np.ascontiguousarray(sw, F32).tobytes()
                    off = self.pool.add(np.frombuffer(img, F32))
                    blocks.append((off, len(img), layer, kb))
                f = dict(K=K, N=N, P=HO * WO, LAYER=layer, BLK0=blk0, B_OFF=self.pool.add(st.bias),
                         AS_OUT=AS, LAST=int(last), OUT_IMG=self.img_bytes(u.output_id), **ep)
                if i == 0:                      # the chain input -> A operand
                    structs.append(_cfg_struct("SA", dict(
                        P=st.input_shapes[0].h * st.input_shapes[0].w, K=K,
                        SRC_IMG=4 * st.input_shapes[0].elements)).replace("\n", "\n  "))
                    calls.append("    nnb::TccLoadA<SA>::run(x);")
                calls.append(f"    nnb::TccPw<Cfg_{len(self.names)}, S{i}>::run(x);")
                layer += 1
            structs.append(_cfg_struct(f"S{i}", f).replace("\n", "\n  "))

        def table(name, vals):
            cases = " ".join(f"case {j}: return {v}LL;" for j, v in enumerate(vals))
            return (f"  __device__ static __forceinline__ long long {name}(int i) "
                    f"{{ switch (i) {{ {cases} default: return 0; }} }}")
        code = "\n".join(["  " + x for x in structs] + [
            table("blk_off", [b[0] for b in blocks]), table("blk_bytes", [b[1] for b in blocks]),
            table("blk_layer", [b[2] for b in blocks]), table("blk_stage", [b[3] for b in blocks]),
            "  __device__ static __forceinline__ void body(nnb::TcChainCtx& x) {"] + calls + ["  }"])
        nstage = max(b[3] for b in blocks) + 1
        stage_bytes = -(-max(b[1] for b in blocks) // 1024) * 1024
        act_floats = 2 * 64 * AS
        fields = dict(IN_OFF=self.arena_off(u.input_ids[0]), IN_IMG=self.img_bytes(u.input_ids[0]),
                      OUT_OFF=self.arena_off(u.output_id), OUT_IMG=self.img_bytes(u.output_id),
                      NSTAGE=nstage, STAGE_BYTES=stage_bytes, ACT_FLOATS=act_floats,
                      NBLK=len(blocks))
        smem = 1024 + nstage * stage_bytes + 4 * act_floats + 256
        n_pw = sum(st.kind == "Conv2D" for st in steps)
        self.emit(pos, "tcchain", "nnb::TcChain", fields, 256, smem, 1, 2,
                  code=code,
                  note=f"tcgen05 chain of {len(steps)} layers ({n_pw} pointwise 3xTF32, A in "
                       f"TMEM) {steps[0].input_shapes[0]} -> {u.output_shape}, 2 images per CTA, "
                       f"{len(blocks)} weight blocks in a {nstage}-stage ring, {smem // 1024} KB "
                       "shared")

    def depthwise(self, pos, u, n_cap=1 << 30):
        H, W, C = u.input_shapes[0].dims
        HO, WO, _ = u.output_shape.dims
        KH, KW = u.kernel_hw
        S = u.stride
        PT = same_padding(H, KH, S)[0] if u.padding == "same" else 0
        PL = same_padding(W, KW, S)[0] if u.padding == "same" else 0
        vec = 4 if C % 4 == 0 else 1
        base = dict(H=H, W=W, C=C, HO=HO, WO=WO, KH=KH, KW=KW, S=S, PT=PT, PL=PL,
                    VEC=vec, IN_OFF=self.arena_off(u.input_ids[0]),
                    IN_IMG=self.img_bytes(u.input_ids[0]),
                    OUT_OFF=self.arena_off(u.output_id), OUT_IMG=self.img_bytes(u.output_id),
                    W_OFF=self.pool.add(u.kernel), B_OFF=self.pool.add(u.bias))
        base.update(self.epilogue_fields(u, C))

        def variant(px, n_min, n_max):
            n_max = min(n_max, n_cap)
            if n_min > n_max:
                return
            per_img = HO * -(-WO // px) * (C // vec)
            self.emit(pos, f"dw{KH}x{KW}", "nnb::Depthwise",
                      dict(base, PX=px, IDX32=int(self.cap * per_img < 2 ** 31)),
                      ELEM_BLOCK, 0, per_img, ELEM_BLOCK, n_min=n_min, n_max=n_max,
                      note=f"{px} px/thread")
        # several output pixels per thread share input columns in registers
        # (measured: 1.4-1.7x at C >= 16); narrow channel vectors keep one
        # pixel per thread (the x-strided warp touches 4x the cache lines),
        # and so do batches too small to fill the GPU with the wide variant
        wide = 1 if C // vec < 4 else min(4 if S == 1 else 2, WO)
        if wide == 1:
            variant(1, 1, 1 << 30)
            return
        per_wide = HO * -(-WO // wide) * (C // vec)
        n_small = (self.sm_count * 512 - 1) // per_wide
        if n_small >= 1:
            variant(1, 1, n_small)
        if n_small < self.max_batch:
            variant(wide, n_small + 1, 1 << 30)

    def pool_unit(self, pos, u, n_max=1 << 30):
        H, W, C = u.input_shapes[0].dims
        PH, PW = u.kernel_hw
        S = u.stride
        out_shape = u.pre_up_shape if u.upsample_after > 1 else u.output_shape
        if out_shape.rank == 1:
            HO = WO = 1
        else:
            HO, WO = out_shape.h, out_shape.w
        PT = same_padding(H, PH, S)[0] if u.padding == "same" else 0
        PL = same_padding(W, PW, S)[0] if u.padding == "same" else 0
        vec = 4 if C % 4 == 0 else 1
        fields = dict(H=H, W=W, C=C, HO=HO, WO=WO, PH=PH, PW=PW, S=S, PT=PT, PL=PL,
                      AVG=u.pool_op == "avg", VEC=vec, UPF=u.upsample_after,
                      IN_OFF=self.arena_off(u.input_ids[0]),
                      IN_IMG=self.img_bytes(u.input_ids[0]),
                      OUT_OFF=self.arena_off(u.output_id), OUT_IMG=self.img_bytes(u.output_id))
        tag = ("gap" if (HO, WO) == (1, 1) and (PH, PW) == (H, W)
               else f"{u.pool_op}pool{PH}x{PW}")
        self.emit(pos, tag, "nnb::Pool", fields, ELEM_BLOCK, 0,
                  HO * WO * (C // vec), ELEM_BLOCK, n_max=n_max)

    def elementwise(self, pos, u):
        shape = u.output_shape
        elems = shape.elements
        ch = shape.dims[-1]
        vec = 4 if (elems % 4 == 0 and (u.scale is None or ch % 4 == 0)) else 1
        ins = list(u.input_ids)
        first = True
        out = u.output_id
        while ins:
            take = ins[:4] if first else ins[:3]
            ins = ins[len(take):]
            srcs = take if first else [out] + take
            fields = dict(ELEMS=elems, IMG=4 * elems, VEC=vec, NIN=len(srcs),
                          OUT_OFF=self.arena_off(out), CH=ch)
            for k in range(4):
                fields[f"IN{k}_OFF"] = self.arena_off(srcs[k]) if k < len(srcs) else 0
            last = not ins
            affine = u.scale is not None and last
            fields.update(AFFINE=affine,
                          S_OFF=self.pool.add(u.scale) if affine else 0,
                          O_OFF=self.pool.add(u.offset) if affine else 0,
                          ACT=ACT_CODE[u.activation] if last else 0,
                          MODE=MODE_CODE[self.opt.activation_mode])
            tag = "add" if u.kind == "Add" else ("bn" if u.scale is not None else "act")
            self.emit(pos, tag, "nnb::Elementwise", fields, ELEM_BLOCK, 0,
                      elems // vec, ELEM_BLOCK)
            first = False

    def gap_dense(self, pos, u):
        """GlobalAveragePooling2D + narrow Dense, one warp per image (nnb_small.cuh GapDense)."""
        H, W, CH = u.input_shapes[0].dims
        CO = u.kernel.shape[1]
        fields = dict(H=H, W=W, CH=CH, CO=CO, IN_OFF=self.arena_off(u.input_ids[0]),
                      IN_IMG=self.img_bytes(u.input_ids[0]), OUT_OFF=self.arena_off(u.output_id),
                      OUT_IMG=self.img_bytes(u.output_id),
                      W_OFF=self.pool.add(np.asarray(u.kernel, F32)), B_OFF=self.pool.add(u.bias),
                      SOFTMAX=bool(u.softmax_after), SMEXP=SMEXP_CODE[self.opt.softmax_exp])
        fields.update(self.epilogue_fields(u, CO))
        self.emit(pos, "gap_dense", "nnb::GapDense", fields, 128, 0, 32, 128,
                  note=f"global average pool {H}x{W}x{CH} + Dense N={CO}, one warp per image")

    def softmax(self, pos, u):
        shape = u.output_shape
        L = shape.dims[-1]
        rows = shape.elements // L
        per_thread = L <= 16
        if L > 2048:
            raise UnsupportedLayer(f"softmax rows longer than 2048 ({L})")
        fields = dict(IN_OFF=self.arena_off(u.input_ids[0]), OUT_OFF=self.arena_off(u.output_id),
                      ROWS=rows, L=L, SMEXP=SMEXP_CODE[self.opt.softmax_exp],
                      PER_THREAD=per_thread)
        if per_thread:
            self.emit(pos, "softmax", "nnb::SoftmaxRows", fields, 128, 0, rows, 128)
        else:
            self.emit(pos, "softmax", "nnb::SoftmaxRows", fields, 128, 0, rows, 4)

    def upsample(self, pos, u):
        H, W, C = u.input_shapes[0].dims
        vec = 4 if C % 4 == 0 else 1
        fields = dict(H=H, W=W, C=C, F=u.factor, VEC=vec,
                      IN_OFF=self.arena_off(u.input_ids[0]), IN_IMG=self.img_bytes(u.input_ids[0]),
                      OUT_OFF=self.arena_off(u.output_id), OUT_IMG=self.img_bytes(u.output_id))
        self.emit(pos, "upsample", "nnb::Upsample", fields, ELEM_BLOCK, 0,
                  H * W * u.factor * u.factor * (C // vec), ELEM_BLOCK)

    def concat(self, pos, u):
        shapes = u.input_shapes
        if u.output_shape.rank == 1:
            P, chans = 1, [s.dims[0] for s in shapes]
        else:
            P, chans = shapes[0].h * shapes[0].w, [s.c for s in shapes]
        if len(shapes) > 4:
            raise UnsupportedLayer("Concatenate of more than four tensors")
        CT = sum(chans)
        vec = 4 if all(c % 4 == 0 for c in chans) else 1
        fields = dict(P=P, CT=CT, NIN=len(chans), VEC=vec,
                      OUT_OFF=self.arena_off(u.output_id))
        for k in range(4):
            fields[f"C{k}"] = chans[k] if k < len(chans) else 0
            fields[f"OFF{k}"] = self.arena_off(u.input_ids[k]) if k < len(chans) else 0
        self.emit(pos, "concat", "nnb::Concat", fields, ELEM_BLOCK, 0, P * CT // vec, ELEM_BLOCK)

    def pad(self, pos, u):
        H, W, C = u.input_shapes[0].dims
        HO, WO, _ = u.output_shape.dims
        (t, _b), (l, _r) = u.pad
        vec = 4 if C % 4 == 0 else 1
        fields = dict(H=H, W=W, C=C, HO=HO, WO=WO, PT=t, PL=l, VEC=vec,
                      IN_OFF=self.arena_off(u.input_ids[0]), IN_IMG=self.img_bytes(u.input_ids[0]),
                      OUT_OFF=self.arena_off(u.output_id), OUT_IMG=self.img_bytes(u.output_id))
        self.emit(pos, "zeropad", "nnb::Pad", fields, ELEM_BLOCK, 0, HO * WO * (C // vec),
                  ELEM_BLOCK)

    def run(self):
        if self.tiny and not self.mega:
            self._tiny()
        for pos, u in enumerate(self.plan.units):
            self._n_cap = self.head_cap.get(pos)
            if u.kind == "Dense" and u.gap is not None:
                self.gap_dense(pos, u)
            elif u.kind in ("Dense", "Conv2D"):
                self._dual_from = self._edw_from = 1 << 30
                self.gemm(pos, u)
                if u.dual_pool is not None and self._dual_from > 1:
                    # batches whose conv kernel has no second (pooled) store
                    self.pool_unit(pos, u.dual_pool, n_max=self._dual_from - 1)
                if u.dw_after is not None and self._edw_from > 1:
                    # batches whose conv kernel has no depthwise epilogue
                    if u.dw_after.kind == "Pool":
                        self.pool_unit(pos, u.dw_after, n_max=self._edw_from - 1)
                    else:
                        self.depthwise(pos, u.dw_after, n_cap=self._edw_from - 1)
            elif u.kind == "DepthwiseConv2D":
                if u.residual_id is not None or u.pool_after or u.softmax_after:
                    raise UnsupportedLayer("depthwise epilogue fusion")
                self.depthwise(pos, u)
            elif u.kind == "Pool":
                self.pool_unit(pos, u)
            elif u.kind in ("ElementwiseActivation", "Add"):
                self.elementwise(pos, u)
            elif u.kind == "Softmax":
                self.softmax(pos, u)
            elif u.kind == "Upsample":
                self.upsample(pos, u)
            elif u.kind == "Concat":
                self.concat(pos, u)
            elif u.kind == "Pad":
                self.pad(pos, u)
            elif u.kind == "Chain":
                self.chain(pos, u)
            elif u.kind == "TcChain":
                self.tc_chain(pos, u)
            else:
                raise UnsupportedLayer(f"no kernel for unit kind {u.kind}")
        self._n_cap = None
        self.mega_source = ""
        arena_extra = self._mega() if self.mega else 0
        head = '#include "nnb_kernels.cuh"\n\n'
        # one TU with every regular unit (inspection, the nvcc build check);
        # the persistent kernel is its own TU (compiled with NNB_MEGA=1)
        src = head + "\n\n".join(c for c in self.chunks if not c.startswith("#define NNB_MEGA")) + "\n"
        sources, index, ks = [], {}, []
        for chunk in self.chunks:
            tu = chunk if chunk.startswith("#define NNB_MEGA") else head + chunk
            if tu not in index:
                index[tu] = len(sources)
                sources.append(tu)
            ks.append(index[tu])
        return Specialization(source=src, launches=self.launches, pool=bytes(self.pool.data),
                              kernel_names=list(self.names), sources=sources,
                              kernel_source=ks, arena_extra=arena_extra,
                              mega_source=self.mega_source)

    def _mega(self):
        """Batch-1 persistent kernel: for n <= NB one
        cooperative launch walks every launch unit of the schedule in order --
        each unit's own template, fed virtual block indices by a grid-stride
        loop -- with a grid-wide barrier between units, instead of one graph
        node per unit.  NB is the largest batch <= MEGA_MAX_N whose units are
        all non-TMA kernels with blocks <= MEGA_THREADS.  The regular launches
        then start at NB + 1.  Returns the arena bytes it needs (the barrier
        counter).

        Opt-in (``mega=True``): measured on B200 it is slower than the graph
        replay with programmatic dependent launch -- batch-1 latency is the
        units' own dependent-load latency, not launch overhead, and a
        grid-wide barrier costs about what a graph node does (cfg0 27 -> 35
        us, cfg2 35 -> 37 us, cfg3 107 -> 126 us; "full" 148-CTA grids and
        backoff in the barrier did not change that)."""
        NB = 0
        for n in range(1, min(MEGA_MAX_N, self.max_batch) + 1):
            act = [l for l in self.launches if l.n_min <= n <= l.n_max]
            if any(l.tmaps or l.block > MEGA_THREADS for l in act):
                break
            NB = n
        if NB == 0:
            return 0
        parts = [i for i, l in enumerate(self.launches) if l.n_min <= NB]
        if len(parts) < 2:
            return 0
        sync_off = self.asg.arena_size * self.cap          # appended 256 bytes
        smem, width, gmax = 0, 0, 1
        body = ["#define NNB_MEGA 1", '#include "nnb_kernels.cuh"', ""]
        code = []
        for k, i in enumerate(parts):
            l = self.launches[i]
            cfg, struct, template, dyn = self.unit_src[i]
            body.append(struct)
            width = max(width, l.block)
            smem = max(smem, l.smem)
            if template == "nnb::DenseSmallM":
                f = dict(re.findall(r"static constexpr long long (\w+) = (-?\d+)LL", struct))
                smem = max(smem, int(f["KS"]) * int(f["MB"]) * 32 * 4)
            gmax = max(gmax, -(-NB * l.items_per_image // l.items_per_block) * l.grid_mult)
            call = (f"{template}<{cfg}>::run(pool, arena, n, *reinterpret_cast<{template}<{cfg}>::Smem*>"
                    f"(nnb_dyn_smem))" if dyn else f"{template}<{cfg}>::run(pool, arena, n)")
            last = k == len(parts) - 1
            code.append(
                f"  if (n >= {l.n_min} && n <= {min(l.n_max, NB)}) {{   // {l.kernel}\n"
                f"    const long long g = (((long long)n * {l.items_per_image} + {l.items_per_block - 1})"
                f" / {l.items_per_block}) * {l.grid_mult};\n"
                f"    for (long long vb = blockIdx.x; vb < g; vb += gridDim.x) {{\n"
                f"      __syncthreads();\n"
                f"      if (threadIdx.x == 0) {{ nnb::nnb_mega_bid = (int)vb; nnb::nnb_mega_bdim = {l.block}; }}\n"
                f"      __syncthreads();\n"
                f"      if (threadIdx.x < {l.block}) {call};\n"
                f"    }}\n"
                + ("" if last else "    nnb::mega_grid_sync(sync, (++epoch) * gridDim.x);\n")
                + "  }\n")
        grid = self.sm_count if self.mega == "full" else min(self.sm_count, gmax)
        body.append(
            f"\nextern \"C\" __global__ void __launch_bounds__({width}, 1) nnb_mega("
            f"const float* __restrict__ pool, float* __restrict__ arena, int n) {{\n"
            f"  NNB_PDL_PROLOGUE\n"
            f"  extern __shared__ __align__(16) unsigned char nnb_dyn_smem[];\n"
            f"  unsigned* sync = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(arena) + {sync_off}LL);\n"
            f"  unsigned epoch = 0;\n" + "".join(code) + "}\n")
        kname = "nnb_mega"
        self.chunks.append("\n".join(body))
        self.names.append(kname)
        # the regular launches take over above NB
        for i in parts:
            self.launches[i].n_min = max(self.launches[i].n_min, NB + 1)
        self.launches = [l for l in self.launches if l.n_min <= l.n_max]
        self.launches.append(Launch(kname, width, smem, 1, 1 << 30, grid_mult=grid, n_min=1,
                                    n_max=NB, unit=-1,
                                    note=f"persistent: {len(parts)} units, {grid} CTAs, n <= {NB}",
                                    cooperative=True, zero_offset=sync_off))
        self.mega_source = self.chunks[-1]
        return 256


def bf16_rn(x):
    """float32 -> bfloat16 bit patterns (uint16), round to nearest even."""
    u = np.ascontiguousarray(x, F32).view(np.uint32)
    return ((u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)).astype(np.uint16)


def bf16_corr_words(hi, lo):
    """B_corr operand of the CORR_BF16 tcgen05 GEMM: per row of the K-major
    [Npad, Kpad] weights and per k-step of 8, 16 bf16 = [bf16(lo) x 8,
    bf16(hi) x 8] (the A side holds [bf16(a_hi) x 8, bf16(a_lo) x 8], so one
    K = 16 MMA forms a_hi*b_lo + a_lo*b_hi), packed little-endian into
    float32 words: the same bytes as the B_lo tile it replaces."""
    n, k = hi.shape
    assert k % 8 == 0
    bh = bf16_rn(hi).reshape(n, k // 8, 8)
    bl = bf16_rn(lo).reshape(n, k // 8, 8)
    words = np.concatenate([bl, bh], axis=2).reshape(n, 2 * k)
    return np.ascontiguousarray(words).view("<u4").view(F32)


def tf32_split_hi(w, rn=True):
    """TF32 'hi' part of a float32 array: rounded to the nearest TF32 (11
    significant bits) when ``rn``, else truncated; ``w - hi`` is exact."""
    u = np.ascontiguousarray(w, F32).view(np.uint32)
    t = u & np.uint32(0xFFFFE000)
    if rn:
        r = (u + np.uint32(0x1000)) & np.uint32(0xFFFFE000)
        ok = np.isfinite(r.view(F32))
        t = np.where(ok, r, t)
    return t.view(F32)


def specialize(plan, assignment, options, max_batch, capacity, **tuning):
    """Specialise every launch unit; ``tuning`` are the Specializer's keyword
    options (use_tc, sm_count, tc_min_rows, ...).  A plan made by the
    reference's planner goes through planner.adopt_plan first."""
    return Specializer(plan, assignment, options, max_batch, capacity, **tuning).run()
