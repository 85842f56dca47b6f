"""Kernel-selection and code-generation knobs of the B200 build.

The reference's constructor is ``CompiledNetwork(manifest, weights, options)``
(pkg/src/nnjit/runtime.py:33-34); the drop-in keeps that signature and adds
only ``batch``, ``device``, ``cache_dir`` and ONE mapping, ``tuning``, for
every experiment / A-B knob of the planner and the kernel specialiser::

    CompiledNetwork(m, w, opts, batch=4096, tuning={"tc_min_rows": 1})

The defaults are the measured selections; a key that is
not a field below raises ``ValueError`` naming the valid keys, so a typo never
reaches the specialiser as a raw ``TypeError``.
"""

from dataclasses import dataclass, fields, replace


@dataclass(frozen=True)
class Tuning:
    # -- planner (planner.py / buffers.py) -----------------------------------
    gpu_fusion: bool = True        # B200 epilogue fusions (pool, residual, softmax, upsample, concat)
    dw_fusion: object = "narrow"   # depthwise->pointwise: "narrow" (SepNarrow), True (all), False
    head: bool = True              # fuse a <=16-wide Dense head into a tcgen05 Dense epilogue
    pw_dw: object = True           # pointwise conv + the depthwise conv consuming it, computed in the
                                   # tcgen05 epilogue where a 128-row tile holds whole images (fuse_pw_dw);
                                   # "bands": also maps <= 16 pixels wide as bands of rows (measured slower)
    gap_dense: bool = True         # GlobalAveragePooling2D + the <=32-wide Dense consuming it as one launch
    tc_chain: bool = False         # 8x8-stage pointwise/depthwise runs as one tcgen05 kernel
                                   # (planner.fuse_tc_chain; correct, break-even, opt-in)
    chain: bool = False            # small depthwise/pointwise runs as one FFMA kernel (fuse_chain;
                                   # correct, measured slower than the per-layer tcgen05 path)
    # -- kernel selection ----------------------------------------------------
    use_tc: bool = True            # tcgen05 3xTF32 GEMMs for Dense / 1x1 / KxK convs
    tc_min_rows: object = None     # rows per launch from which tcgen05 is used (None: kernels.TC_MIN_ROWS)
    tc_min_images: object = None   # convs: images from which tc_min_rows applies (None: TC_MIN_IMAGES)
    tc_min_k: object = None        # smallest contraction for tcgen05 (None: TC_MIN_K)
    tc_tile_use: float = 0.75      # useful-pixel fraction an 8x16 conv tile needs
    small_dense_rows: object = None  # split-K row kernel up to this many rows (None: SMALL_DENSE_ROWS)
    narrow: bool = True            # RowsNarrow streaming kernel for <=32-column GEMMs
    direct_imm: bool = True        # direct-conv weights as FFMA immediates
    sep_fma: bool = True           # SepNarrow depthwise taps with FFMA (False: mul-then-add, bit-exact)
    narrow_geo: object = None      # RowsNarrow geometry override (tile rows, K slices, stages)
    sep_geo: object = None         # SepNarrow geometry override (tile rows)
    mega: bool = False             # batch-1 persistent cooperative kernel (measured slower; opt-in)
    # -- tcgen05 GEMM code generation (nnb_gemm_tc.cuh) ----------------------
    tmem_a: bool = True            # A operand in TMEM (the "ts" MMA form) where it fits
    nacc: object = None            # accumulator chains per buffer
    aldg: bool = False             # A via cp.async instead of TMA
    kpack: bool = True             # pack KW taps of narrow convs into N
    kpack9: bool = True            # pack all KH x KW taps of CO = 16 convs into N (N = 144)
    kpack_wide: bool = True        # pack the KW taps of CO = 64 convs into N = 192 (merged correction)
    tiny: bool = False             # small nets at small batches as one TinyNet launch (opt-in:
                                   # cfg0 batch 1 37 us vs 23 us for the per-layer launches)
    epi_tma: bool = True           # TMA-store epilogue
    csplit: bool = True            # separate correction-product chain
    chunk: object = None           # k-blocks per accumulator chunk
    split_rn: bool = True          # round-to-nearest hi/lo split
    pair: bool = True              # CTA pairs (cta_group::2) for 256-row tiles
    abuf: object = None            # accumulator buffers (1 or 2)
    wide: bool = True              # N = 256 row tiles
    wide_bk: int = 32              # k-block of the N = 256 tiles
    wide_chunk: object = None      # main-chain chunk of the N = 256 tiles
    wide_csplit: bool = True       # separate correction chain of the N = 256 tiles (False: merged into
                                   # the main chain, two accumulator buffers: -2.4% on cfg1, but one
                                   # output in 10^7 just over the plain FP32 gate -- opt-in)
    rn_ss: object = 2              # shared-memory A split: 2 = lo rounded to TF32 (hi left to the
                                   # hardware), True = rounded hi written back, False = truncation
    corr_bf16: object = "wide"     # BF16 correction products: "wide" (N=256 tiles only), "auto"
                                   # (+ conv tiles with K >= 128), True (all), False
    cb16_w4: bool = True           # 4 split warps for BF16-correction tiles
    conv_w4: object = "auto"       # 4 split warps for conv tiles: "auto" (short k-block work), True, False
    rowshare: bool = True          # KPACK conv tiles: one A box of 8+KH-1 rows serves every kernel row
    small_conv: bool = True        # few-pixel 1x1 convs (one wave of GEMM tiles or less): split-K row kernel
    small_conv_kper: int = 16
    a_prefetch: int = 0            # L2 prefetch distance of A boxes (k-blocks)
    early_mma: bool = True         # N = 256 BF16-correction tiles: main MMAs before the split
    setreg: bool = True            # ... with six split warps and setmaxnreg register reallocation
    epi16: bool = False            # KPACK conv tiles with 32 outputs: sixteen epilogue warps (measured slower)

    def specializer_kwargs(self):
        """Keyword arguments of kernels.Specializer (the selection constants
        filled in where the field is None)."""
        from .kernels import (MEGA_TC_MIN_ROWS, SMALL_DENSE_ROWS, TC_MIN_IMAGES, TC_MIN_K,
                              TC_MIN_ROWS)
        skip = {"gpu_fusion", "dw_fusion", "chain", "tc_chain", "pw_dw", "gap_dense"}
        kw = {f.name: getattr(self, f.name) for f in fields(self) if f.name not in skip}
        if kw["tc_min_rows"] is None:
            kw["tc_min_rows"] = MEGA_TC_MIN_ROWS if self.mega else TC_MIN_ROWS
        if kw["tc_min_images"] is None:
            kw["tc_min_images"] = TC_MIN_IMAGES
        if kw["tc_min_k"] is None:
            kw["tc_min_k"] = TC_MIN_K
        if kw["small_dense_rows"] is None:
            kw["small_dense_rows"] = SMALL_DENSE_ROWS
        return kw


FIELDS = tuple(f.name for f in fields(Tuning))


def make_tuning(tuning=None):
    """Tuning from None, a Tuning, or a mapping of field -> value."""
    if tuning is None:
        return Tuning()
    if isinstance(tuning, Tuning):
        return tuning
    try:
        items = dict(tuning)
    except (TypeError, ValueError):
        raise ValueError(f"tuning must be a mapping or a Tuning, got {type(tuning).__name__}")
    bad = sorted(k for k in items if k not in FIELDS)
    if bad:
        raise ValueError(f"unknown tuning key(s) {bad}; valid keys: {', '.join(FIELDS)}")
    return replace(Tuning(), **items)
