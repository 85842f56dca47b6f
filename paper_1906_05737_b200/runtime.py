"""Compile-and-run facade: drop-in for pkg/src/nnjit/runtime.py:33-107.

``CompiledNetwork(manifest, weights, options)`` builds the graph, plans
fusion and the device arena, specialises one sm_100a kernel per launch unit,
compiles them with NVRTC inside the C-ABI runtime (libnnb.so) and keeps the
whole schedule ready for CUDA-graph replay.  A steady-state inference is the
reference's: write ``input_views``, call ``apply()``, read ``output_views``.

Differences from the reference, all additive:

* views are ``torch.Tensor`` objects on the GPU aliasing the device arena
  (zero-copy; stable objects for the lifetime of the network);
* ``batch=N`` compiles for up to N images: views then carry a leading batch
  axis and ``apply(n)`` runs the first ``n`` images; without ``batch`` the
  views have exactly the reference's per-image shapes;
* inputs are never clobbered, so ``apply()`` is idempotent (buffers.py);
* ``run_host(xs)`` is the end-to-end host-buffer path through the C ABI.

There is no CPU fallback: without libnnb.so or an sm_100 device the
constructor raises (``ImportError`` / ``UnsupportedDevice``).
"""

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .buffers import plan_buffers
from .errors import InputShapeMismatch
from .graph import build_graph
from .kernels import specialize
from .model_format import load_model
from .options import ApproximationOptions
from .planner import build_plan
from .tuning import make_tuning


def _capacity(batch):
    return (batch + 15) // 16 * 16


@dataclass
class CodeArtifact:
    """What compile() produced (cf. pkg/src/nnjit/codegen/compile.py:11-22)."""
    source: str
    kernel_names: list
    launches: list
    pool_data: bytes
    arena_size: int                 # bytes per image
    capacity: int                   # images the arena holds
    offsets: dict                   # tensor -> (offset, size) per image
    metadata: dict = field(default_factory=dict)


class _DeviceArray:
    """__cuda_array_interface__ exporter that keeps the owning net alive."""

    def __init__(self, owner, ptr, shape):
        self._owner = owner
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape),
                                         "typestr": "<f4", "version": 3, "strides": None}


class _Handle:
    """Owns the nnb_net*; destroyed when the last view/network drops it."""

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            if self.ptr:
                _native.lib().nnb_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


class CompiledNetwork:
    def __init__(self, manifest, weights, options=None, *, batch=None, device=0,
                 cache_dir=None, tuning=None):
        """pkg/src/nnjit/runtime.py:33-67 plus ``batch`` (images per replay),
        ``device``, ``cache_dir`` (cubin cache; "" disables it) and
        ``tuning`` (a mapping of tuning.Tuning fields; unknown keys raise
        ValueError)."""
        import torch

        t0 = time.perf_counter()
        self.options = options or ApproximationOptions()
        self.tuning = make_tuning(tuning)
        tn = self.tuning
        self.manifest = manifest
        self.device = device
        self.batch = batch
        self.max_batch = int(batch) if batch is not None else 1
        if self.max_batch < 1:
            raise ValueError("batch must be >= 1")
        _, _, sm_count = _native.device_check(device)
        self.graph = build_graph(manifest, weights)
        dw_fusion = tn.dw_fusion
        if tn.mega and dw_fusion == "narrow":
            dw_fusion = False      # the persistent kernel walks the unfused templates
        self.plan = build_plan(self.graph, gpu_fusion=tn.gpu_fusion, dw_fusion=dw_fusion,
                               chain=tn.chain and not tn.mega, tc_chain=tn.tc_chain and not tn.mega,
                               pw_dw=tn.pw_dw if (tn.use_tc and not tn.mega and not tn.tiny) else False,
                               gap_dense=tn.gap_dense and not tn.mega and not tn.tiny)
        self.assignment = plan_buffers(self.plan, reserve_heads=tn.head)
        cap = _capacity(self.max_batch)
        spec = specialize(self.plan, self.assignment, self.options, self.max_batch, cap,
                          sm_count=sm_count, **tn.specializer_kwargs())
        arena_bytes = self.assignment.arena_size * cap + spec.arena_extra

        def io(tids):
            return [(self.assignment.offsets[t][0] * cap, 4 * self.plan.tensors[t].elements)
                    for t in tids]

        ins, outs = io(self.plan.input_ids), io(self.plan.output_ids)
        L = _native.lib()
        names = (ctypes.c_char_p * max(len(spec.kernel_names), 1))(
            *[n.encode() for n in spec.kernel_names])
        srcs = (ctypes.c_char_p * len(spec.sources))(*[s.encode() for s in spec.sources])
        ksrc = (ctypes.c_int32 * max(len(spec.kernel_source), 1))(*spec.kernel_source)
        launches = (_native.Launch * max(len(spec.launches), 1))()
        index = {n: i for i, n in enumerate(spec.kernel_names)}
        for i, l in enumerate(spec.launches):
            tm = (_native.TMap * _native.MAX_TMAPS)()
            for k, t in enumerate(l.tmaps):
                tm[k] = _native.make_tmap(t)
            launches[i] = _native.Launch(index[l.kernel], l.block, l.smem, l.grid_mult,
                                         l.items_per_image, l.items_per_block,
                                         l.n_min, min(l.n_max, 1 << 30), l.grid_cap,
                                         len(l.tmaps), tm, l.cluster, int(l.cooperative),
                                         l.zero_offset)
        in_arr = (_native.IO * max(len(ins), 1))(*[_native.IO(o, b) for o, b in ins])
        out_arr = (_native.IO * max(len(outs), 1))(*[_native.IO(o, b) for o, b in outs])
        pool_buf = ctypes.create_string_buffer(spec.pool, max(len(spec.pool), 1))
        cache = cache_dir if cache_dir is not None else _native.default_cache_dir()
        desc = _native.NetDesc(
            device, srcs, len(spec.sources), str(_native.KERNEL_DIR).encode(),
            cache.encode() if cache else None, names, ksrc, len(spec.kernel_names),
            launches, len(spec.launches), ctypes.cast(pool_buf, ctypes.c_void_p),
            len(spec.pool), arena_bytes, self.max_batch, in_arr, len(ins), out_arr, len(outs))
        ptr = ctypes.c_void_p()
        _native.check(L.nnb_create(ctypes.byref(desc), ctypes.byref(ptr)), "nnb_create")
        self._h = _Handle(ptr.value)
        info = [ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_int32(), ctypes.c_double(),
                ctypes.c_int32()]
        _native.check(L.nnb_net_info(self._h.ptr, *[ctypes.byref(v) for v in info]))
        self.nvrtc_ms = info[3].value
        self.cubin_cache_hit = bool(info[4].value)
        self.artifact = CodeArtifact(
            source=spec.source, kernel_names=spec.kernel_names, launches=spec.launches,
            pool_data=spec.pool, arena_size=self.assignment.arena_size, capacity=cap,
            offsets=dict(self.assignment.offsets),
            metadata={"units": len(self.plan.units), "kernels": len(spec.kernel_names),
                      "launches": len(spec.launches), "pool_bytes": len(spec.pool),
                      "arena_bytes": arena_bytes, "code_bytes": len(spec.source),
                      "activation_mode": self.options.activation_mode,
                      "softmax_exp": self.options.softmax_exp,
                      "nvrtc_ms": self.nvrtc_ms, "cubin_cache_hit": self.cubin_cache_hit})
        self._io_in, self._io_out = ins, outs
        self._torch = torch
        self._tdev = torch.device("cuda", device)
        self.input_views = [self._view(off, self.graph.nodes[nid].output_shape.dims)
                            for (off, _), nid in zip(ins, self.graph.input_ids)]
        self.output_views = [self._view(off, self.graph.nodes[nid].output_shape.dims)
                             for (off, _), nid in zip(outs, self.graph.output_ids)]
        self.compile_ms = (time.perf_counter() - t0) * 1e3

    # -- views ------------------------------------------------------------
    def _view(self, offset, dims):
        torch = self._torch
        p = ctypes.c_void_p()
        _native.check(_native.lib().nnb_arena_ptr(self._h.ptr, offset, ctypes.byref(p)))
        shape = (self.artifact.capacity,) + tuple(dims)
        t = torch.as_tensor(_DeviceArray(self._h, p.value, shape), device=self._tdev)
        t = t[:self.max_batch]
        return t[0] if self.batch is None else t

    def _stream(self):
        return ctypes.c_void_p(self._torch.cuda.current_stream(self._tdev).cuda_stream)

    # -- execution ------------------------------------------------------------
    def apply(self, n=None):
        """Replay the compiled schedule (one CUDA graph) over the first ``n``
        images (default: all ``batch``) on the current torch stream.  Only the
        first ``n`` rows of the output views are defined afterwards (the arena
        space of rows ``>= n`` is shared with intermediate tensors)."""
        n = self.max_batch if n is None else int(n)
        _native.check(_native.lib().nnb_apply(self._h.ptr, n, self._stream()), "apply")

    def synchronize(self):
        _native.check(_native.lib().nnb_sync(self._h.ptr, self._stream()))

    def run(self, inputs, n=None):
        """Copy inputs into the views, apply, return the output views (the same
        objects on every call, pkg/src/nnjit/runtime.py:75-87)."""
        torch = self._torch
        if len(inputs) != len(self.input_views):
            raise InputShapeMismatch(f"expected {len(self.input_views)} inputs, got {len(inputs)}")
        count = None
        for view, x in zip(self.input_views, inputs):
            if not isinstance(x, torch.Tensor):
                x = np.asarray(x, np.float32)
                if not x.flags.writeable:             # torch.from_numpy wants writable memory
                    x = x.copy()
            t = x if isinstance(x, torch.Tensor) else torch.from_numpy(x)
            if self.batch is None:
                if tuple(t.shape) != tuple(view.shape):
                    raise InputShapeMismatch(f"input shape {tuple(t.shape)} does not match "
                                             f"{tuple(view.shape)}")
                view.copy_(t, non_blocking=False)
                count = 1
            else:
                if tuple(t.shape[1:]) != tuple(view.shape[1:]) or not 1 <= t.shape[0] <= self.max_batch:
                    raise InputShapeMismatch(f"input shape {tuple(t.shape)} does not match "
                                             f"(<= {self.max_batch}, {tuple(view.shape[1:])})")
                if count is not None and t.shape[0] != count:
                    raise InputShapeMismatch("inputs disagree on the batch size")
                count = int(t.shape[0])
                view[:count].copy_(t)
        self.apply(n if n is not None else count)
        return list(self.output_views)

    def run_host(self, inputs, outputs=None, n=None):
        """End-to-end call through the C ABI with host buffers: H2D copy of the
        inputs, one graph replay, D2H copy of the outputs, synchronise.
        ``inputs``/``outputs`` are C-contiguous float32 numpy arrays (pinned
        memory from ``pinned_empty`` is fastest) holding at least ``n`` images;
        anything else raises ``InputShapeMismatch`` before the C ABI sees a
        pointer."""
        n = n if n is not None else self.max_batch
        if not 1 <= n <= self.max_batch:
            raise InputShapeMismatch(f"batch {n} outside [1, {self.max_batch}]")
        per = lambda v: tuple(v.shape[1:]) if self.batch is not None else tuple(v.shape)
        xs = _host_buffers(inputs, [per(v) for v in self.input_views], n, "input",
                           batched=self.batch is not None)
        if outputs is None:
            outputs = [np.empty(((n,) if self.batch is not None else ()) + per(v), np.float32)
                       for v in self.output_views]
        _host_buffers(outputs, [per(v) for v in self.output_views], n, "output",
                      batched=self.batch is not None, writable=True)
        ip = (ctypes.c_void_p * len(xs))(*[x.ctypes.data for x in xs])
        op = (ctypes.c_void_p * len(outputs))(*[o.ctypes.data for o in outputs])
        _native.check(_native.lib().nnb_run_host(self._h.ptr, n, ip, op, self._stream()), "run_host")
        return outputs

    def time_apply(self, n=None, iters=10):
        """Mean milliseconds per replay measured with CUDA events."""
        n = self.max_batch if n is None else n
        ms = ctypes.c_double()
        _native.check(_native.lib().nnb_time_apply(self._h.ptr, n, iters, self._stream(),
                                                   ctypes.byref(ms)))
        return ms.value

    def time_launch(self, index, n=None, iters=10):
        """Mean milliseconds of one schedule launch run alone (CUDA events)."""
        n = self.max_batch if n is None else n
        ms = ctypes.c_double()
        _native.check(_native.lib().nnb_time_launch(self._h.ptr, index, n, iters, self._stream(),
                                                    ctypes.byref(ms)))
        return ms.value

    def time_sequence(self, n=None, iters=10):
        """Per-launch mean milliseconds within full passes over ``n`` images
        (direct launches in replay order, CUDA events between them).
        Returns {launch index: ms} for the launches of the pass."""
        n = self.max_batch if n is None else n
        L = len(self.artifact.launches)
        ms = (ctypes.c_double * max(L, 1))()
        _native.check(_native.lib().nnb_time_sequence(self._h.ptr, n, iters, self._stream(), ms))
        return {i: ms[i] for i in range(L) if ms[i] >= 0}

    def launches_for(self, n=None):
        """Indices of the launches a replay over ``n`` images runs."""
        n = self.max_batch if n is None else n
        return [i for i, l in enumerate(self.artifact.launches) if l.n_min <= n <= l.n_max]

    def describe(self):
        lines = [f"units ({len(self.plan.units)}):"]
        for pos, u in enumerate(self.plan.units):
            lines.append(f"  {pos:3d}: {u.describe()}")
        lines.append("launches:")
        for l in self.artifact.launches:
            lines.append(f"  {l.kernel}  block {l.block} smem {l.smem}  {l.note}")
        lines.append("buffers:")
        lines.append(self.assignment.describe())
        md = self.artifact.metadata
        lines.append(f"{md['kernels']} kernels, pool {md['pool_bytes']} bytes, arena "
                     f"{md['arena_bytes']} bytes (capacity {self.artifact.capacity}), "
                     f"compiled in {self.compile_ms:.2f} ms (NVRTC {self.nvrtc_ms:.1f} ms, "
                     f"cache {'hit' if self.cubin_cache_hit else 'miss'})")
        return "\n".join(lines)


def _host_buffers(arrays, shapes, n, what, batched=True, writable=False):
    """Validate host buffers before their raw pointers cross the C ABI: one
    per network input/output, float32, C-contiguous, per-image shape
    ``shapes[i]`` and at least ``n`` images (``batched``), writable for
    outputs.  Inputs that are not float32 C-contiguous are converted (a copy);
    outputs must already be right, since the D2H copy writes through them."""
    arrays = list(arrays)
    if len(arrays) != len(shapes):
        raise InputShapeMismatch(f"expected {len(shapes)} {what}s, got {len(arrays)}")
    out = []
    for i, (a, shape) in enumerate(zip(arrays, shapes)):
        if not isinstance(a, np.ndarray):
            if writable:
                raise InputShapeMismatch(f"{what} {i} must be a numpy array")
            a = np.asarray(a)
        if not writable:
            a = np.ascontiguousarray(a, np.float32)
        elif a.dtype != np.float32 or not a.flags.c_contiguous or not a.flags.writeable:
            raise InputShapeMismatch(f"{what} {i} must be a writable C-contiguous float32 array "
                                     f"(got {a.dtype}, contiguous={a.flags.c_contiguous}, "
                                     f"writable={a.flags.writeable})")
        got = tuple(a.shape[1:]) if batched else tuple(a.shape)
        if got != tuple(shape) or (batched and a.shape[0] < n):
            want = f"(>= {n}, {tuple(shape)})" if batched else f"{tuple(shape)}"
            raise InputShapeMismatch(f"{what} {i} shape {tuple(a.shape)} does not match {want}")
        out.append(a)
    return out


def pinned_empty(shape):
    """A page-locked float32 numpy array (fast H2D/D2H for run_host)."""
    n = int(np.prod(shape)) * 4
    p = ctypes.c_void_p()
    _native.check(_native.lib().nnb_host_alloc(max(n, 4), ctypes.byref(p)))
    buf = (ctypes.c_char * max(n, 4)).from_address(p.value)
    arr = np.frombuffer(buf, np.float32, count=n // 4).reshape(shape)
    arr_holder = _PinnedHolder(p.value)
    arr = arr.view(_PinnedArray)
    arr._holder = arr_holder
    return arr


class _PinnedHolder:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            _native.lib().nnb_host_free(self.ptr)
        except Exception:
            pass


class _PinnedArray(np.ndarray):
    pass


class PipelinedNetwork:
    """Host-buffer inference over a large batch with the PCIe copies hidden
    behind the compute: ``chunks`` CompiledNetworks of ceil(batch/chunks)
    images each (same model, same device, one CUDA stream each; the
    specialised kernels are shared through the cubin cache).  ``run_host``
    hands the host buffers to ``nnb_run_host_chunked``, which queues every
    chunk's H2D copy, replay and D2H copy before waiting for any, so chunk
    j's upload overlaps chunk j-1's replay and download.  Outputs are
    identical to one CompiledNetwork over the whole batch (images are
    independent and every kernel is batch-size invariant per image)."""

    def __init__(self, manifest, weights, options=None, *, batch, chunks=4, device=0, **kw):
        import torch
        if batch < 1 or chunks < 1:
            raise ValueError("batch and chunks must be >= 1")
        self._torch = torch
        self.batch = self.max_batch = int(batch)
        self.chunks = max(1, min(int(chunks), self.batch))
        per = -(-self.batch // self.chunks)
        self.nets = [CompiledNetwork(manifest, weights, options, batch=per, device=device, **kw)
                     for _ in range(self.chunks)]
        self.streams = [torch.cuda.Stream(device=torch.device("cuda", device))
                        for _ in range(self.chunks)]
        self.options = self.nets[0].options
        self.plan = self.nets[0].plan
        self.artifact = self.nets[0].artifact
        self.compile_ms = sum(n.compile_ms for n in self.nets)

    @property
    def output_shapes(self):
        return [tuple(v.shape[1:]) for v in self.nets[0].output_views]

    def run_host(self, inputs, outputs=None, n=None):
        """``n`` (default ``batch``) images of C-contiguous float32 host
        ``inputs`` (pinned: ``pinned_empty``) in, the outputs written into
        ``outputs`` (allocated when None) and returned."""
        n = self.batch if n is None else int(n)
        if not 1 <= n <= self.batch:
            raise InputShapeMismatch(f"batch {n} outside [1, {self.batch}]")
        xs = _host_buffers(inputs, [tuple(v.shape[1:]) for v in self.nets[0].input_views], n,
                           "input")
        if outputs is None:
            outputs = [np.empty((n,) + s, np.float32) for s in self.output_shapes]
        _host_buffers(outputs, self.output_shapes, n, "output", writable=True)
        VP = ctypes.c_void_p
        nets = (VP * self.chunks)(*[net._h.ptr for net in self.nets])
        streams = (VP * self.chunks)(*[st.cuda_stream for st in self.streams])
        ip = (VP * len(xs))(*[x.ctypes.data for x in xs])
        op = (VP * len(outputs))(*[o.ctypes.data for o in outputs])
        _native.check(_native.lib().nnb_run_host_chunked(nets, streams, self.chunks, n, ip, op),
                      "run_host_chunked")
        return outputs


def compile_model(manifest, weights, options=None, devices=None, host_chunks=None, **kw):
    """pkg/src/nnjit/runtime.py:101-104.  ``devices=[...]`` (additive) shards
    ``batch`` over one replica per listed GPU (``replicas.MultiDeviceNetwork``);
    ``host_chunks=k`` (additive) returns a ``PipelinedNetwork`` whose
    ``run_host`` overlaps the host copies of k batch chunks with compute."""
    if devices is not None:
        from .replicas import MultiDeviceNetwork
        return MultiDeviceNetwork(manifest, weights, options, devices=devices, **kw)
    if host_chunks is not None:
        return PipelinedNetwork(manifest, weights, options, chunks=host_chunks, **kw)
    return CompiledNetwork(manifest, weights, options, **kw)


def compile_file(manifest_path, blob_path=None, options=None, devices=None, host_chunks=None,
                 **kw):
    """pkg/src/nnjit/runtime.py:105-107 (same ``devices`` / ``host_chunks``
    extensions)."""
    manifest, weights = load_model(manifest_path, blob_path)
    return compile_model(manifest, weights, options, devices=devices, host_chunks=host_chunks,
                         **kw)
