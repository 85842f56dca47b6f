"""The reference's own CPU path as the measured baseline (TEST / BENCH INFRASTRUCTURE ONLY).

Only bench.py's ``cpu_baseline`` and ``--impl reference`` legs (and tests/)
may import this module; nothing under ``paper_1906_05737_b200/`` does.

``build_ref()`` installs the UNMODIFIED reference package (``nnjit``,
/root/reference/pkg) into ``oracle/_ref`` with pip from a /tmp copy (the
source tree is read-only; the build writes ``build/`` and ``*.egg-info``).
``oracle/_ref`` is git-ignored but travels to the GPU box with the gpurun
snapshot, so the box -- which has no /root/reference -- runs the reference's
stock compiled path: ``nnjit.CompiledNetwork`` (pkg/src/nnjit/runtime.py:33-107)
generating SSE4.1 x86-64 code for its host CPU.

Protocol:

* nets: the BASELINE configs in the reference's vocabulary
  (``zoo.build(cfg, reference_compatible=True)``) with the cost stand-ins
  ELU -> tanh (cfg1), ReLU6 -> ReLU (cfg3), per-pixel softmax omitted (cfg4);
  default ``ApproximationOptions``;
* every ``apply()`` is preceded by a rewrite of the input view (the reference
  planner recycles the input's arena range, memory_planner.py:57-79);
* batch-1 latency: median of ``view[...] = x; apply()`` over >= ``seconds``
  after >= 10 warm-up calls, one thread;
* throughput: P = all usable host cores, one ``CompiledNetwork`` per worker.
  The workers are processes forked after ONE compile (each owns a private
  copy-on-write copy of the network: arena, pool and code mapping), which is
  the "one instance per thread" protocol without P serial compiles of the
  pure-Python compiler (cfg1 compiles in ~1.4 s); images/s = images / wall.
"""

import json
import multiprocessing as mp
import os
import pathlib
import shutil
import subprocess
import sys
import tempfile
import time

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REF_TARGET = HERE / "_ref"
REF_SRC = pathlib.Path("/root/reference/pkg")

_NET = None      # the compiled reference network inherited by forked workers
_X = None        # the worker's input images


def build_ref(force=False):
    """pip-install /root/reference/pkg into oracle/_ref (only where the
    reference exists, i.e. in the build container).  Returns the target or
    None when the reference is absent."""
    if not REF_SRC.exists():
        return REF_TARGET if (REF_TARGET / "nnjit").exists() else None
    stamp = REF_TARGET / ".installed"
    if stamp.exists() and not force:
        return REF_TARGET
    with tempfile.TemporaryDirectory() as tmp:
        src = pathlib.Path(tmp) / "pkg"
        shutil.copytree(REF_SRC, src, ignore=shutil.ignore_patterns("tests", "test_output.txt",
                                                                    "__pycache__"))
        if REF_TARGET.exists():
            shutil.rmtree(REF_TARGET)
        subprocess.check_call([sys.executable, "-m", "pip", "install", "--quiet", "--no-index",
                               "--no-build-isolation", "--no-deps", "--find-links",
                               "/opt/wheelhouse", "--target", str(REF_TARGET), str(src)])
    stamp.write_text("pip install --no-index --no-deps --target oracle/_ref /root/reference/pkg\n")
    return REF_TARGET


def nnjit():
    """The installed reference package (import from oracle/_ref)."""
    if not (REF_TARGET / "nnjit").exists():
        raise ImportError("oracle/_ref is not installed (run oracle.refbench.build_ref() where "
                          "/root/reference exists)")
    if str(REF_TARGET) not in sys.path:
        sys.path.insert(0, str(REF_TARGET))
    import nnjit as mod
    assert pathlib.Path(mod.__file__).resolve().is_relative_to(REF_TARGET.resolve()), mod.__file__
    return mod


def host_info():
    """CPU model and usable core count of this host."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    return {"cpu_model": model, "cores": cores, "machine": os.uname().machine}


def reference_model(cfg):
    """(manifest, weights) of BASELINE config ``cfg`` as reference objects,
    encoded in the reference vocabulary with BASELINE.md's stand-ins."""
    ref = nnjit()
    root = str(HERE.parent)
    if root not in sys.path:
        sys.path.insert(0, root)
    from paper_1906_05737_b200 import zoo
    from paper_1906_05737_b200.model_format import manifest_to_json
    m, _, arrays = zoo.build(cfg, reference_compatible=True, with_arrays=True)
    doc = manifest_to_json(m)
    rm = ref.parse_manifest(doc)
    refs = [r for l in rm.layers for r in l.weight_refs]
    blob = bytearray(max((r.offset + r.length for r in refs), default=0))
    for r in refs:
        blob[r.offset:r.offset + r.length] = np.asarray(arrays[r.name], "<f4").tobytes()
    return rm, ref.load_weights(rm, bytes(blob))


def compile_reference(cfg):
    """(CompiledNetwork of the reference, compile ms)."""
    ref = nnjit()
    m, w = reference_model(cfg)
    net = ref.CompiledNetwork(m, w, ref.ApproximationOptions())
    return net, net.compile_ms


def _inputs(cfg, n, seed=7):
    root = str(HERE.parent)
    if root not in sys.path:
        sys.path.insert(0, root)
    from paper_1906_05737_b200 import zoo
    return zoo.inputs(cfg, n, seed=seed)


def _loop(net, xs, n):
    view = net.input_views[0]
    k = len(xs)
    for i in range(n):
        view[...] = xs[i % k]
        net.apply()


def batch1_latency_us(cfg, seconds=2.0, warmup=10, net=None):
    """Median latency (µs) of ``view[...] = x; apply()`` on one thread."""
    if net is None:
        net, _ = compile_reference(cfg)
    xs = _inputs(cfg, 4)
    _loop(net, xs, warmup)
    view = net.input_views[0]
    times = []
    t_end = time.perf_counter() + seconds
    i = 0
    while time.perf_counter() < t_end or len(times) < 5:
        x = xs[i % len(xs)]
        t0 = time.perf_counter()
        view[...] = x
        net.apply()
        times.append(time.perf_counter() - t0)
        i += 1
    return float(np.median(times)) * 1e6, len(times)


def _worker(n):
    t0 = time.perf_counter()
    _loop(_NET, _X, n)
    return time.perf_counter() - t0


class Throughput:
    """P forked workers, each with its own copy of one compiled reference
    network.  ``step(images)`` runs ``images`` (split evenly) and returns
    images / wall seconds."""

    def __init__(self, cfg, procs=None):
        global _NET, _X
        self.cfg = cfg
        self.procs = procs or host_info()["cores"]
        _NET, self.compile_ms = compile_reference(cfg)
        _X = _inputs(cfg, 8)
        self.net = _NET
        self.pool = mp.get_context("fork").Pool(self.procs)
        self.pool.map(_worker, [2] * self.procs)          # warm every worker
        t0 = time.perf_counter()
        self.pool.map(_worker, [4] * self.procs)
        self.per_image_s = (time.perf_counter() - t0) / (4 * self.procs) * self.procs

    def images_for(self, seconds):
        """Images a step of about ``seconds`` processes (a multiple of P)."""
        n = int(seconds / max(self.per_image_s, 1e-9)) * self.procs
        return max(self.procs, n // self.procs * self.procs)

    def step(self, images):
        per = max(1, images // self.procs)
        t0 = time.perf_counter()
        self.pool.map(_worker, [per] * self.procs, chunksize=1)
        dt = time.perf_counter() - t0
        return per * self.procs / dt, per * self.procs, dt

    def close(self):
        self.pool.close()
        self.pool.join()


def interpreter_one_image_ms(cfg):
    """The reference interpreter (oracle A, pkg/src/nnjit/interpreter.py) on
    one image -- the secondary figure of BASELINE.md section 2."""
    ref = nnjit()
    m, w = reference_model(cfg)
    g = ref.build_graph(m, w)
    x = _inputs(cfg, 1)[0]
    t0 = time.perf_counter()
    ref.interpret(g, [x])
    return (time.perf_counter() - t0) * 1e3


STAND_INS = {0: "none", 1: "ELU -> tanh", 2: "none", 3: "ReLU6 -> ReLU",
             4: "per-pixel softmax omitted"}


if __name__ == "__main__":
    build_ref(force="--force" in sys.argv)
    print(json.dumps({"installed": str(REF_TARGET), **host_info()}))
