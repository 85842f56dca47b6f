#!/usr/bin/env python3
"""Benchmark of the B200 CompiledNN path (contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl nnb|reference]
                    [--config C] [--batch B] [--global-batch G]
                    [--options default|exact] [--no-extra]

Workload: BASELINE.json configs[1] (the dense MLP, 1024 -> 512 tanh -> 256
sigmoid -> 128 elu -> 10 softmax) at batch 65536 per GPU, FP32 in and out,
the reference's DEFAULT ApproximationOptions (rational tanh/sigmoid, fast
softmax exp: pkg/src/nnjit/options.py:9-27 -- the options the reference arm
runs too; ``--options exact`` for interpreter-grade transcendentals).  A
*step* is one ``apply()`` -- one CUDA-graph replay of the whole network over
the batch already resident in HBM.  Inputs (256 MiB per GPU) are larger than
the 126 MB L2, so no flush is needed between steps (smaller batches flush L2
before every timed replay).  N GPUs run N independent replicas with no
collective on the data path; the time is the max over ranks.  Weak scaling by
default (B images per GPU); ``--global-batch G`` shards G images over the
ranks instead (strong scaling, BASELINE configs[3] and [4]: cfg3 @256, cfg4
@64 over 1/2/4/8 GPUs).

Keys beyond the base contract:
  e2e          the same metric through ``compile_model(host_chunks=8).run_host``
               (the C-ABI host-buffer call): H2D of the step's inputs from
               pinned memory, replay, D2H of the outputs, every step.
  roofline     dominant kernel: algorithmic work per launch / its CUDA-event
               time against its own pipe (roofline.py: tcgen05 -> TF32 = half
               the measured bf16 rate x products per MAC; FFMA -> the measured
               FFMA peak; HBM -> measured copy bandwidth).
  launches     every launch of the step: pipe, algorithmic flops / bytes, roof
               and measured µs, fraction.
  cpu_baseline the unmodified reference (oracle/_ref nnjit.CompiledNetwork) on
               all host cores over a bounded sample; the C port of its
               interpreter as a secondary figure.
  parity       sampled images of the timed batch vs the oracle on EVERY rank;
               a failure marks the line invalid and exits 1.
  configs      all five BASELINE configs: batch-1 latency and large-batch
               throughput (L2 flushed between timed replays), per-launch
               roofline fractions, the reference's CPU batch-1 latency.
"""

import argparse
import json
import os
import sys
import pathlib
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

RTOL, ATOL = 1e-4, 1e-5           # BASELINE.json north_star FP32 tolerance
ARITHMETIC = ("FP32 in HBM, FP32 FFMA kernels; tcgen05 GEMMs (Dense, 1x1 and KxK convs above "
              "the selection thresholds) as a 3xTF32 split a_hi*b_hi + a_hi*b_lo + a_lo*b_hi "
              "with FP32 accumulation in TMEM (chunked every 16 k-blocks); N=256 row tiles form "
              "the two correction products as one BF16 K=16 MMA.  Stated bound per output: "
              "|d| <= 1e-4|ref| + 1e-5 + 2^-19 sum|a_k b_k| (TF32 split), + 2^-17 sum|a_k b_k| "
              "(BF16 correction) -- DESIGN.md section 4; every bench/test case passes the "
              "plain FP32 gate")
METRIC = "images/sec per net (batch-1 latency + batched) at 1/2/4/8 B200; % roofline"
BIG_BATCH = {0: 4096, 1: 65536, 2: 1024, 3: 256, 4: 64}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="nnb", choices=("nnb", "reference"))
    p.add_argument("--config", type=int, default=1)
    p.add_argument("--batch", type=int, default=None)
    p.add_argument("--global-batch", type=int, default=None,
                   help="strong scaling: shard this many images over the ranks")
    p.add_argument("--options", default="default", choices=("default", "exact"))
    p.add_argument("--no-extra", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    return p.parse_args()


def options(args):
    from paper_1906_05737_b200 import EXACT, ApproximationOptions
    return EXACT if args.options == "exact" else ApproximationOptions()


def options_desc(opts):
    return (f"activation_mode={opts.activation_mode} softmax_exp={opts.softmax_exp}"
            + (" (the reference's defaults)" if (opts.activation_mode, opts.softmax_exp)
               == ("rational", "fast") else " (interpreter-grade: float64 rounded once)"))


class ClockSampler:
    """NVML SM-clock / throttle-reason sampler for the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting"}

    def __init__(self, index, period=0.005):
        self.index, self.period = index, period
        self.mhz, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _loop(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.mhz.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.mhz:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.mhz)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.mhz)}


def dist_setup(gpus):
    """One process per GPU (torchrun).  The data path has no collective; the
    process group only carries the barrier and the MAX of per-rank device
    time, so it runs over NCCL when every rank owns a GPU and over gloo
    otherwise (e.g. a functional check with several ranks on one device)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        import torch
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        ndev = max(torch.cuda.device_count(), 1) if torch.cuda.is_available() else 1
        own = ndev >= int(os.environ.get("LOCAL_WORLD_SIZE", world))
        local = local % ndev
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        if own and torch.cuda.is_available():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, value, local):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    dev = f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_port(cfg, batch, seconds, opts, threads=None):
    """The C restatement of the reference interpreter (oracle/nnoracle.c) on
    host threads over a bounded sample -- the secondary CPU figure.
    Returns (images/s, sample images, threads, seconds)."""
    from oracle import oracle
    from paper_1906_05737_b200 import zoo
    from paper_1906_05737_b200.graph import build_graph
    threads = threads or os.cpu_count() or 1
    g = build_graph(*zoo.build(cfg))
    probe = max(threads, 1)
    x = zoo.inputs(cfg, probe, seed=7)
    t0 = time.perf_counter()
    oracle.run_graph(g, [x], opts, threads)
    per_img = (time.perf_counter() - t0) / probe
    sample = int(min(batch, max(probe, seconds / max(per_img, 1e-9))))
    sample = max(threads, sample // threads * threads)
    x = zoo.inputs(cfg, sample, seed=7)
    t0 = time.perf_counter()
    oracle.run_graph(g, [x], opts, threads)
    dt = time.perf_counter() - t0
    return sample / dt, sample, threads, dt


def oracle_check(cfg, xs, got, opts):
    """The sampled GPU outputs against the oracle on the same images and the
    same approximation options (the oracle's use here: the checker)."""
    from oracle import oracle
    from paper_1906_05737_b200 import zoo
    from paper_1906_05737_b200.graph import build_graph
    want = oracle.run_graph(build_graph(*zoo.build(cfg)), [xs], opts)[0]
    return {"images": len(xs), "max_abs": float(np.abs(got - want).max()),
            "ok": bool(np.allclose(got, want, rtol=RTOL, atol=ATOL)),
            "tolerance": f"rtol {RTOL:g} / atol {ATOL:g} vs oracle/nnoracle.c with the same "
                         "ApproximationOptions (models of pkg/src/nnjit/codegen/approx.py)"}


def reference_cpu(cfg, seconds, steps=1, warmup=0):
    """The reference's own compiled x86 path (oracle/_ref: the unmodified
    nnjit package, CompiledNetwork, default options, BASELINE.md stand-ins)
    on every usable host core, one network per forked worker.  Returns
    (per-step images/s list, images per step, info) or None when oracle/_ref
    is not installed."""
    from oracle import refbench
    try:
        refbench.nnjit()
    except ImportError:
        return None
    tp = refbench.Throughput(cfg)
    try:
        n = tp.images_for(seconds)
        vals = []
        for i in range(warmup + steps):
            v, n_done, _ = tp.step(n)
            if i >= warmup:
                vals.append(v)
    finally:
        tp.close()
    info = {**refbench.host_info(), "workers": tp.procs, "compile_ms": tp.compile_ms,
            "stand_ins": refbench.STAND_INS[cfg]}
    return vals, n_done, info


def reference_extras(seconds=2.0):
    """Batch-1 latency of the reference's compiled path for all five configs
    (median over >= ``seconds``), its compile time and the interpreter on one
    image."""
    from oracle import refbench
    from paper_1906_05737_b200 import zoo
    out = {}
    for c in range(5):
        try:
            net, cms = refbench.compile_reference(c)
            us, calls = refbench.batch1_latency_us(c, seconds, net=net)
            out[zoo.CONFIGS[c]["name"]] = {
                "batch1_latency_us": us, "calls": calls, "compile_ms": cms,
                "interpreter_one_image_ms": refbench.interpreter_one_image_ms(c),
                "stand_ins": refbench.STAND_INS[c]}
        except Exception as e:  # report, never hide
            out[zoo.CONFIGS[c]["name"]] = {"error": repr(e)[:300]}
    return out


def reference_arm(args, world, rank):
    """``--impl reference``: the reference's own CPU implementation of the
    path on this host, on this arm's config / metric (rank 0 only)."""
    if rank != 0:
        return
    cfg = args.config
    batch = args.batch or BIG_BATCH[cfg]
    from paper_1906_05737_b200 import zoo
    budget = min(5.0, max(1.0, 120.0 / max(1, args.steps + args.warmup)))
    got = reference_cpu(cfg, budget, args.steps, args.warmup)
    if got is not None:
        vals, sample, info = got
        kind, cores = "reference", info["workers"]
        what = (f"{sample} images of {zoo.CONFIGS[cfg]['name']} per step through the unmodified "
                f"reference (oracle/_ref nnjit.CompiledNetwork, SSE4.1 code, default options, "
                f"stand-in: {info['stand_ins']}), {cores} forked workers x one network each, input "
                f"view rewritten before every apply()")
    else:   # oracle/_ref absent: the C restatement of the interpreter
        vals, sample, threads = [], None, None
        for i in range(args.warmup + args.steps):
            v, sample, threads, _ = cpu_port(cfg, batch, budget, options(args))
            if i >= args.warmup:
                vals.append(v)
        kind, cores, info = "port", threads, {}
        what = (f"{sample} images of {zoo.CONFIGS[cfg]['name']} per step through "
                "oracle/nnoracle.c (reference interpreter restated; oracle/_ref not installed)")
    v = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sample / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, BASELINE.md section 2)",
        "config": {"workload": zoo.CONFIGS[cfg]["name"], "global_batch": batch,
                   "parallelism": f"{cores} host workers", "sample_images_per_step": sample},
        "cpu_baseline": {"value": v, "unit": "images/s", "cores": cores, "kind": kind,
                         "sample": what, **info},
        "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if kind == "reference" and not args.no_extra:
        line["configs"] = reference_extras()
    print(json.dumps(line), flush=True)


def ncu_traffic(kernel):
    """dram read + write bytes per launch of `kernel` from a committed
    `ncu --set full` capture (profiles/*_ncu_raw.csv: one row per launch), or
    None when no capture of that kernel is committed."""
    import csv
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    # kernel names end in a schedule index (nnb_u<unit>_<kind>_<i>); a capture
    # matches when the unit and kind agree
    stem = lambda k: k.rsplit("_", 1)[0]
    for p in sorted((pathlib.Path(ROOT) / "profiles").glob("*_ncu_raw.csv"), reverse=True):
        try:
            rows = list(csv.reader(open(p)))
            h, units = rows[0], rows[1]
            for v in rows[2:]:
                if stem(v[h.index("Kernel Name")].strip('"')) != stem(kernel):
                    continue
                tot = sum(float(v[h.index(m)].replace(",", "")) * scale[units[h.index(m)]]
                          for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
                return {"traffic": tot,
                        "traffic_source": f"profiles/{p.name} (ncu --set full, one launch)"}
        except (OSError, ValueError, IndexError, KeyError):
            continue
    return {"traffic": None}


def flush_l2(buf):
    buf.zero_()


def time_config(cfg, batch, device, torch, opts, iters=20):
    """(ms per replay with L2 flushed before each, net)."""
    from paper_1906_05737_b200 import compile_model, zoo
    m, w = zoo.build(cfg)
    net = compile_model(m, w, opts, batch=batch, device=device)
    net.input_views[0].copy_(torch.from_numpy(zoo.inputs(cfg, batch)))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=device)   # 256 MiB > L2
    for _ in range(3):
        net.apply()
    torch.cuda.synchronize(device)
    times = []
    s = torch.cuda.current_stream(device)
    for _ in range(iters):
        flush_l2(flush)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        net.apply()
        e1.record(s)
        torch.cuda.synchronize(device)
        times.append(e0.elapsed_time(e1))
    return float(np.median(times)), net


def dominant_roofline(net, B, lt, peaks, ffma):
    """The `roofline` object of the launch with the largest share of the pass."""
    from paper_1906_05737_b200 import roofline
    dom = max(lt, key=lt.get)
    L = net.artifact.launches[dom]
    r = roofline.launch_roofline(net.plan.units[L.unit], L, B, peaks, ffma[0])
    t = lt[dom] / 1e3
    share = lt[dom] / sum(lt.values())
    if r["bound"] == "hbm":
        achieved = r["bytes"] / t / 1e9
        roof = {"bound": "hbm", "unit": "GB/s", "achieved": achieved, "peak": peaks["hbm_gbs"],
                "frac": achieved / peaks["hbm_gbs"],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"}
    elif r["pipe"] == "tensor":
        achieved = r["products_per_mac"] * r["flops"] / t / 1e12
        roof = {"bound": "tensor", "unit": "TFLOP/s", "achieved": achieved,
                "peak": r["peak_tflops"], "frac": achieved / r["peak_tflops"],
                "peak_source": "dense TF32 = MEASURED_PEAKS.json bf16_tflops / 2 "
                               f"({peaks['bf16_tflops']} / 2)",
                "achieved_counts": (f"{r['products_per_mac']} x 2MNK TF32-equivalent tensor "
                                    "flops per launch ("
                                    + ("1 TF32 product a_hi*b_hi + the two correction products "
                                       "as one BF16 K=16 MMA" if r["products_per_mac"] == 2
                                       else "3xTF32 split") + ")"),
                "fp32_equivalent_tflops": r["flops"] / t / 1e12}
    else:
        achieved = r["flops"] / t / 1e12
        roof = {"bound": "fp32_ffma", "unit": "TFLOP/s", "achieved": achieved,
                "peak": ffma[0], "frac": achieved / ffma[0], "peak_source": ffma[1]}
    roof.update({"kernel": L.kernel, "algorithmic_per_launch": {"flops": r["flops"],
                                                               "bytes": r["bytes"]},
                 "kernel_ms": lt[dom], "share_of_step": share,
                 "hbm_frac_at_same_time": r["bytes"] / t / 1e9 / peaks["hbm_gbs"],
                 "timing": "CUDA events between consecutive launches of full passes on the "
                           "launching stream (nnb_time_sequence), mean over the step count",
                 **ncu_traffic(L.kernel)})
    return roof


def launch_table(net, B, lt, peaks, ffma):
    from paper_1906_05737_b200 import roofline
    rows, roof_us = roofline.net_roofline(net, B, peaks, ffma[0], lt)
    meas_us = sum(r.get("measured_us", 0.0) for r in rows)
    return rows, roof_us, meas_us


def main():
    args = parse()
    world, rank, local = dist_setup(args.gpus)
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return
    import torch
    from paper_1906_05737_b200 import _native, compile_model, roofline, zoo
    from paper_1906_05737_b200.planner import build_reference_plan
    from paper_1906_05737_b200.graph import build_graph
    from paper_1906_05737_b200.replicas import shard

    opts = options(args)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = args.config
    if args.global_batch:
        start, B = shard(args.global_batch, world, rank)
        scaling, G = "strong", args.global_batch
    else:
        B = args.batch or BIG_BATCH[cfg]
        start, scaling, G = rank * B, "weak", world * B
    m, w = zoo.build(cfg)
    net = compile_model(m, w, opts, batch=B, device=local)
    x = zoo.inputs(cfg, B, seed=1 + rank)
    net.input_views[0].copy_(torch.from_numpy(x))
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        net.apply()
    torch.cuda.synchronize(dev)
    flush = None
    if x.nbytes < 126e6:
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MiB

    # ---------------- timed region: K replays, inputs resident --------------
    barrier(world)
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        if flush is None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                net.apply()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1)
        else:   # inputs smaller than L2: flush before every replay, time replays only
            ms = 0.0
            for _ in range(args.steps):
                flush_l2(flush)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                net.apply()
                e1.record(stream)
                torch.cuda.synchronize(dev)
                ms += e0.elapsed_time(e1)
    barrier(world)
    ms = max_over_ranks(world, ms, local)
    ms_step = ms / args.steps
    value = G * args.steps / (ms / 1e3)
    n_launch = len(net.launches_for(B))

    # ---------------- parity: sampled images of this batch, every rank -------
    idx = np.unique(np.linspace(0, B - 1, min(B, 16)).astype(int))
    got = net.output_views[0][torch.as_tensor(idx, device=dev)].cpu().numpy()
    parity = oracle_check(cfg, x[idx], got, opts)
    ok = max_over_ranks(world, 0.0 if parity["ok"] else 1.0, local) == 0.0
    parity["ranks_ok"] = ok

    # ---------------- e2e through the C-ABI host-buffer call ----------------
    from paper_1906_05737_b200 import pinned_empty
    hx = pinned_empty(x.shape)
    hx[...] = x
    hy = pinned_empty((B,) + tuple(net.output_views[0].shape[1:]))
    e2e_steps = max(3, min(args.steps, 10))
    # the public host-buffer call for a large batch: compile_model(...,
    # host_chunks=8) -> PipelinedNetwork.run_host -> nnb_run_host_chunked
    # (chunk j's H2D overlaps chunk j-1's replay + D2H; 8 chunks measured
    # best: 1 / 2 / 4 / 8 / 16 -> 12.3 / 12.8 / 13.0 / 13.0 / 12.9 M img/s)
    chunks = 8 if B >= 8192 else 1
    pnet = compile_model(m, w, opts, batch=B, device=local, host_chunks=chunks)
    pnet.run_host([hx], [hy])
    # same outputs as the resident-input path (checked on the sampled images)
    np.testing.assert_allclose(hy[idx], got, rtol=RTOL, atol=ATOL)
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        pnet.run_host([hx], [hy])
    e2e_s = max_over_ranks(world, time.perf_counter() - t0, local)
    e2e = {"value": G * e2e_steps / e2e_s, "unit": "images/s",
           "h2d_bytes_per_step": int(hx.nbytes), "d2h_bytes_per_step": int(hy.nbytes),
           "path": f"compile_model(host_chunks={chunks}).run_host -> nnb_run_host_chunked "
                   f"(pinned host buffers, {chunks} chunk(s) on {chunks} stream(s))"}
    del pnet

    # ---------------- roofline of the dominant kernel + every launch --------
    peaks = roofline.measured_peaks()
    ffma = roofline.ffma_peak_tflops(_native.ffma_peak(local, 4096)[0])
    # per-launch CUDA-event durations inside full passes (same order, same
    # inputs as the timed replays, events between consecutive launches)
    lt = net.time_sequence(B, iters=max(3, args.steps))
    roof = dominant_roofline(net, B, lt, peaks, ffma)
    rows, roof_us, meas_us = launch_table(net, B, lt, peaks, ffma)
    clocks = clk.summary()

    # ---------------- per-config extras (rank 0, N == 1) ---------------------
    extra = None
    cpu = None
    if rank == 0 and world == 1:
        ref = reference_cpu(cfg, min(10.0, args.cpu_seconds))
        c_val, c_n, c_thr, c_dt = cpu_port(cfg, B, min(5.0, args.cpu_seconds), opts)
        port = {"value": c_val, "unit": "images/s", "cores": c_thr,
                "sample": f"{c_n} images through oracle/nnoracle.c (the reference interpreter "
                          f"restated in C, {options_desc(opts)}) in {c_dt:.1f} s"}
        if ref is not None:
            vals, n_ref, info = ref
            cpu = {"value": float(np.mean(vals)), "unit": "images/s", "cores": info["workers"],
                   "kind": "reference",
                   "sample": f"{n_ref} images of {zoo.CONFIGS[cfg]['name']} through the "
                             "unmodified reference (oracle/_ref nnjit.CompiledNetwork, SSE4.1, "
                             f"default options, stand-in: {info['stand_ins']}), "
                             f"{info['workers']} forked workers x one network",
                   "cpu_model": info["cpu_model"], "secondary_port": port}
        else:
            cpu = dict(port, kind="port")
        ref_b1 = {}
        if not args.no_extra and ref is not None:
            ref_b1 = reference_extras(seconds=1.0)
        if not args.no_extra:
            extra = {}
            for c in range(5):
                name = zoo.CONFIGS[c]["name"]
                try:
                    big = BIG_BATCH[c]
                    ms_b, netb = time_config(c, big, local, torch, opts)
                    ms_1, net1 = time_config(c, 1, local, torch, opts, iters=50)
                    ltb = netb.time_sequence(big, iters=5)
                    rws, r_us, m_us = launch_table(netb, big, ltb, peaks, ffma)
                    rp = build_reference_plan(build_graph(*zoo.build(c)))
                    t_s = roofline.survey_layerwise_roof_s(rp, big, peaks["hbm_gbs"],
                                                           roofline.fp32_peak_tflops())
                    lr_us, _ = roofline.layer_roofline(netb, rp, big, peaks, ffma[0])
                    # cold compile(): NVRTC of every kernel of a replay over `big` images, no cubin cache
                    cold = compile_model(*zoo.build(c), opts, batch=big, device=local, cache_dir="")
                    cold_ms = cold.compile_ms
                    del cold
                    e = {"batch": big, "ms": ms_b, "images_per_s": big / (ms_b / 1e3),
                         "batch1_latency_us": ms_1 * 1e3,
                         "launches": len(netb.launches_for(big)),
                         "roof_us": r_us, "roofline_frac": r_us / (ms_b * 1e3),
                         "layer_roof_us": lr_us, "layer_roofline_frac": lr_us / (ms_b * 1e3),
                         "sum_launch_us": m_us,
                         "launch_rows": [{k: (round(v, 3) if isinstance(v, float) else v)
                                          for k, v in r.items()} for r in rws],
                         "survey_ffma_only_frac": t_s * 1e3 / ms_b,
                         "gflop_per_batch": big * roofline.total_flops(rp) / 1e9,
                         "compile_ms": netb.compile_ms, "cold_compile_ms": cold_ms}
                    if name in ref_b1 and "batch1_latency_us" in ref_b1[name]:
                        e["reference_cpu"] = ref_b1[name]
                        e["batch1_speedup_vs_reference_cpu"] = (
                            ref_b1[name]["batch1_latency_us"] / e["batch1_latency_us"])
                    extra[name] = e
                    del netb, net1
                except Exception as ex:  # report, never hide
                    extra[name] = {"error": repr(ex)[:300]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded weights/inputs, BASELINE.md section 2)",
            "config": {"workload": zoo.CONFIGS[cfg]["name"], "global_batch": G,
                       "per_gpu_batch": B, "parallelism": f"replicas x{world}",
                       "l2": "inputs larger than L2 (no flush)" if flush is None
                       else "L2 flushed (256 MiB write) before every timed replay",
                       "options": options_desc(opts), "arithmetic": ARITHMETIC},
            "e2e": e2e, "gpu_launches": n_launch * args.steps, "clocks": clocks,
            "roofline": roof, "step_roofline": {"roof_us": roof_us, "sum_launch_us": meas_us,
                                                "frac": roof_us / (ms_step * 1e3)},
            "launches": [{k: (round(v, 3) if isinstance(v, float) else v)
                          for k, v in r.items()} for r in rows],
            "ffma_peak": {"tflops": ffma[0], "source": ffma[1]},
            "cpu_baseline": cpu, "parity": parity,
            "compile_ms": net.compile_ms, "configs": extra,
        }
        if not ok:
            line["invalid"] = "parity check against the oracle failed on at least one rank"
        import torch as _t
        if world > max(1, _t.cuda.device_count()):
            # several ranks on one device: their replays time-slice the GPU, so
            # per-rank device times do not add up to a job rate
            line["config"]["note"] = (f"{world} ranks share {_t.cuda.device_count()} GPU(s): "
                                      "functional check only, value is not a throughput")
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    if not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
