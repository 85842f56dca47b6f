#!/usr/bin/env python3
"""Benchmark of the B200 CompiledNN path (contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl nnb|reference]
                    [--config C] [--batch B] [--no-extra]

Workload: BASELINE.json configs[1] (the dense MLP, 1024 -> 512 tanh -> 256
sigmoid -> 128 elu -> 10 softmax) at batch 65536 per GPU, FP32 in and out,
exact (interpreter-grade) transcendentals.  A *step* is one ``apply()`` --
one CUDA-graph replay of the whole network over the batch already resident
in HBM.  Inputs (256 MiB per GPU) are larger than the 126 MB L2, so no flush
is needed between steps.  N GPUs run N independent replicas (weak scaling,
no collective on the data path); the time is the max over ranks.

Keys beyond the base contract:
  e2e          the same metric through ``CompiledNetwork.run_host`` (the C-ABI
               host-buffer call): H2D of the step's inputs from pinned memory,
               replay, D2H of the softmax outputs, every step.
  roofline     dominant kernel: algorithmic FLOPs per launch / its CUDA-event
               time, against the FP32 FFMA peak (SIMT kernels) or TF32 tensor
               peak (tcgen05 kernels).
  cpu_baseline the C oracle (oracle/nnoracle.c, the reference interpreter
               restated) on all host threads over a bounded sample.
  parity       max |GPU - oracle| over sampled images of the timed batch
               (evaluated by the cpu_baseline leg, rank 0 at N=1).
  configs      all five BASELINE configs: batch-1 latency and large-batch
               throughput (L2 flushed between timed replays), fraction of the
               layerwise roofline of SURVEY.md 8(d).
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
    p.add_argument("--no-extra", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    return p.parse_args()


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


def cpu_reference(cfg, batch, seconds, threads=None, check=None):
    """Time the C oracle (reference interpreter restated) on host threads.
    Returns (images/s, sample images, threads, seconds, parity).  ``check`` =
    (inputs, gpu_outputs) of sampled images of the timed batch: the oracle
    also evaluates those, as the checker of the GPU outputs (the only other
    use of oracle/ in this file)."""
    from oracle import oracle
    from paper_1906_05737_b200 import zoo
    threads = threads or os.cpu_count() or 1
    m, w = zoo.build(cfg)
    from paper_1906_05737_b200.graph import build_graph
    g = build_graph(m, w)
    probe = max(threads, 1)
    x = zoo.inputs(cfg, probe, seed=7)
    t0 = time.perf_counter()
    oracle.run_graph(g, [x], "exact", threads)
    dt = time.perf_counter() - t0
    per_img = dt / probe
    sample = int(min(batch, max(probe, seconds / max(per_img, 1e-9))))
    sample = max(threads, sample // threads * threads)
    x = zoo.inputs(cfg, sample, seed=7)
    t0 = time.perf_counter()
    oracle.run_graph(g, [x], "exact", threads)
    dt = time.perf_counter() - t0
    parity = None
    if check is not None:
        xs, got = check
        want = oracle.run_graph(g, [xs], "exact", threads)[0]
        parity = {"images": len(xs), "max_abs": float(np.abs(got - want).max()),
                  "ok": bool(np.allclose(got, want, rtol=1e-4, atol=1e-5)),
                  "tolerance": "rtol 1e-4 / atol 1e-5 vs oracle/nnoracle.c (exact)"}
    return sample / dt, sample, threads, dt, parity


def reference_arm(args, world, rank):
    if rank != 0:
        return
    cfg = args.config
    batch = args.batch or BIG_BATCH[cfg]
    from paper_1906_05737_b200 import zoo  # noqa: F401
    vals = []
    sample = threads = None
    budget = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    for i in range(args.warmup + args.steps):
        v, sample, threads, _, _ = cpu_reference(cfg, batch, budget)
        if i >= args.warmup:
            vals.append(v)
    v = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sample / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, BASELINE.md section 2)",
        "config": {"workload": zoo.CONFIGS[cfg]["name"], "global_batch": batch,
                   "parallelism": "host threads", "sample_images_per_step": sample},
        "cpu_baseline": {"value": v, "unit": "images/s", "cores": threads, "kind": "port",
                         "sample": f"{sample} images of {zoo.CONFIGS[cfg]['name']} per step "
                                   "through oracle/nnoracle.c (reference interpreter "
                                   "restated, float32 per-op rounding)"},
        "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


_TF32 = {}


def ncu_traffic(kernel):
    """dram read + write bytes per launch of `kernel` from the committed
    `ncu --set full` capture (profiles/r01_dense_tc_ncu_raw.csv), or None."""
    import csv
    p = pathlib.Path(ROOT) / "profiles" / "r01_dense_tc_ncu_raw.csv"
    try:
        rows = list(csv.reader(open(p)))
        h, units, v = rows[0], rows[1], rows[2]
        # kernel names end in a schedule index (nnb_u<unit>_<kind>_<i>); the
        # capture matches when the unit and kind agree
        stem = lambda k: k.rsplit("_", 1)[0]
        if stem(v[h.index("Kernel Name")].strip('"')) != stem(kernel):
            return {"traffic": None}
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = sum(float(v[h.index(m)]) * scale[units[h.index(m)]]
                  for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        return {"traffic": tot, "traffic_source": f"{p.name} (ncu --set full, cold cache, one launch)"}
    except (OSError, ValueError, IndexError, KeyError):
        return {"traffic": None}


def measure_tf32_peak(torch, dev):
    """cuBLAS TF32 dense throughput on this GPU (the roofline denominator for
    the 3xTF32 tcgen05 kernels)."""
    if dev in _TF32:
        return _TF32[dev]
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device=dev)
        b = torch.randn(n, n, device=dev)
        for _ in range(2):
            a @ b
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            a @ b
            e1.record()
            torch.cuda.synchronize(dev)
            best = min(best, e0.elapsed_time(e1))
        _TF32[dev] = 2 * n ** 3 / (best / 1e3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return _TF32[dev]


def flush_l2(buf):
    buf.zero_()


def time_config(cfg, batch, device, torch, iters=20):
    """(ms per replay with L2 flushed before each, net)."""
    from paper_1906_05737_b200 import EXACT, compile_model, zoo
    m, w = zoo.build(cfg)
    net = compile_model(m, w, EXACT, batch=batch, device=device)
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


def main():
    args = parse()
    world, rank, local = dist_setup(args.gpus)
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return
    import torch
    from paper_1906_05737_b200 import EXACT, compile_model, roofline, zoo
    from paper_1906_05737_b200.planner import build_reference_plan
    from paper_1906_05737_b200.graph import build_graph

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = args.config
    B = args.batch or BIG_BATCH[cfg]
    m, w = zoo.build(cfg)
    net = compile_model(m, w, EXACT, batch=B, device=local)
    x = zoo.inputs(cfg, B, seed=1 + rank)
    net.input_views[0].copy_(torch.from_numpy(x))
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        net.apply()
    torch.cuda.synchronize(dev)

    # ---------------- timed region: K replays, inputs resident --------------
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            net.apply()
        e1.record(stream)
        torch.cuda.synchronize(dev)
    barrier(world)
    ms = max_over_ranks(world, e0.elapsed_time(e1), local)
    ms_step = ms / args.steps
    value = world * B * args.steps / (ms / 1e3)
    n_launch = len(net.launches_for(B))

    # sampled outputs of this batch (checked against the oracle on the
    # cpu_baseline leg, and against the e2e path below)
    idx = np.linspace(0, B - 1, 16).astype(int)
    got = net.output_views[0][torch.as_tensor(idx, device=dev)].cpu().numpy()
    parity = None

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
    pnet = compile_model(m, w, EXACT, batch=B, device=local, host_chunks=8)
    pnet.run_host([hx], [hy])
    # same outputs as the resident-input path (checked on the sampled images)
    np.testing.assert_allclose(hy[idx], got, rtol=1e-4, atol=1e-5)
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        pnet.run_host([hx], [hy])
    e2e_s = max_over_ranks(world, time.perf_counter() - t0, local)
    e2e = {"value": world * B * e2e_steps / e2e_s, "unit": "images/s",
           "h2d_bytes_per_step": int(hx.nbytes), "d2h_bytes_per_step": int(hy.nbytes),
           "path": "compile_model(host_chunks=8).run_host -> nnb_run_host_chunked (pinned host "
                   "buffers, 8 chunks on 8 streams)"}
    del pnet

    # ---------------- roofline of the dominant kernel -----------------------
    peaks = roofline.measured_peaks()
    # per-launch CUDA-event durations inside full passes (same order, same
    # inputs as the timed replays, events between consecutive launches)
    lt = net.time_sequence(B, iters=max(3, args.steps))
    dom = max(lt, key=lt.get)
    L = net.artifact.launches[dom]
    u = net.plan.units[L.unit]
    f, io, wb = roofline.unit_work(u)
    share = lt[dom] / sum(lt.values())
    clocks = clk.summary()
    peak_fp32 = roofline.fp32_peak_tflops()
    fp32_equiv = B * f / (lt[dom] / 1e3) / 1e12
    if "_tc_" in L.kernel:
        # 3xTF32: the tensor pipe executes three TF32 products per FP32 MAC;
        # with the BF16 correction split (note "bf16 corr") one TF32 product
        # plus one K = 16 BF16 MMA per tf32 k-step, which issues in the time of
        # a TF32 MMA (BF16 runs at 2x the TF32 rate): 2 TF32-equivalents
        cb16 = "bf16 corr" in L.note
        mult = 2 if cb16 else 3
        tf32 = measure_tf32_peak(torch, dev)
        achieved = mult * fp32_equiv
        roof = {"bound": "tensor", "kernel": L.kernel, "unit": "TFLOP/s",
                "achieved": achieved, "peak": tf32, "frac": achieved / tf32,
                "peak_source": "TF32 dense, cuBLAS fp32 matmul with allow_tf32 on this GPU "
                               "(8192^3, best of 5; MEASURED_PEAKS.json has bf16 only: "
                               f"{peaks['bf16_tflops']} TF/s)",
                "achieved_counts": ("2 x 2MNK TF32-equivalent tensor flops per launch (1 TF32 "
                                    "product a_hi*b_hi + the two correction products as one "
                                    "BF16 K=16 MMA = 2MNK TF32 + 4MNK BF16 flops)") if cb16
                else "3 x 2MNK tensor flops (3xTF32 split) per launch",
                "peak_note": "the live cuBLAS TF32 GEMM is the measured denominator (a good "
                             "kernel can read a little above it); nominal dense TF32 is "
                             "1100 TFLOP/s (B200_PROFILING.md)",
                "frac_of_nominal_tf32": achieved / 1100.0,
                "fp32_equivalent_tflops": fp32_equiv,
                "fp32_ffma_peak_tflops": peak_fp32}
    else:
        achieved = fp32_equiv
        roof = {"bound": "fp32_ffma", "kernel": L.kernel, "unit": "TFLOP/s",
                "achieved": achieved, "peak": peak_fp32, "frac": achieved / peak_fp32,
                "peak_source": "derived 148 SM x 128 FFMA lanes x 2 x 1965 MHz (no tensor "
                               "cores in this kernel)"}
    roof.update({"algorithmic_per_launch": {"flops": B * f, "bytes": B * io + wb},
                 "kernel_ms": lt[dom], "share_of_step": share,
                 "hbm_frac_at_same_time": (B * io + wb) / (lt[dom] / 1e3) / 1e9 / peaks["hbm_gbs"],
                 "launch_ms": {net.artifact.launches[i].kernel: v for i, v in lt.items()},
                 "timing": "CUDA events between consecutive launches of the pass, "
                           "mean over the step count",
                 **ncu_traffic(L.kernel)})

    # ---------------- per-config extras (rank 0, N == 1) ---------------------
    extra = None
    cpu = None
    if rank == 0 and world == 1:
        c_val, c_n, c_thr, c_dt, parity = cpu_reference(cfg, B, args.cpu_seconds,
                                                        check=(x[idx], got))
        cpu = {"value": c_val, "unit": "images/s", "cores": c_thr, "kind": "port",
               "sample": f"{c_n} images of {zoo.CONFIGS[cfg]['name']} through "
                         f"oracle/nnoracle.c in {c_dt:.1f} s"}
        if not args.no_extra:
            extra = {}
            for c in range(5):
                try:
                    big = BIG_BATCH[c]
                    ms_b, netb = time_config(c, big, local, torch)
                    ms_1, net1 = time_config(c, 1, local, torch, iters=50)
                    g = build_graph(*zoo.build(c))
                    rp = build_reference_plan(g)
                    t_roof = roofline.layerwise_roof_s(rp, big, peaks["hbm_gbs"], peak_fp32)
                    t_fused = roofline.fused_ideal_s(rp, big, peaks["hbm_gbs"], peak_fp32)
                    extra[zoo.CONFIGS[c]["name"]] = {
                        "batch": big, "ms": ms_b, "images_per_s": big / (ms_b / 1e3),
                        "batch1_latency_us": ms_1 * 1e3,
                        "launches": len(netb.launches_for(big)),
                        "layerwise_roof_ms": t_roof * 1e3,
                        "layerwise_roofline_frac": t_roof * 1e3 / ms_b,
                        "fused_ideal_frac": t_fused * 1e3 / ms_b,
                        "gflop_per_batch": big * roofline.total_flops(rp) / 1e9,
                        "compile_ms": netb.compile_ms,
                    }
                    del netb, net1
                except Exception as e:  # report, never hide
                    extra[zoo.CONFIGS[c]["name"]] = {"error": repr(e)[:300]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded weights/inputs, BASELINE.md section 2)",
            "config": {"workload": zoo.CONFIGS[cfg]["name"], "global_batch": world * B,
                       "per_gpu_batch": B, "parallelism": f"replicas x{world}",
                       "l2": "inputs larger than L2 (no flush)" if x.nbytes > 126e6
                       else "inputs smaller than L2",
                       "transcendentals": "exact mode (tanh/sigmoid/elu float64-rounded in "
                                          "FFMA kernels; FP32 within 2 ulp in tcgen05 epilogues)"},
            "e2e": e2e, "gpu_launches": n_launch * args.steps, "clocks": clocks,
            "roofline": roof, "cpu_baseline": cpu, "parity": parity,
            "compile_ms": net.compile_ms, "configs": extra,
        }
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


if __name__ == "__main__":
    main()
