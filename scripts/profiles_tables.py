"""Markdown tables for profiles/README.md from a committed bench line, so the
README's numbers are the bench line's numbers.

    python scripts/profiles_tables.py profiles/r02_bench.json profiles/r02_bench_reference.json
"""
import json
import sys


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def main(bench, ref=None):
    d = last_json(bench)
    r = last_json(ref) if ref else None
    e2e = d["e2e"]
    rl = d["roofline"]
    print(f"## Headline: cfg1 @ {d['config'].get('global_batch', 65536)}\n")
    print(f"`bench.py`: {d['ms_per_step'] * 1e3:.1f} µs/step = {d['value'] / 1e6:.1f} M images/s "
          f"(clocks {d['clocks']['sm_mhz']:.0f} MHz, reasons {d['clocks']['reasons'] or 'none'}); "
          f"e2e {e2e['value'] / 1e6:.2f} M images/s ({e2e['h2d_bytes_per_step'] / 1e6:.0f} MB H2D + "
          f"{e2e['d2h_bytes_per_step'] / 1e6:.1f} MB D2H per step).")
    if r:
        print(f"Reference arm: {r['value'] / 1e3:.1f} K images/s ({r['cpu_baseline']['sample']}).")
    print(f"Dominant kernel `{rl['kernel']}`: {rl['kernel_ms'] * 1e3:.1f} µs in-bench, "
          f"{rl['achieved']:.0f} {rl['unit']} = **{rl['frac']:.2f}** of {rl['peak']:.0f}; "
          f"share of step {rl['share_of_step']:.2f}; DRAM traffic {rl['traffic'] / 1e6:.0f} MB vs "
          f"{rl['algorithmic_per_launch']['bytes'] / 1e6:.0f} MB algorithmic.\n")
    print("| config | batch | ms | images/s | roof µs | roofline frac (per fused launch) | per-layer roof µs "
          "| frac of the per-layer roofline | launches | batch-1 µs (L2 flushed) "
          "| reference CPU batch-1 µs | speed-up at batch 1 | cold compile() ms (no cubin cache) "
          "| reference compile ms |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for name, v in d["configs"].items():
        rc = (r or {}).get("configs", {}).get(name, {}) if r else {}
        rb1 = rc.get("batch1_latency_us") or (v.get("reference_cpu") or {}).get("batch1_latency_us")
        tail = f"{rb1:.1f} | {rb1 / v['batch1_latency_us']:.2f}" if rb1 else "— | —"
        print(f"| {name} | {v['batch']} | {v['ms']:.4f} | {v['images_per_s'] / 1e6:.3f} M | {v['roof_us']:.1f} "
              f"| {v['roofline_frac']:.3f} | {v.get('layer_roof_us', float('nan')):.1f} "
              f"| {v.get('layer_roofline_frac', float('nan')):.3f} | {v['launches']} "
              f"| {v['batch1_latency_us']:.1f} | {tail} | {v.get('cold_compile_ms', float('nan')):.0f} "
              f"| {(v.get('reference_cpu') or {}).get('compile_ms', float('nan')):.0f} |")
    for name, v in d["configs"].items():
        print(f"\n### {name} @ {v['batch']}: replay {v['ms'] * 1e3:.1f} µs, roof {v['roof_us']:.1f} µs\n")
        print("| launch | pipe | GFLOP | MB | roof µs (bound) | measured µs | frac |")
        print("|---|---|---|---|---|---|---|")
        for l in v["launch_rows"]:
            pipe = l["pipe"] if l["pipe"] != "tensor" else f"tensor x{l['products_per_mac']}"
            print(f"| `{l['kernel']}` | {pipe} | {l['flops'] / 1e9:.2f} | {l['bytes'] / 1e6:.1f} "
                  f"| {l['roof_us']:.1f} ({'compute' if l['bound'] != 'hbm' else 'hbm'}) "
                  f"| {l['measured_us']:.1f} | {l['frac']:.2f} |")


if __name__ == "__main__":
    main(*sys.argv[1:])
