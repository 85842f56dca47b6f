"""compile() wall time per BASELINE config: cold (no cubin cache, every
kernel through NVRTC) and warm (cubin cache hit), batch as in the bench."""
import sys, pathlib, tempfile, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_1906_05737_b200 import EXACT, compile_model, zoo
BATCH = {0: 4096, 1: 65536, 2: 1024, 3: 256, 4: 64}
with tempfile.TemporaryDirectory() as d:
    for cfg, b in BATCH.items():
        m, w = zoo.build(cfg)
        t0 = time.perf_counter()
        net = compile_model(m, w, EXACT, batch=b, cache_dir=d)
        cold = (time.perf_counter() - t0) * 1e3
        t0 = time.perf_counter()
        net2 = compile_model(m, w, EXACT, batch=b, cache_dir=d)
        warm = (time.perf_counter() - t0) * 1e3
        print(f"cfg{cfg}: {len(net.artifact.kernel_names)} kernels, cold {cold:.0f} ms "
              f"(nvrtc {net.compile_ms:.0f} ms), warm {warm:.0f} ms")
