#!/bin/bash
# Round-2 GPU check: FFMA peak probe, GPU test-suite, bench line.
# usage: gpurun -- bash scripts/gpu_round2.sh <tag>
tag=${1:-r2}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
lscpu > $out/lscpu.txt 2>&1
python -c "
from paper_1906_05737_b200 import _native
import json
tf, ms = _native.ffma_peak(0, 4096)
print(json.dumps({'ffma_tflops': tf, 'ms': ms}))
" > $out/ffma.json 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $out/gpu_tests.log 2>&1
echo "tests rc=$?" >> $out/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err
echo "bench rc=$?" >> $out/bench.err
