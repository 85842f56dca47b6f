#!/bin/bash
# build, run the GPU tests matching a -k expression, then A/B keyword variants
# on several configs:  gpu_ab.sh 'PYTEST_K' 'VARIANT_A' 'VARIANT_B' "cfg batch" ...
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
k=$1; va=$2; vb=$3; shift 3
if [ -n "$k" ]; then timeout 900 python -m pytest tests -m gpu -q -x -k "$k" 2>&1 | tail -15; fi
for cb in "$@"; do echo "== cfg/batch $cb"; timeout 300 python scripts/ab_kw.py $cb "$va" "$vb" 2>&1; done
