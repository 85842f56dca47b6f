#!/bin/bash
# A/B runs of scripts/ab_kw.py: gpurun -- bash scripts/gpu_ab.sh TAG 'CFG BATCH' 'variant' ... -- 'CFG BATCH' ...
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
i=0
while [ $# -gt 0 ]; do
  cb=$1; shift; vars=()
  while [ $# -gt 0 ] && [ "$1" != "--" ]; do vars+=("$1"); shift; done
  [ "$1" == "--" ] && shift
  i=$((i+1))
  timeout 900 python scripts/ab_kw.py $cb "${vars[@]}" > $out/ab_$i.log 2>&1; echo "rc=$?" >> $out/ab_$i.log
done
