#!/bin/bash
# NNB_TC_DBG ablation of a config's tcgen05 launches (bit 0 no MMAs, 1 no TMA loads, 2 no A split,
# 3 no TMEM reads, 4 no output path): where a launch's time goes.
# usage: gpurun -- bash scripts/gpu_dbg.sh CONFIG BATCH [BITS...]      (default bits: 1 2 4 8 16 7 24 31)
cfg=${1:-3}; batch=${2:-256}; shift 2
bits=${*:-1 2 4 8 16 7 24 31}
out=gpurun_out/dbg; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
v='M:rational S:fast'
args=("use_tc=True $v")
for b in $bits; do args+=("use_tc=True $v D:NNB_TC_DBG=$b"); done
timeout 900 python scripts/ab_kw.py $cfg $batch "${args[@]}" 2>&1 | grep "replay\|_tc_" | cut -c1-100 > $out/ab_cfg$cfg.log
cat $out/ab_cfg$cfg.log
