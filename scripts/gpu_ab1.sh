#!/bin/bash
out=gpurun_out/ab1; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
v='M:rational S:fast'
timeout 900 python scripts/ab_kw.py 1 65536 "wide=True $v" "wide=False $v" "wide=False tmem_a=False $v" "wide=False tmem_a=False corr_bf16=True $v" "wide=True wide_chunk=8 $v" "wide=True early_mma=False $v" "wide=False tmem_a=False abuf=2 corr_bf16=True pair=False $v" 2>&1 | grep "replay\|_tc_" | cut -c1-150 > $out/ab.log; cat $out/ab.log
