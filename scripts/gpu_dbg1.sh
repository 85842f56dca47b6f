#!/bin/bash
out=gpurun_out/dbg1; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
v='M:rational S:fast'
timeout 900 python scripts/ab_kw.py 1 65536 "pw_dw=True $v" "pw_dw=True $v D:NNB_TC_DBG=1" "pw_dw=True $v D:NNB_TC_DBG=4" "pw_dw=True $v D:NNB_TC_DBG=8" "pw_dw=True $v D:NNB_TC_DBG=16" "pw_dw=True $v D:NNB_TC_DBG=7" "pw_dw=True $v D:NNB_TC_DBG=24" "pw_dw=True $v D:NNB_TC_DBG=32" 2>&1 | grep "replay\|_tc_" | cut -c1-60 > $out/ab.log; cat $out/ab.log
