#!/bin/bash
out=gpurun_out/dbg; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 600 python scripts/ab_kw.py 3 256 'pw_dw=True M:rational S:fast' 'pw_dw=True M:rational S:fast D:NNB_TC_DBG=1' 'pw_dw=True M:rational S:fast D:NNB_TC_DBG=2' 'pw_dw=True M:rational S:fast D:NNB_TC_DBG=4' 'pw_dw=True M:rational S:fast D:NNB_TC_DBG=8' 'pw_dw=True M:rational S:fast D:NNB_TC_DBG=15' 'pw_dw=True M:rational S:fast D:NNB_TC_DBG=31' 2>&1 | grep "replay\|u10_\|u11_\|u15_\|u16_\|u07_" | cut -c1-90 > $out/ab.log; cat $out/ab.log
