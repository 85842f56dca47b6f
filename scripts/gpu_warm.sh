#!/bin/bash
out=gpurun_out/warm; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "pointwise_with_depthwise_epilogue" > $out/t_edw.log 2>&1; echo "rc=$?" >> $out/t_edw.log; tail -3 $out/t_edw.log
for cb in "3 256" "1 65536" "4 64" "2 1024" "0 4096"; do set -- $cb
timeout 600 python scripts/ab_kw.py $1 $2 'pw_dw=True M:rational S:fast' 'pw_dw=True M:rational S:fast D:NNB_TC_DBG=64' 'pw_dw=True M:rational S:fast' 'pw_dw=True M:rational S:fast D:NNB_TC_DBG=64' 2>&1 | grep "replay\|_tc_" | cut -c1-90 > $out/ab$1.log; grep replay $out/ab$1.log; done
head -12 $out/ab3.log
