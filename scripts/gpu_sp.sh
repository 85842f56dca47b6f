#!/bin/bash
out=gpurun_out/sp; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "sep_narrow" > $out/t_sep.log 2>&1; echo "rc=$?" >> $out/t_sep.log
tail -5 $out/t_sep.log
for cb in "3 256" "2 1024"; do set -- $cb
timeout 300 python scripts/ab_kw.py $1 $2 'sep_geo=None M:rational S:fast' 2>&1 | head -6 > $out/ab_cfg$1.log; cat $out/ab_cfg$1.log; done
timeout 300 python scripts/ab_kw.py 3 256 'sep_geo=(2,2,2) M:rational S:fast' 'sep_geo=(2,2,1) M:rational S:fast' 'sep_geo=(4,2,1) M:rational S:fast' 2>&1 | grep "replay\|sep3x3" > $out/ab_cfg3_geo.log; cat $out/ab_cfg3_geo.log
timeout 300 python scripts/ab_kw.py 2 1024 'sep_geo=(3,2,1) M:rational S:fast' 'sep_geo=(3,2,2) M:rational S:fast' 2>&1 | grep "replay\|sep3x3" > $out/ab_cfg2_geo.log; cat $out/ab_cfg2_geo.log
