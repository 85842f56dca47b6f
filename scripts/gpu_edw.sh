#!/bin/bash
# pw -> dw epilogue fusion: its tests, cfg3 with and without it, then the GPU suite
out=gpurun_out/edw; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "pointwise_with_depthwise_epilogue" > $out/t_edw.log 2>&1; echo "rc=$?" >> $out/t_edw.log
tail -5 $out/t_edw.log
timeout 300 python scripts/prof_net.py --config 3 --batch 256 --mode default > $out/prof_cfg3.log 2>&1; tail -25 $out/prof_cfg3.log
timeout 300 python scripts/ab_kw.py 3 256 'pw_dw=True M:rational S:fast' 'pw_dw=False M:rational S:fast' 2>&1 | grep -v '^   ' > $out/ab_cfg3.log; tail -8 $out/ab_cfg3.log
timeout 2400 python -m pytest tests -m gpu -q -x > $out/gpu_tests.log 2>&1; echo "rc=$?" >> $out/gpu_tests.log; tail -4 $out/gpu_tests.log
