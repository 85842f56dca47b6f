mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python scripts/ab_kw.py 1 65536 'wide=True' 'D:NNB_TC_DBG=1' 'D:NNB_TC_DBG=24' 'D:NNB_TC_DBG=31' > gpurun_out/l3.log 2>&1
bash scripts/gpu_multi.sh > gpurun_out/multi.log 2>&1; echo multi_rc=$?
