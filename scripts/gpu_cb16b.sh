mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python scripts/ab_kw.py 1 65536 'corr_bf16=True' 'corr_bf16=True D:NNB_CB16_WB=0' 'corr_bf16=True D:NNB_TC_DBG=4' 'corr_bf16=True D:NNB_TC_DBG=8' 'corr_bf16=True D:NNB_TC_DBG=24' 'corr_bf16=True D:NNB_TC_DBG=1' > gpurun_out/cb16b_ab.log 2>&1
timeout 600 python scripts/tc_error_wide.py 'corr_bf16=True' > gpurun_out/cb16b_err_wide.log 2>&1
