mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python scripts/ab_kw.py 1 65536 'corr_bf16=True D:NNB_CB16_WB=0' 'corr_bf16=True D:NNB_CB16_WB=0 D:NNB_SPIN_WAIT=1' 'corr_bf16=True D:NNB_CB16_WB=0 D:NNB_SPIN_WAIT=1 D:NNB_TC_DBG=31' 'corr_bf16=True D:NNB_CB16_WB=0 D:NNB_TC_DBG=27' 'corr_bf16=True D:NNB_CB16_WB=0 D:NNB_TC_DBG=29' > gpurun_out/cb16d_ab.log 2>&1
