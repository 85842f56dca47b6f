mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python scripts/ab_kw.py 1 65536 'corr_bf16=True D:NNB_CB16_WB=0' 'corr_bf16=True D:NNB_CB16_WB=0 D:NNB_TC_DBG=30' 'corr_bf16=True D:NNB_CB16_WB=0 D:NNB_TC_DBG=2' 'corr_bf16=True D:NNB_CB16_WB=0 D:NNB_TC_DBG=3' 'corr_bf16=True D:NNB_CB16_WB=0 D:NNB_TC_DBG=31' 'corr_bf16=True D:NNB_CB16_WB=0 wide_chunk=32' 'corr_bf16=True D:NNB_CB16_WB=0 wide_bk=16' > gpurun_out/cb16c_ab.log 2>&1
