mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "bf16 or wide" > gpurun_out/cb16f_t.log 2>&1
timeout 900 python scripts/tc_error_wide.py 'corr_bf16=False' 'corr_bf16=True' 'corr_bf16=True D:NNB_CB16_WB=1' > gpurun_out/cb16f_err_wide.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
