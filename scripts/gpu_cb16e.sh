mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "bf16 or wide or dense" > gpurun_out/cb16e_t.log 2>&1
timeout 600 python scripts/tc_error_wide.py 'corr_bf16=False' 'corr_bf16=True' > gpurun_out/cb16e_err_wide.log 2>&1
timeout 900 python -m pytest tests/ -q -x -m gpu > gpurun_out/cb16e_all.log 2>&1
