mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python scripts/act_err.py > gpurun_out/elu_err.log 2>&1
timeout 600 python scripts/ab_kw.py 1 65536 'wide=True' 'D:NNB_ELU_LIBM=1' 'csplit=False head=False' > gpurun_out/elu_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_fuzz_tc.py -q -x > gpurun_out/elu_t.log 2>&1
