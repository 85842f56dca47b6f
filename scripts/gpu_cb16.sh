# bf16 correction products (corr_bf16) vs the 3xTF32 default: speed and error
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python scripts/ab_kw.py 1 65536 'corr_bf16=False' 'corr_bf16=True' > gpurun_out/cb16_ab.log 2>&1
timeout 600 python scripts/tc_error_wide.py 'corr_bf16=False' 'corr_bf16=True' > gpurun_out/cb16_err_wide.log 2>&1
timeout 600 python scripts/tc_error.py 'corr_bf16=False' 'corr_bf16=True' 'corr_bf16=True pair=False wide=False' > gpurun_out/cb16_err.log 2>&1
timeout 600 python scripts/ab_kw.py 4 64 'corr_bf16=False' 'corr_bf16=True' > gpurun_out/cb16_ab4.log 2>&1
