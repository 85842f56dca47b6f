mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python scripts/ab_sep.py 2 1024 32,32 64,64 > gpurun_out/ab_sep2.log 2>&1
timeout 600 python scripts/ab_sep.py 3 256 32,32 64,64 > gpurun_out/ab_sep3.log 2>&1
timeout 600 python scripts/ab_sep.py 2 1 32,32 64,64 > gpurun_out/ab_sep2_b1.log 2>&1
