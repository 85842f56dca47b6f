# A/B of tcgen05 tuning options on cfg1 plus per-launch profiles of cfg2/cfg3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python scripts/ab_kw.py 1 65536 'wide=True' 'tmem_a=False' 'tmem_a=False abuf=2' 'csplit=False' 'wide_chunk=8' 'abuf=2' > gpurun_out/ab_cfg1.log 2>&1
timeout 300 python scripts/prof_net.py --config 3 --batch 256 > gpurun_out/prof_cfg3.log 2>&1
timeout 300 python scripts/prof_net.py --config 2 --batch 1024 > gpurun_out/prof_cfg2.log 2>&1
timeout 300 python scripts/prof_net.py --config 0 --batch 4096 > gpurun_out/prof_cfg0.log 2>&1
timeout 300 python scripts/prof_net.py --config 4 --batch 64 > gpurun_out/prof_cfg4.log 2>&1
