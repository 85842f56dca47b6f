mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python scripts/ab_kw.py 1 65536 'a_prefetch=0' 'a_prefetch=2' 'a_prefetch=4' 'a_prefetch=8' 'a_prefetch=16' > gpurun_out/apf.log 2>&1
