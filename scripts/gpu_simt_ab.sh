mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for c in "3 256" "2 1024" "0 4096" "3 64"; do
timeout 600 python scripts/ab_kw.py $c 'wide=True' 'tc_min_rows=10**9' > gpurun_out/simt_${c// /_}.log 2>&1
done
