mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for c in "3 64" "3 32" "2 64" "2 8" "0 256" "1 512" "1 1024" "4 4"; do
timeout 600 python scripts/ab_kw.py $c 'tc_min_rows=2048' 'tc_min_rows=512' 'tc_min_rows=128' > gpurun_out/tcmin_${c// /_}.log 2>&1
done
