mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for c in "1 512" "1 256" "1 128" "1 64" "1 32" "3 16" "0 64"; do
timeout 600 python scripts/ab_kw.py $c 'tc_min_rows=512' 'tc_min_rows=128 small_dense_rows=128' 'tc_min_rows=128 small_dense_rows=32' 'tc_min_rows=128 small_dense_rows=8' > gpurun_out/sdr_${c// /_}.log 2>&1
done
