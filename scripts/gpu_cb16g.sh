mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for c in "4 64" "3 256" "0 4096" "2 1024"; do
timeout 600 python scripts/ab_kw.py $c 'corr_bf16=True' 'corr_bf16="all"' 'corr_bf16="all" cb16_w4=False' > gpurun_out/cb16g_${c// /_}.log 2>&1
done
