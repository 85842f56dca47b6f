set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python scripts/prof_net.py --config 1 --mode exact > gpurun_out/prof_exact.txt 2>&1
python scripts/prof_net.py --config 1 --mode rational > gpurun_out/prof_rational.txt 2>&1
cat gpurun_out/prof_exact.txt gpurun_out/prof_rational.txt
python scripts/prof_net.py --config 1 --reps 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dense_tc_1 -s 1 -c 1 -o gpurun_out/r01_dense_tc python scripts/prof_net.py --config 1 --reps 2 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
