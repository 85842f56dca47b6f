set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?
tail -c 2000 gpurun_out/bench.err
python bench.py --steps 2 --warmup 1 --no-extra > gpurun_out/b_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-extra > gpurun_out/ncu.log 2>&1; echo ncu_rc=$?
python scripts/prof_net.py --config 1 --reps 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:nnb_u00_dense_tc_ -s 1 -c 1 -o gpurun_out/r01_dense_tc python scripts/prof_net.py --config 1 --reps 2 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
