set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?
tail -c 3000 gpurun_out/bench.err
cat gpurun_out/bench.json
python bench.py --steps 2 --warmup 1 --no-extra > gpurun_out/b_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-extra > gpurun_out/ncu.log 2>&1; echo ncu_rc=$?
tail -5 gpurun_out/ncu.log
