set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15
python scripts/prof_net.py --config 1 --mode exact 2>&1 | tail -6
python scripts/prof_net.py --config 1 --mode rational 2>&1 | tail -6
