python -c "import __graft_entry__ as g; g.build()" > /dev/null
python scripts/tc_error.py 2>&1 | tail -12
python scripts/prof_net.py --config 1 --mode exact 2>&1 | tail -6
