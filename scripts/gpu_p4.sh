python -c "import __graft_entry__ as g; g.build()" > /dev/null
python scripts/prof_net.py --config 4 --batch 64 2>&1 | tail -14
python scripts/prof_net.py --config 2 --batch 1024 2>&1 | tail -12
