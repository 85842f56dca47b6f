python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -30
