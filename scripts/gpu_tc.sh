set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python -m pytest tests/test_gpu_configs.py -x -q -k tensor_core 2>&1 | tail -30
