#!/bin/bash
# GPU tests + per-launch profile of the given "cfg batch" pairs
python -c "import __graft_entry__ as g; g.build()" >/dev/null || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in "$@"; do set -- $c; echo "== cfg$1 b$2"; timeout 300 python scripts/prof_net.py --config $1 --batch $2; done
