python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -4
for c in 0 4 3; do
  case $c in 0) B=4096;; 2) B=1024;; 3) B=256;; 4) B=64;; esac
  python scripts/prof_net.py --config $c --batch $B 2>&1 | grep -E "replay|direct"
  python scripts/prof_net.py --config $c --batch 1 2>&1 | grep -E "replay"
done
