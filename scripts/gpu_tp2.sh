python -c "import __graft_entry__ as g; g.build()" > /dev/null
python scripts/prof_net.py --config 4 --batch 64 2>&1 | grep -E "replay|_tc_|direct"
python scripts/prof_net.py --config 4 --batch 64 --no-tmem-a 2>&1 | grep -E "replay|_tc_"
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -4
python scripts/tc_error.py 2>&1 | grep "tc=True"
for c in 0 2 3; do
  case $c in 0) B=4096;; 2) B=1024;; 3) B=256;; 4) B=64;; esac
  python scripts/prof_net.py --config $c --batch $B 2>&1 | grep -E "replay|_tc_|direct"
done
