python -c "import __graft_entry__ as g; g.build()" > /dev/null
for c in 0 2 3 4; do
  case $c in 0) B=4096;; 2) B=1024;; 3) B=256;; 4) B=64;; esac
  echo "=== cfg$c batch $B"; python scripts/prof_net.py --config $c --batch $B 2>&1 | tail -40
  echo "=== cfg$c batch 1"; python scripts/prof_net.py --config $c --batch 1 2>&1 | tail -40
done
