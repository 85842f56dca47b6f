python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
for pdl in 0 1; do
for c in 0 1 2 3 4; do
  case $c in 0) B=4096;; 1) B=65536;; 2) B=1024;; 3) B=256;; 4) B=64;; esac
  echo "pdl=$pdl cfg$c b=$B $(NNB_PDL=$pdl python scripts/prof_net.py --config $c --batch $B 2>&1 | grep replay)   b=1 $(NNB_PDL=$pdl python scripts/prof_net.py --config $c --batch 1 2>&1 | grep replay)"
done; done
