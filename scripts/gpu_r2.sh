#!/bin/bash
# Round-2 GPU pass: build, pytest -m gpu, bench (both arms), ncu launch lists of
# every config.  usage: gpurun -- bash scripts/gpu_r2.sh TAG [tests|bench|launches]...
tag=${1:-r2}; shift
stages=${*:-tests bench launches}
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; tail $out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
for s in $stages; do
case $s in
tests)
  timeout 3000 python -m pytest tests -m gpu -q -x > $out/gpu_tests.log 2>&1; echo "tests rc=$?" >> $out/gpu_tests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log ;;
bench)
  timeout 1200 python bench.py --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $out/bench.err
  timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?" >> $out/bench_ref.err ;;
launches)
  for cb in "0 4096" "1 65536" "2 1024" "3 256" "4 64"; do
    set -- $cb
    timeout 300 python scripts/prof_net.py --config $1 --batch $2 --mode default > $out/prof_cfg$1.log 2>&1 && \
    timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
      --log-file $out/launches_cfg$1.csv python scripts/prof_net.py --config $1 --batch $2 --mode default --reps 1 > $out/ncu_cfg$1.log 2>&1
  done ;;
esac
done
