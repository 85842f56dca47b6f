#!/bin/bash
# several ncu --set full captures: gpu_ncu_many.sh TAG "CFG BATCH KERNEL_REGEX" ...
tag=$1; shift
out=gpurun_out/ncu_$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail $out/build.log; exit 1; }
for spec in "$@"; do
  set -- $spec
  name=cfg$1_$3
  timeout 300 python scripts/prof_net.py --config $1 --batch $2 --mode default --reps 1 > $out/$name.prof.log 2>&1 || { tail -3 $out/$name.prof.log; continue; }
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$3 -c 1 -o $out/$name \
    python scripts/prof_net.py --config $1 --batch $2 --mode default --reps 1 > $out/$name.ncu.log 2>&1
  ncu -i $out/$name.ncu-rep --page raw --csv > $out/${name}_raw.csv 2>/dev/null
  ncu -i $out/$name.ncu-rep --page details --csv > $out/${name}_details.csv 2>/dev/null
  ncu -i $out/$name.ncu-rep --page source --csv > $out/${name}_source.csv 2>/dev/null
  rm -f $out/$name.ncu-rep
  echo "$name done"
done
