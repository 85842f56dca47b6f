#!/bin/bash
# ncu --set full of each config's dominant kernel at its bench batch (default
# options), plus raw-page CSV exports.  usage: gpurun -- bash scripts/gpu_profiles.sh TAG
tag=${1:-r02}
out=gpurun_out/prof_$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || exit 1
for spec in "0 4096 conv3x3_direct_1" "1 65536 dense_tc_3" "2 1024 sep3x3_narrow_1" "3 256 sep3x3_narrow_1" "3 256 conv1x1_dw3x3_tc" "4 64 conv3x3_tc_4"; do
  set -- $spec
  name=${tag}_cfg$1_$3
  timeout 300 python scripts/prof_net.py --config $1 --batch $2 --mode default --reps 1 > $out/$name.prof.log 2>&1 || continue
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:nnb_u0._$3 -c 1 -o $out/$name \
    python scripts/prof_net.py --config $1 --batch $2 --mode default --reps 1 > $out/$name.ncu.log 2>&1
  ncu -i $out/$name.ncu-rep --page raw --csv > $out/${name}_raw.csv 2>/dev/null
  ncu -i $out/$name.ncu-rep --page details --csv > $out/${name}_details.csv 2>/dev/null
done
