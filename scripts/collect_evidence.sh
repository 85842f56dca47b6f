#!/bin/bash
# Copy a gpu_final.sh run (gpurun_out/TAG, gpurun_out/prof_TAG) into profiles/ under the round's
# names and regenerate the README tables.  usage: bash scripts/collect_evidence.sh r02b [r02]
tag=${1:-r02b}; rnd=${2:-r02}
src=gpurun_out/$tag; prof=gpurun_out/prof_$tag
cp $src/bench.json profiles/${rnd}_bench.json
cp $src/bench_ref.json profiles/${rnd}_bench_reference.json
for c in 0 1 2 3 4; do cp $src/launches_cfg$c.csv profiles/${rnd}_launches_cfg$c.csv; done
for f in $prof/${tag}_cfg*.ncu-rep; do
  b=$(basename $f .ncu-rep); n=${b#${tag}_}
  cp $f profiles/${rnd}_$n.ncu-rep
  cp $prof/${b}_raw.csv profiles/${rnd}_${n}_ncu_raw.csv
  cp $prof/${b}_details.csv profiles/${rnd}_${n}_ncu_details.csv
done
python scripts/profiles_tables.py profiles/${rnd}_bench.json profiles/${rnd}_bench_reference.json > /tmp/profiles_tables.md
echo "tables in /tmp/profiles_tables.md"
python - <<'PY'
import re
p = "profiles/README.md"
s = open(p).read()
t = open("/tmp/profiles_tables.md").read()
a = s.index("## Headline")
b = s.index("## Round-2 changes")
open(p, "w").write(s[:a] + t.rstrip() + "\n\n" + s[b:])
PY
