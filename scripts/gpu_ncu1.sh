#!/bin/bash
# one ncu --set full capture: gpu_ncu1.sh OUTNAME KERNEL_REGEX prof_net-args...
out=$1; kre=$2; shift 2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python scripts/prof_net.py "$@" --reps 2 > gpurun_out/${out}_plain.txt 2>&1 || { tail gpurun_out/${out}_plain.txt; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 -o gpurun_out/$out \
    python scripts/prof_net.py "$@" --reps 2 > gpurun_out/${out}_ncu.log 2>&1
tail -2 gpurun_out/${out}_ncu.log
