python -c "import __graft_entry__ as g; g.build()" > /dev/null
python scripts/prof_net.py --config 4 --batch 64 --reps 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv3x3_tc_10 -s 1 -c 1 -o gpurun_out/r01_conv_tc10 python scripts/prof_net.py --config 4 --batch 64 --reps 2 > gpurun_out/ncu4.log 2>&1
tail -2 gpurun_out/ncu4.log
