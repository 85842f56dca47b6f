python -c "import __graft_entry__ as g; g.build()" > /dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-extra > gpurun_out/multi.json 2> gpurun_out/multi.err; echo rc=$?
tail -5 gpurun_out/multi.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/multi_ref.json 2> gpurun_out/multi_ref.err; echo rc=$?
cat gpurun_out/multi_ref.json | head -c 600
