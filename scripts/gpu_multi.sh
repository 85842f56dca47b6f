#!/bin/bash
# torchrun paths of bench.py on one GPU (2 ranks share it: a functional check
# of the distributed plumbing -- barrier, MAX over ranks, per-rank parity).
out=gpurun_out/multi; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-extra > $out/weak.json 2> $out/weak.err; echo "weak rc=$?" >> $out/weak.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --config 3 --global-batch 256 --steps 3 --warmup 3 --no-extra > $out/strong.json 2> $out/strong.err; echo "strong rc=$?" >> $out/strong.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 --no-extra > $out/ref.json 2> $out/ref.err; echo "ref rc=$?" >> $out/ref.err
