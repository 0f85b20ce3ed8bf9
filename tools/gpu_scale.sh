#!/bin/bash
# Scaling run on one box: the multi-GPU tests, then the bench at N = 1, 2, 4
# (torchrun, one process per GPU, NCCL) — run via gpurun --gpus 4.
O=gpurun_out
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -k "multi_gpu or lpt_shards" > $O/pytest_multi.log 2>&1; echo pytest=$?; tail -3 $O/pytest_multi.log
NS=${NS:-"1 2 4"}
for n in $NS; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline --no-dense --no-wall-time --no-sweep > $O/scale_$n.log 2>&1; echo n=$n rc=$?
done
