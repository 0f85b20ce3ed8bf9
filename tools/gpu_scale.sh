#!/bin/bash
# Scaling run on one box: bench at N = 1, 2, 4 (torchrun, NCCL) + GPU tests.
O=gpurun_out
nvidia-smi topo -m > $O/topo.txt 2>&1
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$?
NS=${NS:-"1 2 4"}
for n in $NS; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 5 --warmup 3 --no-cpu-baseline --no-dense --no-wall-time > $O/scale_$n.log 2>&1; echo n=$n rc=$?
done
