#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 > gpurun_out/torchrun_cfg1.json 2> gpurun_out/torchrun_cfg1.err; echo "rc=$?" >> gpurun_out/torchrun_cfg1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/torchrun_ref.json 2> gpurun_out/torchrun_ref.err; echo "rc=$?" >> gpurun_out/torchrun_ref.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --config cfg3 --gpus 1 --steps 2 --warmup 3 --run-steps 8000 > gpurun_out/torchrun_cfg3.json 2> gpurun_out/torchrun_cfg3.err; echo "rc=$?" >> gpurun_out/torchrun_cfg3.err
