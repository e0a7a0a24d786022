#!/bin/bash
# multi-rank checks on one GPU: tests + co-located torchrun bench
free -g | head -2; nproc
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x 2>&1 | tail -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 2 --warmup 3 --size 16384 --nb 1024 --mxp-n 16384 --e2e-steps 1 --no-cusolver 2>&1 | tail -5 > gpurun_out/bench_coloc2.log
tail -c 3000 gpurun_out/bench_coloc2.log
timeout 600 python bench.py --steps 2 --warmup 3 --size 16384 --nb 1024 --mxp-n 16384 --e2e-steps 1 --no-cusolver --no-cpu 2>&1 | tail -3 > gpurun_out/bench_1.log
tail -c 3000 gpurun_out/bench_1.log
