#!/bin/bash
# round-2 GPU pass: green-context partitions + peer aggregation tests, heterogeneous emulation
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q -s > gpurun_out/peer.log 2>&1; echo "peer rc=$?" >> gpurun_out/peer.log
timeout 600 python scripts/hetero_emulation.py --clients 1000 --rounds 6 --out gpurun_out/hetero_f4.json > gpurun_out/hetero.log 2>&1; echo "hetero rc=$?" >> gpurun_out/hetero.log
timeout 600 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench8.json 2>/dev/null
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 600 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench32.json 2>/dev/null
