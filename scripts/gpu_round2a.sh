#!/bin/bash
# first round-2 GPU pass: new production-size parity tests, the full GPU suite, bench
cd "$(dirname "$0")/.."
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests/test_gpu_production.py -x -q -s -m gpu > gpurun_out/prod.log 2>&1; echo "prod rc=$?" >> gpurun_out/prod.log
timeout 900 python -m pytest tests -q -m gpu --deselect tests/test_gpu_production.py > gpurun_out/gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
