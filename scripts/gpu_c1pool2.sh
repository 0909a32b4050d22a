#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -k "conv1 or C3_full or C2_full or cnn_round" > gpurun_out/cnn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cnn_tests.log
