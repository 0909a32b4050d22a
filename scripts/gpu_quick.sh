#!/bin/bash
# quick check of a kernel change: layer tests + C2/C3 parity + bench lines (C3 default with C2)
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_speech_tc.py tests/test_gpu_parity.py -x -q > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
timeout 600 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
