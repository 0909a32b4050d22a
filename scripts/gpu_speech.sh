#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_speech_tc.py -x -q > gpurun_out/speech_tc.log 2>&1; echo "rc=$?" >> gpurun_out/speech_tc.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -x -q > gpurun_out/gpu_parity.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_parity.log
timeout 900 python -m pytest tests/test_gpu_production.py -x -q -s -k speech > gpurun_out/prod_speech.log 2>&1; echo "rc=$?" >> gpurun_out/prod_speech.log
timeout 600 python bench.py --config C4 --no-cpu --no-e2e --steps 2 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
