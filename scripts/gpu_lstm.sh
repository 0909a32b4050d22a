#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py -q -s -k "lstm" > gpurun_out/lstm.log 2>&1; echo "rc=$?" >> gpurun_out/lstm.log
true
