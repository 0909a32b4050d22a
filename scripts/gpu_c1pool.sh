#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q > gpurun_out/cnn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cnn_tests.log
timeout 900 python -m pytest tests/test_gpu_production.py -x -q -s -k C2 > gpurun_out/prod_c2.log 2>&1; echo "rc=$?" >> gpurun_out/prod_c2.log
timeout 600 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
KNOB_SETS=C2,C3 timeout 900 python scripts/knob_sweep.py "" "FL_GROUPS=3" > gpurun_out/knobs.txt 2>&1
