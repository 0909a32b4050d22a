#!/bin/bash
# Iteration check: build, conv1 layer tests, the whole GPU suite, one bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/i_build.log 2>&1 || { echo build failed; tail gpurun_out/i_build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "conv1" > gpurun_out/i_conv1.log 2>&1; echo "conv1 tests rc=$?"; tail -15 gpurun_out/i_conv1.log
[ "${QUICK:-0}" = 1 ] && exit 0
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/i_gpu.log 2>&1; echo "gpu suite rc=$?"; tail -5 gpurun_out/i_gpu.log
timeout 600 python bench.py --no-cpu --steps 5 > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/i_bench.json').readline()); print(d['ms_per_step'], d['value'], d.get('c2',{}).get('ms_per_step') if isinstance(d.get('c2'),dict) else None)
for k,v in d['kernels'].items(): print(k, v)
"
