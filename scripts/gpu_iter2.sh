#!/bin/bash
# Quick loop: build, layer tests of the kernels under work, a C3 bench line, ncu --set full of KERNELS.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/j_build.log 2>&1 || { echo build failed; tail gpurun_out/j_build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "${TESTK:-conv1}" > gpurun_out/j_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/j_tests.log
if [ -n "${PARITY:-}" ]; then
  timeout 1200 python -m pytest -x -q -s ${PARITY} > gpurun_out/j_parity.log 2>&1; echo "parity rc=$?"
  grep -E "C3:|C2|passed|failed|Error" gpurun_out/j_parity.log | tail -8
fi
timeout 600 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/j_bench.json 2> gpurun_out/j_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/j_bench.json').readline()); print(d['ms_per_step'], d['value'], d.get('c2',{}).get('ms_per_step') if isinstance(d.get('c2'),dict) else None)
for k,v in d['kernels'].items(): print(k, v['ms'], v['frac'])
"
for k in ${KERNELS:-}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 1 -c 1 \
    -o gpurun_out/j_full_$k python scripts/wave_once.py 100 3 2 > gpurun_out/j_ncu_$k.log 2>&1
  echo "full $k exit $?"
done
