#!/bin/bash
# Bench the C3 line under each value of one env knob: VAR=name VALUES="a b c" bash scripts/gpu_sweep_env.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s_build.log 2>&1 || { echo build failed; exit 1; }
for v in $VALUES; do
  env $VAR=$v timeout 600 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/s_bench_$v.json 2> gpurun_out/s_bench_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/s_bench_$v.json').readline()); k=d['kernels']
print('$VAR=$v', round(d['ms_per_step'],2), 'c2', round(d['c2']['ms_per_step'],3) if isinstance(d.get('c2'),dict) else None, {n: k[n]['ms'] for n in ('fc1_dw_sgd','fc1_fwd','conv1_fwd','conv1_dw')})"
done
