#!/bin/bash
# Re-measure after the last kernel change: GPU suite, smoke, bench default (C3 + C2, e2e, cpu
# baseline), reference arm, C4, launch list of one timed C3 round, conv1 fwd --set full.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/h5_build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/h5_gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/h5_gpu_tests.log
tail -3 gpurun_out/h5_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h5_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/h5_smoke.log
timeout 900 python bench.py > gpurun_out/h5_bench.json 2> gpurun_out/h5_bench.err; echo "bench rc=$?" >> gpurun_out/h5_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/h5_bench_ref.json 2> gpurun_out/h5_bench_ref.err
timeout 900 python bench.py --config C4 --no-cpu --no-e2e --steps 3 > gpurun_out/h5_bench_c4.json 2> gpurun_out/h5_bench_c4.err
L=$(python -c "import json; d=json.loads(open('gpurun_out/h5_bench.json').readline()); print(d['round_stats']['kernels'])" 2>/dev/null || echo 7252)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3 * L + 2)) -c $L --csv \
  --log-file gpurun_out/h5_launches_c3.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-c2 > gpurun_out/h5_ncu_l.log 2>&1
echo "launches exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_conv1_fwd_tc" -s 1 -c 1 \
  -o gpurun_out/h5_full_k_conv1_fwd_tc python scripts/wave_once.py 100 3 2 > gpurun_out/h5_ncu_full.log 2>&1
echo done
