#!/bin/bash
# One gpurun call producing the round's measurement evidence under gpurun_out/:
#   bench.json / bench_ref.json   the contract lines (ours, --impl reference)
#   launches.csv                  ncu launch list (gpu__time_duration) of one timed C2 round
#   traffic.csv                   dram bytes of every launch of the tensor-core kernels in one round
#   full_<k>.ncu-rep              one --set full capture per listed kernel (A=100 full wave)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref exit $?" >> gpurun_out/bench_ref.err
# launches per round (from the bench line) -> skip the warm-up rounds of a --steps 1 --warmup 3 run
L=$(python -c "import json; d=json.loads(open('gpurun_out/bench.json').readline()); print(d['gpu_launches'] // d['steps'])" 2>/dev/null || echo 2600)
SKIP=$(( 3 * L + 10 ))
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $SKIP -c $(( L + 20 )) --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "launches exit $?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k "regex:k_conv|k_fc1|k_dw|k_head|k_pack|k_fedavg" -s $SKIP -c $(( L + 20 )) --csv \
  --log-file gpurun_out/traffic.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_traffic.log 2>&1
echo "traffic exit $?"
for k in ${FULL_KERNELS:-k_fc1_bwd_tc k_conv5_tc k_conv2_dw_tc k_conv1_dw_tc k_conv1_fwd_tc}; do
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s 1 -c 1 \
    -o gpurun_out/full_$k python scripts/wave_once.py 100 3 2 > gpurun_out/ncu_full_$k.log 2>&1
  echo "full $k exit $?"
done
ls -la gpurun_out | tail -20
head -c 1500 gpurun_out/bench.json; echo; head -c 800 gpurun_out/bench_ref.json
