#!/bin/bash
# roofline.traffic of bench.py: DRAM bytes of EVERY launch of the dominant kernel class in one
# timed round of the default workload (C3), so the per-launch mean covers the same launches as the
# bench's achieved bandwidth; plus the launch list (gpu__time_duration) of that whole round.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
W=${WAVES:-252}   # waves (= fc1_bwd launches) per C3 round on one GPU; 3 warm-up rounds precede the timed one
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k "regex:k_fc1_bwd_tc" -s $((3 * W)) -c $W --csv --log-file gpurun_out/traffic_fc1bwd.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-c2 > gpurun_out/ncu_tr.log 2>&1
echo "traffic exit $?"
L=${LAUNCHES:-2472}
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3 * L + 2)) -c $L --csv \
  --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-c2 > gpurun_out/ncu_l.log 2>&1
echo "launches exit $?"
