#!/bin/bash
# Tensor-pipe utilization of client training over one timed C3 round (north star: ">= 50 %
# tensor-pipe utilization in client training"): sm__pipe_tc_cycles_active (elapsed-normalised)
# and the duration of every launch; the time-weighted mean is the round's tensor-pipe utilization.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=7253
timeout 2400 ncu --metrics sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum \
  --clock-control none -s $((3 * L + 2)) -c $L --csv --log-file gpurun_out/tcutil_c3.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-c2 > gpurun_out/ncu_tcutil.log 2>&1
echo "tcutil exit $?"
