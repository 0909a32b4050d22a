#!/bin/bash
# conv1 / conv2 --set full captures at a full wave (A = 100) + one bench line (current code).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p_build.log 2>&1
timeout 600 python bench.py --no-cpu --steps 5 > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err; echo "bench exit $?" >> gpurun_out/p_bench.err
for k in k_conv1_fwd_tc k_conv1_dw_tc k_conv5_tc; do
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s 1 -c 1 \
    -o gpurun_out/p_full_$k python scripts/wave_once.py 100 3 2 > gpurun_out/p_ncu_full_$k.log 2>&1
  echo "full $k exit $?"
done
