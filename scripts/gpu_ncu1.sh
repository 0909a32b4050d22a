#!/bin/bash
# --set full capture of the listed kernels at a full wave (A = 100 clients x 32 samples).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/n_build.log 2>&1 || { echo build failed; exit 1; }
timeout 120 python scripts/wave_once.py 100 3 2 > gpurun_out/n_wave.log 2>&1; echo "wave rc=$?"; cat gpurun_out/n_wave.log
for k in ${KERNELS:-k_conv1_fwd_tc k_conv1_dw_tc}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 1 -c 1 \
    -o gpurun_out/n_full_$k python scripts/wave_once.py 100 3 2 > gpurun_out/n_ncu_$k.log 2>&1
  echo "full $k exit $?"
done
