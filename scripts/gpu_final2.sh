#!/bin/bash
# Round-end evidence in one gpurun call (after scripts/gpu_final.sh): GPU suite, smoke, the bench
# lines (default C3 with C2, e2e and cpu_baseline; reference arm; C4, C5, C1), the fc1_bwd DRAM
# traffic of one timed C3 round + the launch list of that round, --set full of the top kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/f_gpu.txt 2>&1
nproc > gpurun_out/f_nproc.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/f_gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/f_gpu_tests.log
tail -3 gpurun_out/f_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f_smoke.log
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?" >> gpurun_out/f_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
timeout 900 python bench.py --config C4 --no-cpu --no-e2e --steps 3 > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err
timeout 900 python bench.py --config C5 --no-cpu --no-e2e --steps 2 > gpurun_out/f_bench_c5.json 2> gpurun_out/f_bench_c5.err
timeout 600 python bench.py --config C1 --no-cpu --no-e2e --steps 10 > gpurun_out/f_bench_c1.json 2> gpurun_out/f_bench_c1.err
bash scripts/gpu_traffic.sh
for k in k_fc1_bwd_tc k_conv1_fwd_tc k_conv1_dw_tc k_fc1_fwd_tc; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 1 -c 1 \
    -o gpurun_out/f_full_$k python scripts/wave_once.py 100 3 2 > gpurun_out/f_ncu_full_$k.log 2>&1
done
echo done
